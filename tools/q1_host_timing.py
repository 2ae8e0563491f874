import os, sys, time
sys.path.insert(0, '.')
import ctypes as C
from paper_2508_05029_b200 import queries
from paper_2508_05029_b200.ops import Context, lib
ctx = Context(0)
li = ctx.datagen(1, 10.0)
scan = li.select(queries.Q1_SCAN)
for _ in range(5):
    queries.q1_scan(ctx, scan).free()
ctx.sync()
ctx.profile(True)
t0 = time.perf_counter()
N = 20
for _ in range(N):
    queries.q1_scan(ctx, scan).free()
ctx.sync()
t1 = time.perf_counter()
print("wall per step ms", (t1 - t0) * 1e3 / N)
print(ctx.profile_report())
buf = C.create_string_buffer(1 << 16)
lib().tq_host_timing_report(buf, len(buf))
print(buf.value.decode())
