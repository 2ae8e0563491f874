"""Host-phase timing of one hash_partition call (TQ_HOST_TIMING=1)."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.expr import Col  # noqa: E402
from paper_2508_05029_b200.ops import Context, lib  # noqa: E402

ctx = Context(0)
li = ctx.datagen(Q.TABLE_IDS["lineitem"], 10)
L = li.select([Q.L_ORDERKEY, Q.L_EXTPRICE, Q.L_DISCOUNT, Q.L_SHIPDATE])
proj = ctx.project_execute(L, [Col(0), Col(1) * (Q.Dec(100) - Col(2))])
for i in range(4):
    if i == 3:
        lib().tq_host_timing_report(C.create_string_buffer(1 << 16), 1 << 16)
    ctx.sync()
    t0 = time.perf_counter()
    b, offs = ctx.hash_partition(proj, [0], 8)
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    b.free()
    t3 = time.perf_counter()
    print(f"call {1e3*(t1-t0):.3f} ms, sync {1e3*(t2-t1):.3f} ms, free {1e3*(t3-t2):.3f} ms")
buf = C.create_string_buffer(1 << 16)
lib().tq_host_timing_report(buf, len(buf))
print(buf.value.decode())
