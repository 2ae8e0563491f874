"""Wall vs device time per Q1 step (host overhead between kernels)."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2508_05029_b200 import queries
from paper_2508_05029_b200.ops import Context
ctx = Context(0)
li = ctx.datagen(1, 10.0)
scan = li.select(queries.Q1_SCAN)
st = torch.cuda.ExternalStream(ctx.stream())
for _ in range(5):
    queries.q1_scan(ctx, scan).free()
ctx.sync()
ctx.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
t0 = time.perf_counter()
e0.record(st)
for _ in range(n):
    queries.q1_scan(ctx, scan).free()
e1.record(st)
torch.cuda.synchronize()
ctx.sync()
wall = (time.perf_counter() - t0) / n * 1e3
prof = ctx.profile_report()
print(f"wall/step {wall:.3f} ms  device/step {e0.elapsed_time(e1)/n:.3f} ms  kernels", prof)
t0 = time.perf_counter()
for _ in range(n):
    queries.q1_scan(ctx, scan).free()
print(f"wall/step (no profiling) {(time.perf_counter() - t0) / n * 1e3:.3f} ms")
