"""Host-side cost of one operator call on tiny inputs (pure launch/sync/
bookkeeping overhead), wall clock with the stream drained before and after.

    python tools/op_overhead.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.expr import Col  # noqa: E402
from paper_2508_05029_b200.ops import Context  # noqa: E402

ctx = Context(0)
t = {n: ctx.datagen(Q.TABLE_IDS[n], 0.001) for n in ("customer", "orders", "lineitem")}
ct0 = ctx.pipeline_build(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Q.C_CUSTKEY])
ops = {
    "materialize(filter)": lambda: ctx.pipeline_materialize(t["orders"], Col(Q.O_ORDERDATE) < 9204, [Col(Q.O_ORDERKEY)]),
    "pipeline_build": lambda: ctx.pipeline_build(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Q.C_CUSTKEY]),
    "pipeline_probe": lambda: ctx.pipeline_probe(ct0, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                                 [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE)], [1], []),
    "aggregate": lambda: ctx.aggregate_execute(t["orders"], [1], [(Q.AGG_SUM, 0)]),
    "q1_scan": lambda: Q.q1_scan(ctx, t["lineitem"].select(Q.Q1_SCAN)),
}
for name, fn in ops.items():
    for _ in range(5):
        fn().free()
    ctx.sync()
    if os.environ.get("TQ_HOST_TIMING") == "1":
        import ctypes as C
        from paper_2508_05029_b200.ops import lib
        lib().tq_host_timing_report(C.create_string_buffer(1 << 16), 1 << 16)  # drop the warm-up
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        fn().free()
    ctx.sync()
    print(f"{name:22s} {(time.perf_counter() - t0) / n * 1e6:8.1f} us/call", flush=True)
    if os.environ.get("TQ_HOST_TIMING") == "1":
        import ctypes as C
        from paper_2508_05029_b200.ops import lib
        buf = C.create_string_buffer(1 << 16)
        lib().tq_host_timing_report(buf, len(buf))
        print("  " + buf.value.decode().replace("\n", "\n  ").rstrip(), flush=True)

if os.environ.get("PROFILE"):
    import cProfile
    import pstats
    fn = ops[os.environ["PROFILE"]]
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        fn().free()
    ctx.sync()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)
