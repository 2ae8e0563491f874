"""Stage-by-stage device timing of the single-GPU Q3 plan (config 3, queries.q3).

    python tools/profile_q3_local.py --sf 10 [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.expr import Col  # noqa: E402
from paper_2508_05029_b200.ops import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ctx = Context(0)
    st = torch.cuda.ExternalStream(ctx.stream())
    t = {n: ctx.datagen(Q.TABLE_IDS[n], a.sf) for n in ("customer", "orders", "lineitem")}
    ctx.sync()
    for rep in range(a.reps):
        marks = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            marks.append((name, e))
        ctx.profile(True)
        mark("start")
        ct = ctx.pipeline_build(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Q.C_CUSTKEY], semi=True)
        mark("customer build")
        of = ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE), Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)],
                                [3], [])
        mark("orders probe")
        ot = ctx.join_build(of, [0])
        mark("orders_f build")
        j = ctx.pipeline_probe(ot, t["lineitem"], Col(Q.L_SHIPDATE) > 9204, [Col(Q.L_ORDERKEY), Q.REV], [0], [1, 2])
        mark("lineitem probe")
        out = ctx.aggregate_execute(j, [2, 0, 1], [(Q.AGG_SUM, 3)])
        mark("aggregate")
        torch.cuda.synchronize()
        ctx.sync()
        prof = ctx.profile_report()
        ctx.profile(False)
        print(f"rep {rep}: orders_f={of.rows} join={j.rows} groups={out.rows}")
        for (n0, e0), (n1, e1) in zip(marks, marks[1:]):
            print(f"  {n1:40s} {e0.elapsed_time(e1):8.3f} ms")
        print("  total", marks[0][1].elapsed_time(marks[-1][1]))
        print("  kernels:", {k: (v[0], round(v[1], 3)) for k, v in prof.items()})
        for x in (of, j, out):
            x.free()
        ct.free()
        ot.free()
    # whole query, events around queries.q3; host phase timers on the last rep
    import ctypes as C
    import time
    from paper_2508_05029_b200.ops import lib
    ht = os.environ.get("TQ_HOST_TIMING") == "1"
    for rep in range(4):
        if ht and rep == 3:
            lib().tq_host_timing_report(C.create_string_buffer(1 << 16), 1 << 16)  # drop earlier reps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h0 = time.perf_counter()
        r = Q.q3(ctx, t["customer"], t["orders"], t["lineitem"])
        e1.record(st)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        print("q3 whole:", round(e0.elapsed_time(e1), 3), "ms device;", round((h1 - h0) * 1e3, 3), "ms host")
        r.free()
    if ht:
        buf = C.create_string_buffer(1 << 16)
        lib().tq_host_timing_report(buf, len(buf))
        print(buf.value.decode())
    print("jit:", ctx.jit_report())
    ctx.close()


if __name__ == "__main__":
    main()
