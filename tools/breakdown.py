"""Per-query device-time breakdown at SF10 on one GPU: whole-query CUDA-event
time next to the pipeline kernels' own event times (ctx.profile), so the
host/launch/sync overhead between kernels is visible.

    python tools/breakdown.py [--sf 10] [--reps 5] [--queries q1,q6,q3,q5,q9]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2508_05029_b200 import queries  # noqa: E402
from paper_2508_05029_b200.ops import Context  # noqa: E402


def q3_stages(ctx, st, t):
    from paper_2508_05029_b200.expr import Col
    Q = queries
    for rep in range(3):
        marks = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            marks.append((name, e))
        mark("start")
        ct = ctx.pipeline_build(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Q.C_CUSTKEY])
        mark("customer filter+build")
        of = ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE), Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])
        mark(f"orders filter+probe -> {of.rows} rows")
        ot = ctx.join_build(of, [0])
        mark("orders_f build")
        j = ctx.pipeline_probe(ot, t["lineitem"], Col(Q.L_SHIPDATE) > 9204, [Col(Q.L_ORDERKEY), Q.REV], [0], [1, 2])
        mark(f"lineitem filter+probe -> {j.rows} rows")
        out = ctx.aggregate_execute(j, [2, 0, 1], [(Q.AGG_SUM, 3)])
        mark(f"aggregate -> {out.rows} groups")
        torch.cuda.synchronize()
        if rep == 2:
            for (n0, e0), (n1, e1) in zip(marks, marks[1:]):
                print(f"  {n1:45s} {e0.elapsed_time(e1):7.3f} ms")
            print(f"  total {marks[0][1].elapsed_time(marks[-1][1]):.3f} ms", flush=True)
        for x in (ct, of, ot, j, out):
            x.free()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--queries", default="q1,q6,q3,q5,q9")
    ap.add_argument("--stages", action="store_true", help="Q3 operator-by-operator timing")
    a = ap.parse_args()
    ctx = Context(0)
    st = torch.cuda.ExternalStream(ctx.stream())
    names = ["customer", "orders", "lineitem", "supplier", "part", "partsupp", "nation", "region"]
    t = {n: ctx.datagen(queries.TABLE_IDS[n], a.sf) for n in names}
    li1 = t["lineitem"].select(queries.Q1_SCAN)
    li6 = t["lineitem"].select(queries.Q6_SCAN)
    fns = {"q1": lambda: queries.q1_scan(ctx, li1), "q6": lambda: queries.q6_scan(ctx, li6)}
    for q in (3, 5, 9):
        fns[f"q{q}"] = (lambda q=q: queries.run_join_query(ctx, q, t))
    if a.stages:
        q3_stages(ctx, st, t)
        return
    for name in a.queries.split(","):
        fn = fns[name]
        for _ in range(3):
            fn().free()
        ctx.sync()
        ctx.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(a.reps):
            fn().free()
        e1.record(st)
        torch.cuda.synchronize()
        ctx.sync()
        total = e0.elapsed_time(e1) / a.reps
        prof = ctx.profile_report()
        ctx.profile(False)
        kern = sum(v[1] for v in prof.values()) / a.reps
        parts = ", ".join(f"{k} {v[0] / a.reps:g}x {v[1] / a.reps:.3f}" for k, v in sorted(prof.items()))
        print(f"{name}: {total:.3f} ms/query  pipeline kernels {kern:.3f} ms ({100 * kern / total:.0f}%)  [{parts}]",
              flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
