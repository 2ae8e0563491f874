"""Stage-by-stage device timing of the config-4 Q3 shuffle plan on one GPU
(world=1 communicator).   python tools/profile_q3.py --sf 50"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.expr import Col  # noqa: E402
from paper_2508_05029_b200.ops import Comm, Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=50)
    ap.add_argument("--nparts", type=int, default=2)
    a = ap.parse_args()
    ctx = Context(0)
    comm = Comm(ctx, 0, 1, Comm.unique_id())
    st = torch.cuda.ExternalStream(ctx.stream())
    t = {n: ctx.datagen(Q.TABLE_IDS[n], a.sf) for n in ("customer", "orders", "lineitem")}
    ctx.sync()
    for rep in range(2):
        marks = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            marks.append((name, e))
        ctx.profile(True)
        mark("start")
        cf = ctx.pipeline_materialize(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Col(Q.C_CUSTKEY)])
        mark("customer filter")
        cb, _ = comm.allgather(cf)
        mark("customer allgather")
        ct = ctx.join_build(cb, [0])
        mark("customer build")
        of = ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE), Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])
        mark("orders probe")
        op, ooff = ctx.hash_partition(of, [0], a.nparts)
        mark("orders partition")
        lp, loff = ctx.pipeline_partition(t["lineitem"], Col(Q.L_SHIPDATE) > 9204, [Col(Q.L_ORDERKEY), Q.REV], [0],
                                          a.nparts)
        mark("lineitem filter+project+partition")
        lrx, _ = comm.exchange(lp, [0, lp.rows])
        mark("lineitem exchange (self)")
        ot = ctx.join_build(op, [0])
        mark("orders_f build")
        j = ctx.pipeline_probe(ot, lrx, None, None, [0], [1, 2])
        mark("lineitem probe")
        out = ctx.aggregate_execute(j, [2, 0, 1], [(Q.AGG_SUM, 3)])
        mark("aggregate")
        torch.cuda.synchronize()
        ctx.sync()
        prof = ctx.profile_report()
        ctx.profile(False)
        print(f"rep {rep}: rows lineitem={t['lineitem'].rows} orders_f={of.rows} lineitem_f={lp.rows} join={j.rows} groups={out.rows}")
        for (n0, e0), (n1, e1) in zip(marks, marks[1:]):
            print(f"  {n1:40s} {e0.elapsed_time(e1):8.3f} ms")
        print("  total", marks[0][1].elapsed_time(marks[-1][1]))
        print("  kernels:", {k: (v[0], round(v[1], 3)) for k, v in prof.items()})
        for x in (cf, cb, of, op, lp, lrx, j, out):
            x.free()
        ct.free()
        ot.free()
    comm.close()
    ctx.close()


if __name__ == "__main__":
    main()
