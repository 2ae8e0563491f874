"""Kernel times of the Q3 probes (orders -> customer table, lineitem -> orders_f
table) under the current env knobs (TQ_JIT_DEFS, TQ_MAXSTAGES, --ctas).

    TQ_JIT_DEFS=TQ_PB=4 python tools/probe_exp.py --sf 10
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
    ap.add_argument("--ctas", type=int, default=0)
    a = ap.parse_args()
    ctx = Context(0, ctas_per_sm=a.ctas)
    st = torch.cuda.ExternalStream(ctx.stream())
    t = {n: ctx.datagen(Q.TABLE_IDS[n], a.sf) for n in ("customer", "orders", "lineitem")}
    ct = ctx.pipeline_build(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Q.C_CUSTKEY], semi=True)
    of = ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                            [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE), Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])
    ot = ctx.join_build(of, [0])
    cf = ctx.pipeline_materialize(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Col(Q.C_CUSTKEY)])
    ct2 = ctx.join_build(cf, [0])  # table sized for the filtered rows
    res = {}
    for name, fn in (("orders_probe", lambda: ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                                                  [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE),
                                                                   Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])),
                     ("no_pass", lambda: ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 0,
                                                            [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE),
                                                             Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])),
                     ("one_out_col", lambda: ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                                                [Col(Q.O_CUSTKEY)], [0], [])),
                     ("orderkey_probe(miss)", lambda: ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                                                          [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE),
                                                                           Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)],
                                                                          [0], [])),
                     ("no_pred", lambda: ctx.pipeline_probe(ct, t["orders"], None,
                                                            [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE),
                                                             Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])),
                     ("orders_probe_small_table", lambda: ctx.pipeline_probe(
                         ct2, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                         [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE), Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)], [3], [])),
                     ("lineitem_probe", lambda: ctx.pipeline_probe(ot, t["lineitem"], Col(Q.L_SHIPDATE) > 9204,
                                                                    [Col(Q.L_ORDERKEY), Q.REV], [0], [1, 2]))):
        fn().free()
        ctx.sync()
        ctx.profile(True)
        for _ in range(5):
            fn().free()
        ctx.sync()
        prof = ctx.profile_report()
        ctx.profile(False)
        n, ms = prof.get("pipe_probe1", prof.get("pipe_emit"))
        r = fn()
        res[name] = (round(ms / n * 1e3, 1), r.rows)
        r.free()
    print(os.environ.get("TQ_JIT_DEFS", "-"), os.environ.get("TQ_MAXSTAGES", "-"), a.ctas, res, ctx.jit_report()["failed"])
    ctx.close()


if __name__ == "__main__":
    main()
