"""Device time of the SF10 join queries (as bench.py's suite) + parity vs the oracle at SF 0.05.

    python tools/time_queries.py [--sf 10]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.columnar import assert_batches_equal  # noqa: E402
from paper_2508_05029_b200.ops import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10)
    a = ap.parse_args()
    ctx = Context(0)
    st = torch.cuda.ExternalStream(ctx.stream())
    import oracle as O
    for q in (3, 5, 9):
        names = Q.QUERY_TABLES[q]
        small = {n: ctx.datagen(Q.TABLE_IDS[n], 0.05) for n in names}
        got = Q.run_join_query(ctx, q, small).to_host()
        want = O.query(q, {Q.TABLE_IDS[n]: O.datagen(Q.TABLE_IDS[n], 0.05) for n in names}, 4)
        assert_batches_equal(got, want)
        t = {n: ctx.datagen(Q.TABLE_IDS[n], a.sf) for n in names}
        Q.run_join_query(ctx, q, t).free()
        ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = Q.run_join_query(ctx, q, t)
            e1.record(st)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            r.free()
        print(f"q{q} sf{a.sf:g}: {statistics.median(ms):.3f} ms (parity ok at SF0.05)", flush=True)
        for v in list(t.values()) + list(small.values()):
            v.free()
    ctx.close()


if __name__ == "__main__":
    main()
