"""Small driver for ncu captures: one query over device-generated lineitem.

    python tools/profile_query.py --query q1 --sf 10 --reps 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_05029_b200 import queries  # noqa: E402
from paper_2508_05029_b200.ops import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--query", default="q1")
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    ctx = Context(0)
    li = ctx.datagen(1, a.sf)
    if a.query == "q1":
        scan = li.select(queries.Q1_SCAN)
        fn = lambda: queries.q1_scan(ctx, scan)  # noqa: E731
    else:
        scan = li.select(queries.Q6_SCAN)
        fn = lambda: queries.q6_scan(ctx, scan)  # noqa: E731
    for _ in range(a.reps):
        r = fn()
        print(r.to_host().to_rows()[:2])
        r.free()
    ctx.sync()
    ctx.close()


if __name__ == "__main__":
    main()
