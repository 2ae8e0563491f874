"""Experiment: Q1-shaped aggregation with fewer accumulators, at 2 vs 3+
pipeline stages (TQ_MAXSTAGES), to see whether ring depth limits the kernel.

    TQ_MAXSTAGES=2 python tools/stage_exp.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.queries import AGG_COUNT_STAR, AGG_SUM  # noqa: E402
from paper_2508_05029_b200.ops import Context  # noqa: E402

ctx = Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
li = ctx.datagen(1, 10.0)
scan = li.select(Q.Q1_SCAN)
variants = {
    "6acc": (Q.Q1_KEYS, Q._Q1_PARTIAL_AGGS),
    "4acc": (Q.Q1_KEYS, [(AGG_SUM, 2), (AGG_SUM, 3), (AGG_SUM, 5), (AGG_COUNT_STAR, 0)]),
    "2acc": (Q.Q1_KEYS, [(AGG_SUM, 6), (AGG_COUNT_STAR, 0)]),
    "cnt": (Q.Q1_KEYS, [(AGG_COUNT_STAR, 0)]),
    "nokey6": ([], Q._Q1_PARTIAL_AGGS),
    "nokeycnt": ([], [(AGG_COUNT_STAR, 0)]),
}
only = os.environ.get("VARIANTS")
for name, (keys, aggs) in variants.items():
    if only and name not in only.split(","):
        continue
    fn = lambda: ctx.pipeline_aggregate(scan, Q._Q1_SCAN_PRED, Q._Q1_SCAN_EXPRS, keys, aggs)  # noqa: E731
    for _ in range(3):
        fn().free()
    ctx.sync()
    ctx.profile(True)
    for _ in range(10):
        fn().free()
    ctx.sync()
    prof = ctx.profile_report()
    ctx.profile(False)
    ms = prof["pipe_agg"][1] / prof["pipe_agg"][0]
    print(f"{name} stages<={os.environ.get('TQ_MAXSTAGES', '6')}: pipe_agg {ms:.3f} ms "
          f"({scan.rows * 88 / ms / 1e6:.0f} GB/s of the 88 B/row scan)", flush=True)
