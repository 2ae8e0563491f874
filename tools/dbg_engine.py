import sys, os
sys.path[:0] = ['/root/repo', '/root/repo/oracle']
import oracle as O
from paper_2508_05029_b200.ops import Context, engine_run_query
ctx = Context(0)
if os.environ.get("NOJIT"): ctx.set_jit(False)
q = 3
tabs = {t: ctx.datagen(t, 0.05) for t in O.QUERY_TABLES[q]}
got, m = engine_run_query(ctx, q, tabs, compute_threads=1, batch_rows=1 << 30)
print("jit" if not os.environ.get("NOJIT") else "nojit", {k: v["rows_out"] for k, v in m["ops"].items()}, flush=True)
