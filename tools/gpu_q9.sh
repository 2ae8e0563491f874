timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "join or semi or probe or engine or q3 or q5 or q9" 2>&1 | tail -2
python tools/time_queries.py --sf 10 2>&1 | tail -4
TQ_HOST_TIMING=1 python - <<'PY'
import os, sys, ctypes as C, torch
sys.path.insert(0, os.getcwd())
from paper_2508_05029_b200 import queries as Q
from paper_2508_05029_b200.ops import Context, lib
ctx = Context(0)
st = torch.cuda.ExternalStream(ctx.stream())
t = {n: ctx.datagen(Q.TABLE_IDS[n], 10) for n in Q.QUERY_TABLES[9]}
for rep in range(3):
    ctx.profile(True)
    Q.run_join_query(ctx, 9, t).free()
    ctx.sync()
    prof = ctx.profile_report(); ctx.profile(False)
print({k: (v[0], round(v[1], 3)) for k, v in prof.items()})
PY
