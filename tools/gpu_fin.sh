timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "aggregate or q1 or q6 or q3 or q5 or q9 or stream or engine or join_queries" 2>&1 | tail -2
python tools/profile_q3_local.py --sf 10 --reps 3 2>&1 | grep -A8 "rep 2"
python tools/time_queries.py --sf 10 2>&1 | tail -3
TQ_OPS=aggregate_high_card,aggregate_q1 python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
