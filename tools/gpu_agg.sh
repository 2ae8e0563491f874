timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "aggregate or q1 or q6 or q3 or q5 or q9 or stream or engine" > gpurun_out/pytest_agg.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_agg.log
TQ_OPS=aggregate_high_card,aggregate_q1 python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
python tools/profile_q3_local.py --sf 10 --reps 3 2>&1 | grep "q3 whole"
