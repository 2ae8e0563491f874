timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "join or probe or build or q3 or q5 or q9 or engine or exact" > gpurun_out/pytest_join.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_join.log
TQ_OPS=join_build python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
python tools/profile_q3_local.py --sf 10 --reps 3 2>&1 | grep "q3 whole"
