mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "join or probe or build or q3 or q5 or q9 or partition or engine" > gpurun_out/pytest_join.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_join.log
python tools/probe_exp.py --sf 10 2>&1 | tail -1
TQ_HOST_TIMING=1 python tools/profile_q3_local.py --sf 10 --reps 3 > gpurun_out/q3local.log 2>&1; echo q3=$?
