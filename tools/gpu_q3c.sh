mkdir -p gpurun_out/jitdump
TQ_JIT_DUMP=gpurun_out/jitdump TQ_HOST_TIMING=1 python tools/profile_q3_local.py --sf 10 --reps 3 > gpurun_out/q3local.log 2>&1; echo q3=$?
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "join or probe or build or q3 or q5 or q9 or partition or engine" > gpurun_out/pytest_join.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_join.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q3_launches.csv python tools/profile_q3_local.py --sf 10 --reps 1 > gpurun_out/q3ncu.log 2>&1; echo ncu=$?
