mkdir -p gpurun_out
python tools/profile_q3_local.py --sf 10 --reps 3 > gpurun_out/q3local.log 2>&1; echo q3=$?
python bench.py --suite 0 --steps 10 --warmup 3 > gpurun_out/bench_s0.log 2>&1; echo b=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q3_launches.csv python tools/profile_q3_local.py --sf 10 --reps 1 > gpurun_out/q3ncu.log 2>&1; echo ncu=$?
