mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dist1_launches.csv python tools/profile_q3_dist.py --sf 25 --fused --reps 1 > gpurun_out/dist1_ncu.log 2>&1; echo ncu=$?
