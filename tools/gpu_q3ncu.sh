mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:tq_jit_main --launch-skip 1 --launch-count 1 -o gpurun_out/q3_oprobe -f python tools/profile_q3_local.py --sf 10 --reps 1 > gpurun_out/q3ncu1.log 2>&1; echo a=$?
ncu --set full --import-source on --clock-control none -k regex:tq_jit_main --launch-skip 3 --launch-count 1 -o gpurun_out/q3_lprobe -f python tools/profile_q3_local.py --sf 10 --reps 1 > gpurun_out/q3ncu2.log 2>&1; echo b=$?
