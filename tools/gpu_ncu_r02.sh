#!/bin/bash
# Round-2 ncu evidence (run under gpurun, one GPU): the bench's launch list,
# a --set full capture of the Q1 aggregate kernel, and one --set full capture
# per SPEC operator of tools/op_roofline.py (the two setup launches skipped).
set -u
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --suite 0 > $O/r02_ncu_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tq_jit_main --launch-skip 4 -c 1 \
  -o $O/r02_ncu_q1 python bench.py --steps 2 --warmup 1 --suite 0 > $O/r02_ncu_q1.log 2>&1
for op in filter_execute project_execute hash_partition join_build join_probe_pkfk pipeline_probe_filtered; do
  TQ_OPS=$op timeout 600 ncu --set full --clock-control none -k regex:"tq_jit_main|k_" --launch-skip 2 -c 3 \
    -o $O/r02_ncu_op_$op python tools/op_roofline.py > $O/r02_ncu_op_$op.log 2>&1
done
ls -la $O/*.ncu-rep
