#!/bin/bash
# Round-2 ncu evidence (run under gpurun, one GPU): the bench's launch list,
# a --set full capture of the Q1 aggregate kernel, and one --set full capture
# per SPEC operator of tools/op_roofline.py.  op_roofline launches two
# pipeline kernels before the operators (the project that feeds the
# partition / aggregate, the orders table the probes use): skipped.
set -u
O=gpurun_out
if [ "${NCU_OPS_ONLY:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --suite 0 > $O/r02_ncu_launches.log 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:tq_jit_main --launch-skip 4 -c 1 \
    -o $O/r02_ncu_q1 python bench.py --steps 2 --warmup 1 --suite 0 > $O/r02_ncu_q1.log 2>&1
fi
for op in filter_execute hash_partition project_execute join_build join_probe_pkfk pipeline_probe_filtered; do
  n=1; case $op in filter_execute|hash_partition) n=2;; esac
  TQ_OPS=$op timeout 600 ncu --set full --clock-control none -k regex:tq_jit_main --launch-skip 2 -c $n \
    -o $O/r02_ncu_op_$op python tools/op_roofline.py > $O/r02_ncu_op_$op.log 2>&1
done
TQ_OPS=aggregate_high_card timeout 600 ncu --set full --clock-control none -k regex:"tq_jit_main|k_agg_final|k_key_range" \
  --launch-skip 2 -c 3 -o $O/r02_ncu_op_aggregate_high_card python tools/op_roofline.py > $O/r02_ncu_op_agg_hc.log 2>&1
ls -la $O/*.ncu-rep
