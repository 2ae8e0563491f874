#!/bin/bash
# ncu --set full of the two-pass filter / hash partition after the direct-load
# COUNT pass (one GPU): COUNT + EMIT of each operator of tools/op_roofline.py
O=gpurun_out
for op in filter_execute hash_partition; do
  TQ_OPS=$op timeout 600 ncu --set full --import-source on --clock-control none -k regex:tq_jit_main --launch-skip 2 -c 2 \
    -o $O/r02_ncu_cd_$op python tools/op_roofline.py > $O/r02_ncu_cd_$op.log 2>&1
  echo "$op rc=$?"
done
