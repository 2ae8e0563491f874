mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_fused_exchange.py -m gpu -x -q > gpurun_out/pytest_mgpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_mgpu.log
for n in 1 2 4; do
TQ_HOST_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/profile_q3_dist.py --sf 100 --fused > gpurun_out/dist_fused_n$n.log 2>&1; echo n=$n rc=$?
done
