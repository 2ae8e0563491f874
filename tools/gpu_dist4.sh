for n in 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/profile_q3_dist.py --sf 100 --fused > gpurun_out/dist_fused_n$n.log 2>&1; echo n=$n rc=$?
done
