mkdir -p gpurun_out
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > gpurun_out/bench_n$n.log 2>&1; echo n=$n rc=$?
done
