mkdir -p gpurun_out/fin
timeout 1200 python -m pytest tests/test_multigpu.py -q -m gpu -rs > gpurun_out/fin/pytest_multigpu_w4.log 2>&1; echo mg=$?
tail -3 gpurun_out/fin/pytest_multigpu_w4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 > gpurun_out/fin/bench_n2.json 2> gpurun_out/fin/bench_n2.err; echo b2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 > gpurun_out/fin/bench_n4.json 2> gpurun_out/fin/bench_n4.err; echo b4=$?
