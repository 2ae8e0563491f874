timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -x -q -k "join or probe or build or q3 or q5 or q9 or engine or exact or semi" > gpurun_out/pytest_join.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_join.log
python tools/profile_q3_local.py --sf 10 --reps 3 2>&1 | grep -A8 "rep 2"
TQ_OPS=join_build,join_probe_pkfk,pipeline_probe_filtered python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -x -q > gpurun_out/pytest_mgpu.log 2>&1; echo pytest_mgpu=$?
tail -2 gpurun_out/pytest_mgpu.log
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/profile_q3_dist.py --sf 100 --fused > gpurun_out/dist_fused_n$n.log 2>&1; echo n=$n rc=$?
done
