mkdir -p gpurun_out/fin
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -q -m gpu --deselect tests/test_multigpu.py > gpurun_out/fin/pytest_gpu_1.log 2>&1; echo pytest=$?
tail -3 gpurun_out/fin/pytest_gpu_1.log
timeout 900 python bench.py > gpurun_out/fin/bench_n1.json 2> gpurun_out/fin/bench_n1.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/fin/ref.json 2> gpurun_out/fin/ref.err; echo ref=$?
