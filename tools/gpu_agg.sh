timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "aggregate or q1 or q6 or q3 or stream" > gpurun_out/pytest_agg.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_agg.log
python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
