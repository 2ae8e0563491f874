timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fused_exchange.py -m gpu -x -q -k "partition or fused or semi or q3" > gpurun_out/pytest_part.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_part.log
python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
