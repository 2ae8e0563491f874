for ps in 1 4 8 16; do echo "passes=$ps"; TQ_BUILD_PASSES=$ps TQ_OPS=join_build,join_probe_pkfk python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"; done
echo auto; TQ_OPS=join_build python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
TQ_BUILD_PASSES=4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "join or semi or probe or build" 2>&1 | tail -1
