for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q -k "budget" 2>&1 | tail -1; done
TQ_OPS=aggregate_high_card python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
