TQ_HOST_TIMING=1 TQ_OPS=hash_partition python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
TQ_HOST_TIMING=1 TQ_OPS=filter_execute python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
