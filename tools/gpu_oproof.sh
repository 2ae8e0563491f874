python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"
