for ms in 6 24; do echo "MAXSTAGES=$ms"; TQ_MAXSTAGES=$ms python tools/op_roofline.py --sf 10 2>&1 | grep -v "^{"; done
