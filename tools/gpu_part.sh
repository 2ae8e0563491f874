TQ_HOST_TIMING=1 python tools/part_host.py
