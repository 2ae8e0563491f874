python tools/time_queries.py --sf 10 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "join_queries or semi or probe" 2>&1 | tail -2
