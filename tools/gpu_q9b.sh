timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "join_queries or semi or probe" 2>&1 | grep -E "Error|error|FAILED|assert" | head -20
