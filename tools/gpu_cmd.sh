timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | grep -E "Error|assert|error" | head -20
