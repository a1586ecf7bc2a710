timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "odd_and_large" 2>&1 | tail -8
