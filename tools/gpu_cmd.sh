timeout 900 python -m pytest tests/test_gpu_field.py -x -q -k "full_size and C5" -s 2>&1 | tail -4
