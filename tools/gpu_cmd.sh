timeout 300 python tools/real_times.py
timeout 900 python -m pytest tests -m gpu -x -q -k "real or full" 2>&1 | tail -2
