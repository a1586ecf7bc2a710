for c in C5 C4; do timeout 300 python tools/stage_times.py $c tiles; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
