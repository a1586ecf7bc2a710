for m in tiles field; do timeout 300 python tools/stage_times.py C5 $m; done
timeout 300 python tools/stage_times.py C4 tiles
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
