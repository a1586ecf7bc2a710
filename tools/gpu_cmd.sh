REAL_ONLY=1 bash tools/exp_variant.sh real2 "" "-DSE1P_REAL_WARP_CELLS=0"
timeout 900 python -m pytest tests -m gpu -x -q -k "real or full or field" 2>&1 | tail -2
