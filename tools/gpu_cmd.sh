REAL_ONLY=1 bash tools/exp_variant.sh rf "" "-DSE1P_REAL_F32_REJECT=0"
timeout 900 python -m pytest tests -m gpu -x -q -k "real or full or field or planner" 2>&1 | tail -2
