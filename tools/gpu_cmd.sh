REAL_ONLY=1 bash tools/exp_variant.sh rt "" "-DSE1P_REAL_TABLE=0"
timeout 900 python -m pytest tests -m gpu -x -q -k "real or full or field or planner or smoke" 2>&1 | tail -2
