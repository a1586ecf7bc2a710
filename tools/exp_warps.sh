# Expander-warp count experiment: rebuild with each (default, field) count, time C5 stages.
set -x
for v in "8 6" "8 8" "8 5"; do
  set -- $v
  SE1P_NVCC_EXTRA="-DSE1P_EXP_WARPS=$1 -DSE1P_EXP_WARPS_FIELD=$2" timeout 300 python -c "from paper_1611_09538_b200 import build as b; b.build(force=True)" || continue
  echo "== exp=$1 field=$2"
  timeout 200 python tools/stage_times.py C5 field
  timeout 200 python tools/stage_times.py C4 field
done > gpurun_out/exp_warps2.log 2>&1
cat gpurun_out/exp_warps2.log | grep -v "^+"
