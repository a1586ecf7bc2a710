# A/B of compile-time variants: tools/exp_variant.sh TAG "<defines A>" "<defines B>" ...
# rebuilds per variant and times C5/C4 stages (potential and field); restores the default build.
tag=$1; shift
for v in "$@"; do
  SE1P_NVCC_EXTRA="$v" timeout 300 python -c "from paper_1611_09538_b200 import build as b; b.build(force=True)" || continue
  echo "== [$v]"
  if [ -n "$REAL_ONLY" ]; then timeout 300 python tools/real_times.py; continue; fi
  timeout 200 python tools/stage_times.py C5
  [ -z "$NO_FIELD" ] && timeout 200 python tools/stage_times.py C5 field
  timeout 200 python tools/stage_times.py C4
  if [ -n "$RUN_PARITY" ]; then timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py -x -q 2>&1 | tail -2; fi
done > gpurun_out/exp_$tag.log 2>&1
cat gpurun_out/exp_$tag.log
python -c "from paper_1611_09538_b200 import build as b; b.build(force=True)"
