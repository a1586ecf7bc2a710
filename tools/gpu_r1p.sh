set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1p_pytest.log 2>&1
tail -2 gpurun_out/r1p_pytest.log
for c in C4 C5; do timeout 300 python tools/stage_times.py $c; done > gpurun_out/r1p_stages.log 2>&1
cat gpurun_out/r1p_stages.log
