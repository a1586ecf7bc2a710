set -x
timeout 600 python -m pytest tests/test_gpu_field.py -x -q -s > gpurun_out/r1q_field.log 2>&1
tail -30 gpurun_out/r1q_field.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1q_pytest.log 2>&1
tail -3 gpurun_out/r1q_pytest.log
for c in C5; do timeout 300 python tools/stage_times.py $c; done > gpurun_out/r1q_stages.log 2>&1
cat gpurun_out/r1q_stages.log
