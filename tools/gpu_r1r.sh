set -x
timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_field.py -x -q -s > gpurun_out/r1r_new.log 2>&1
tail -30 gpurun_out/r1r_new.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1r_pytest.log 2>&1
tail -3 gpurun_out/r1r_pytest.log
for m in tiles field; do timeout 300 python tools/stage_times.py C5 $m; done > gpurun_out/r1r_stages.log 2>&1
timeout 300 python tools/stage_times.py C4 field >> gpurun_out/r1r_stages.log 2>&1
cat gpurun_out/r1r_stages.log
