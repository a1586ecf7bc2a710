set -x
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/r1h_dist.log 2>&1
tail -25 gpurun_out/r1h_dist.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1h_pytest.log 2>&1
tail -5 gpurun_out/r1h_pytest.log
