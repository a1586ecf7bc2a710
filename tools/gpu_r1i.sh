set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1i_pytest.log 2>&1
tail -5 gpurun_out/r1i_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/r1i_bench.log 2>&1
cat gpurun_out/r1i_bench.log
