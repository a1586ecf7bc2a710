set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r1_pytest.log
timeout 300 python tools/stress.py C4 10 > gpurun_out/r1_stress_c4.log 2>&1
timeout 300 python tools/stress.py C5 5 > gpurun_out/r1_stress_c5.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/r1_bench.log 2>&1
tail -3 gpurun_out/*.log
