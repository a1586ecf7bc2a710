timeout 600 python bench.py --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/bg.log 2>&1; tail -1 gpurun_out/bg.log | cut -c1-400; tail -1 gpurun_out/bg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d['gpu_launches'], d['roofline']['frac'])"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
