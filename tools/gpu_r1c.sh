set -x
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r1c_fullsize.log 2>&1
for c in C3 C4 C5; do timeout 300 python tools/stage_times.py $c; timeout 300 python tools/stage_times.py $c v1; done > gpurun_out/r1c_stages.log 2>&1
nproc > gpurun_out/r1c_nproc.log
