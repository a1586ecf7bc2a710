set -x
timeout 300 python tools/stage_times.py C5 > gpurun_out/r1e_stages.log 2>&1
python tools/profile_one.py C5 1 > gpurun_out/r1e_p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_tiles -c 2 -o gpurun_out/r1e_tiles python tools/profile_one.py C5 1 > gpurun_out/r1e_ncu.log 2>&1
cat gpurun_out/r1e_stages.log
