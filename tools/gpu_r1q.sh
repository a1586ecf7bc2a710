set -x
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-seconds 10 > gpurun_out/r1q_bench.log 2>&1
$B > gpurun_out/r1q_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1q_launches.csv $B > gpurun_out/r1q_ncu1.log 2>&1
python tools/profile_one.py C5 1 > gpurun_out/r1q_p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_tiles -c 2 -o gpurun_out/r1q_tiles python tools/profile_one.py C5 1 > gpurun_out/r1q_ncu2.log 2>&1
