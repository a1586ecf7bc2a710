set -x
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-seconds 10 > gpurun_out/r1o_bench.log 2>&1
cat gpurun_out/r1o_bench.log
$B > gpurun_out/r1o_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1o_launches.csv $B > gpurun_out/r1o_ncu1.log 2>&1
