B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/r1v_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r1v_launches.csv $B > gpurun_out/r1v_ncu1.log 2>&1; tail -1 gpurun_out/r1v_ncu1.log
