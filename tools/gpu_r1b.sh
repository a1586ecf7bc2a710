# launch list of the bench command, phase counters, one full ncu capture of the tile kernels
set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/r1b_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_launches.csv $B > gpurun_out/r1b_ncu1.log 2>&1
python tools/phase_counters.py C5 > gpurun_out/r1b_phase_c5.log 2>&1
python tools/phase_counters.py C4 > gpurun_out/r1b_phase_c4.log 2>&1
python tools/profile_one.py C5 1 > gpurun_out/r1b_p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_tile_mma -c 2 -o gpurun_out/r1b_tiles python tools/profile_one.py C5 1 > gpurun_out/r1b_ncu2.log 2>&1
ls -la gpurun_out
