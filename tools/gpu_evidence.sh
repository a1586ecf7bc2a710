# Evidence refresh for profiles/ (bench line, reference arm, launch list, full tile capture);
# then: python tools/summarize_profiles.py gpurun_out/r1u_launches.csv gpurun_out/r1u_tiles.ncu-rep <tag>
set -x
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-seconds 10 > gpurun_out/r1u_bench.log 2>&1
cat gpurun_out/r1u_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1u_ref.log 2>&1
tail -1 gpurun_out/r1u_ref.log
$B > gpurun_out/r1u_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r1u_launches.csv $B > gpurun_out/r1u_ncu1.log 2>&1
timeout 300 python tools/profile_one.py C5 1 > gpurun_out/r1u_p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_tiles -c 2 -o gpurun_out/r1u_tiles python tools/profile_one.py C5 1 > gpurun_out/r1u_ncu2.log 2>&1
tail -3 gpurun_out/r1u_ncu2.log
