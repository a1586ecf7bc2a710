python tools/profile_one.py C5 1 > gpurun_out/r1n_p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_tiles -c 2 -o gpurun_out/r1n_tiles python tools/profile_one.py C5 1 > gpurun_out/r1n_ncu.log 2>&1
