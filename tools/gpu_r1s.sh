python tools/profile_one.py C5 1 > gpurun_out/r1s_p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_colpass|k_rowfwd|k_zfwd" -c 4 -o gpurun_out/r1s_fft python tools/profile_one.py C5 1 > gpurun_out/r1s_ncu.log 2>&1
