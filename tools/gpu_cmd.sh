timeout 900 python tools/se1p_vs_se3p.py > gpurun_out/se1p_vs_se3p.log 2>&1; tail -15 gpurun_out/se1p_vs_se3p.log
timeout 600 python tools/table2.py > gpurun_out/table2.log 2>&1; tail -3 gpurun_out/table2.log
