# Evidence refresh for profiles/ (bench line, reference arm, launch list, --set full capture of
# every kernel of one C5 k-space call and of the real-space kernel), summarised on the box into
# gpurun_out/${T}_profiles/ (copy into profiles/ afterwards); the big reports stay in /tmp except
# the two sweep kernels' capture (line-level analysis here).
T=${1:-r02}
set -x
mkdir -p /tmp/ev gpurun_out/${T}_profiles
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-seconds 10 > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_ref.log 2>&1
tail -1 gpurun_out/${T}_ref.log
$B > /tmp/ev/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file /tmp/ev/launches.csv $B > /tmp/ev/ncu1.log 2>&1
timeout 300 python tools/profile_one.py C5 1 > /tmp/ev/p1.log 2>&1 &&
ncu --set full --clock-control none -k regex:"k_keys|k_bin_count|k_scan|k_rs_|k_permute|k_records|k_items|k_sweep|k_overhang|k_zfwd|k_zinv|k_persist|k_colpass|k_gather_finish" -c 60 -f -o /tmp/ev/all python tools/profile_one.py C5 1 > /tmp/ev/ncu2.log 2>&1
tail -2 /tmp/ev/ncu2.log
ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 2 -f -o gpurun_out/${T}_sweeps python tools/profile_one.py C5 1 > /tmp/ev/ncu4.log 2>&1
tail -1 /tmp/ev/ncu4.log
cat > /tmp/real1.py <<'PY'
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p
from se1p_synth import CONFIGS, make_system
c = CONFIGS["C5"]
x, q = make_system(c.N, c.L, c.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
se1p.real(xd, qd, c.L, c.xi, c.rc)
torch.cuda.synchronize()
print("ok")
PY
python /tmp/real1.py > /dev/null 2>&1 &&
ncu --set full --clock-control none -k regex:"k_real_warp|k_real_sum" -c 1 -f -o /tmp/ev/real python /tmp/real1.py > /tmp/ev/ncu3.log 2>&1
tail -1 /tmp/ev/ncu3.log
PROFILES_DIR=gpurun_out/${T}_profiles python tools/summarize_profiles.py /tmp/ev/launches.csv /tmp/ev/all.ncu-rep ${T} /tmp/ev/real.ncu-rep > gpurun_out/${T}_summary.log 2>&1
cp /tmp/ev/launches.csv gpurun_out/${T}_profiles/${T}_launches_C5.csv
du -sh gpurun_out
