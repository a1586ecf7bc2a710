"""SASS of one kernel in an ncu report with samples and the top stall reasons per instruction,
around the hottest instructions.  python tools/ncu_sass.py report.ncu-rep <kernel-substring> [lo hi]"""
import csv
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = {"name": line, "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(line)
b = [x for x in blocks if ksub in x["name"]][0]
rows = list(csv.reader(b["rows"]))
hdr = rows[0]
data = [r for r in rows[1:] if len(r) == len(hdr)]
i_s, i_src, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
num = lambda v: int(v) if v.strip().isdigit() else 0
if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3]), int(sys.argv[4])
else:
    top = max(range(len(data)), key=lambda i: num(data[i][i_s]))
    lo, hi = top - 40, top + 40
for i in range(max(lo, 0), min(hi, len(data))):
    r = data[i]
    st = sorted(((num(r[j]), hdr[j][6:]) for j in stalls), reverse=True)[:2]
    sts = " ".join(f"{n}:{v}" for v, n in st if v)
    print(f"{i:5d} {num(r[i_s]):6d} {num(r[i_ex]):10d}  {r[i_src].strip()[:60]:60s} {sts}")
