"""Shared-memory wavefronts (and the excess over ideal, i.e. bank conflicts) per source line of
the kernels in an ncu report.  python tools/ncu_smem.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
funcs, cur = [], None
for line in out:
    if line.startswith('"Function Name"'):
        cur = {"name": line.split('","')[1].rstrip('"'), "rows": []}
        funcs.append(cur)
    elif cur is not None:
        cur["rows"].append(line)
num = lambda v: int(float(v)) if v.strip().replace(".", "", 1).isdigit() else 0
for f in funcs:
    rows = list(csv.reader(f["rows"]))
    hdr = rows[0]
    iw, ie = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
    lines = [(r[0], r[1], num(r[iw]), num(r[ie])) for r in rows[1:] if len(r) > iw and r[0].isdigit()]
    tot = sum(l[2] for l in lines)
    if tot == 0:
        continue
    print(f"== {f['name'][:70]}  wavefronts {tot / 1e6:.0f}M, excessive {sum(l[3] for l in lines) / 1e6:.0f}M")
    for ln, src, wv, ex in sorted(lines, key=lambda l: -l[2])[:top]:
        print(f"{ln:>5} {wv / 1e6:7.1f}M  excess {ex / 1e6:6.1f}M  {src.strip()[:100]}")
