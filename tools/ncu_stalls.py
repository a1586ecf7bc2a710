"""Stall-reason sums per source-line range of the first kernel in an ncu report (needs -lineinfo).
    python tools/ncu_stalls.py report.ncu-rep name:lo-hi [name:lo-hi ...] [--kernel substring] [--lines lo-hi]"""
import csv
import subprocess
import sys

rep, specs = sys.argv[1], [a for a in sys.argv[2:] if ":" in a]
ksel = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Function Name"'):
        cur = {"name": line.split('","')[1].rstrip('"'), "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(line)
big = sorted(blocks, key=lambda b: -len(b["rows"]))
f = max([b for b in blocks if ksel in b["name"]], key=lambda b: len(b["rows"]))   # the kernel's own file
rows = list(csv.reader(f["rows"]))
hdr = rows[0]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
i_ex = hdr.index("Instructions Executed")
num = lambda v: int(v) if v.strip().lstrip("-").isdigit() else 0
print(f["name"])
for sp in specs:
    name, rng = sp.split(":")
    lo, hi = map(int, rng.split("-"))
    agg = {hdr[i]: 0 for i in cols}
    ins = 0
    for r in rows[1:]:
        if len(r) > i_ex and r[0].isdigit() and lo <= int(r[0]) <= hi:
            for i in cols:
                agg[hdr[i]] += num(r[i])
            ins += num(r[i_ex])
    tot = sum(agg.values())
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:7]
    print(f"{name:10s} samples {tot:7d} instr {ins / 1e6:7.0f}M  " + " ".join(f"{k[6:]}={100 * v / max(tot, 1):.0f}%" for k, v in top))

if "--lines" in sys.argv:
    lo, hi = map(int, sys.argv[sys.argv.index("--lines") + 1].split("-"))
    res = []
    for r in rows[1:]:
        if len(r) > i_ex and r[0].isdigit() and lo <= int(r[0]) <= hi:
            agg = {hdr[i][6:]: num(r[i]) for i in cols}
            tot = sum(agg.values())
            if tot:
                res.append((tot, r[0], r[1].strip()[:70], sorted(agg.items(), key=lambda kv: -kv[1])[:3], num(r[i_ex])))
    for tot, ln, src, top, ins in sorted(res, reverse=True)[:30]:
        print(f"{ln:>5} {tot:7d} {ins / 1e6:6.0f}M {' '.join(f'{k}={v}' for k, v in top):45s} {src}")
