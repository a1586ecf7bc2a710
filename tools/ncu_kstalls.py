"""Top source lines (all files) of one kernel in an ncu report, with stall reasons.
    python tools/ncu_kstalls.py report.ncu-rep <kernel-name substring> [top]"""
import csv
import subprocess
import sys

rep, ksel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Function Name"'):
        cur = {"name": line.split('","')[1].rstrip('"'), "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(line)
num = lambda v: int(v) if v.strip().lstrip("-").isdigit() else 0
res, tot_all, seen = [], {}, set()
for b in blocks:
    if ksel not in b["name"]:
        continue
    rows = list(csv.reader(b["rows"]))
    if not rows or "Line No" not in rows[0][0]:
        continue
    hdr = rows[0]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    i_ex = hdr.index("Instructions Executed")
    fname = b["rows"][0] if False else ""
    for r in rows[1:]:
        if len(r) > i_ex and r[0].isdigit():
            agg = {hdr[i][6:]: num(r[i]) for i in cols}
            t = sum(agg.values())
            key = (r[1].strip()[:80], r[0])
            if t and key not in seen:
                seen.add(key)
                res.append((t, r[0], r[1].strip()[:80], sorted(agg.items(), key=lambda kv: -kv[1])[:3], num(r[i_ex])))
                for k, v in agg.items():
                    tot_all[k] = tot_all.get(k, 0) + v
T = sum(tot_all.values())
print(ksel, "samples", T, " ".join(f"{k}={100 * v / T:.0f}%" for k, v in sorted(tot_all.items(), key=lambda kv: -kv[1])[:8]))
for t, ln, src, tp, ins in sorted(res, reverse=True)[:top]:
    print(f"{ln:>5} {100 * t / T:5.1f}% {ins / 1e6:6.1f}M {' '.join(f'{k}={v}' for k, v in tp):42s} {src}")
