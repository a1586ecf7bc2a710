"""Per-source-line warp-stall samples of the kernels in an ncu report (needs -lineinfo and
--import-source).  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
funcs, cur = [], None
for line in out:
    if line.startswith('"Function Name"'):
        cur = {"name": line.split('","')[1].rstrip('"'), "rows": []}
        funcs.append(cur)
    elif cur is not None:
        cur["rows"].append(line)
for f in funcs:
    rows = list(csv.reader(f["rows"]))
    hdr = rows[0]
    i_line, i_src, i_s, i_ex = 0, 1, hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    num = lambda v: int(v) if v.strip().lstrip("-").isdigit() else 0
    lines = [(r[i_line], r[i_src], num(r[i_s]), num(r[i_ex])) for r in rows[1:]
             if len(r) > i_ex and r[i_line] not in ("", "Line No")]
    tot = sum(l[2] for l in lines)
    print(f"== {f['name']}  samples {tot}")
    for ln, src, s, ex in sorted(lines, key=lambda l: -l[2])[:top]:
        print(f"{ln:>5} {100.0 * s / max(tot, 1):5.1f}% {ex:11d}  {src.strip()[:110]}")

# optional: per-role sums over line ranges, e.g. ROLES="producer:200-300,expanders:300-425,consumers:425-700"
import os
if os.environ.get("ROLES"):
    for f in funcs:
        rows = list(csv.reader(f["rows"]))
        hdr = rows[0]
        i_s, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        num = lambda v: int(v) if v.strip().lstrip("-").isdigit() else 0
        agg = {}
        for r in rows[1:]:
            if len(r) <= i_ex or not r[0].isdigit():
                continue
            ln = int(r[0])
            for spec in os.environ["ROLES"].split(","):
                name, rng = spec.split(":")
                lo, hi = map(int, rng.split("-"))
                if lo <= ln < hi:
                    a = agg.setdefault(name, [0, 0])
                    a[0] += num(r[i_s])
                    a[1] += num(r[i_ex])
        if agg:
            print(f["name"][:60], {k: (v[0], f"{v[1]/1e6:.0f}M instr") for k, v in agg.items()})
