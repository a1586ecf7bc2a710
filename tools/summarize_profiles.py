"""Write the committed profile summaries (profiles/) from raw captures in gpurun_out/.

    python tools/summarize_profiles.py <launches.csv> <all_kernels.ncu-rep> <tag> [real.ncu-rep]

Writes profiles/<tag>_launches_C5_summary.txt (per-kernel share of the step from the ncu launch
list), profiles/<tag>_ncu_kernels_C5.txt (key metrics of every kernel of one C5 k-space call, and
of the real-space kernel, from --set full captures) and profiles/traffic.json (dram read+write
bytes per launch of the sweep kernels, read by bench.py for the roofline "traffic" field)."""
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict

import os

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
OUT = os.environ.get("PROFILES_DIR", "profiles")   # (on the GPU box: a directory under gpurun_out/)
os.makedirs(OUT, exist_ok=True)
real_rep = sys.argv[4] if len(sys.argv) > 4 else None

rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
# plan-time kernels (run once per plan, outside every timed step) and the one-off input check
PLAN = ("k_kern_a", "k_kern_b", "k_fft_rows_inplace", "k_transpose", "k_transpose_scale_real", "k_check")
base = lambda k: k.split()[-1].split("<")[0]
step_tot = sum(sum(v) for k, v in d.items() if base(k) not in PLAN)
with open(f"{OUT}/{tag}_launches_C5_summary.txt", "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py (C5)\n")
    f.write("cold-cache serialised launch times over every call of the run (plan, warm-up, timed, profiled, e2e);\n")
    f.write("'step share' leaves out the plan-time kernels (marked *) -- compare it with bench.py's stages_ms\n")
    f.write(f"{'total ms':>9} {'n':>4} {'avg ms':>8} {'share':>6} {'step share':>10}  kernel\n")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        plan = base(k) in PLAN
        ss = "" if plan else f"{100*sum(v)/step_tot:9.1f}%"
        f.write(f"{sum(v)/1e6:9.3f} {len(v):4d} {sum(v)/len(v)/1e6:8.3f} {100*sum(v)/tot:5.1f}% {ss:>10}  {k}{' *' if plan else ''}\n")

COLS = [("gpu__time_duration.sum", "us"),
        ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefr"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem confl"),
        ("launch__registers_per_thread", "regs"), ("launch__block_size", "block"), ("launch__grid_size", "grid")]


def tobytes(v, u):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def table(rep_path, f, title):
    raw = subprocess.run(["ncu", "-i", rep_path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    f.write(f"\n## {title}\n")
    f.write(f"{'kernel':44s} " + " ".join(f"{lab:>11s}" for _, lab in COLS) + "\n")
    out = []
    for row in r[2:]:
        name = re.sub(r"\(.*$", "", row[h.index("Kernel Name")])[:44]
        vals = []
        for c, lab in COLS:
            if c not in h:
                vals.append("-")
                continue
            v, u = row[h.index(c)], units[h.index(c)]
            if c == "gpu__time_duration.sum":
                x = tobytes(v, "") / (1e3 if u == "ns" else (1 if u == "us" else 1e-3))
                vals.append(f"{x:.1f}")
            elif c.startswith("dram__bytes"):
                vals.append(f"{tobytes(v, u) / 1e6:.1f}MB")
            else:
                vals.append(v)
        f.write(f"{name:44s} " + " ".join(f"{x:>11s}" for x in vals) + "\n")
        out.append((row[h.index("Kernel Name")], {c: (row[h.index(c)], units[h.index(c)]) for c, _ in COLS if c in h}))
    return out


with open(f"{OUT}/{tag}_ncu_kernels_C5.txt", "w") as f:
    f.write("ncu --set full --clock-control none: every kernel of one C5 k-space call (tools/profile_one.py C5 1), "
            "cold and serialised (the mode stage's concurrent streams run one after the other here);\n"
            "DMMA% = FP64 tensor pipe (DMMA) active, FP64% = non-tensor FP64 pipe, issue% = issue slots busy, "
            "occ% = achieved warp occupancy, smem% = shared-memory wavefronts of peak\n")
    kern = table(rep, f, "k-space step kernels (C5)")
    if real_rep:
        table(real_rep, f, "real space (C5, rc = 0.1)")

traffic = {}
for name, vals in kern:
    m = re.search(r"k_sweep<([^>]*)>", name)
    if not m:
        continue
    args = [t.strip() for t in m.group(1).split(",")]
    gather = args[0] in ("1", "true", "(bool)1")
    fm = args[1] if len(args) > 1 else "0"
    key = ("gather" if fm in ("0", "(int)0") else f"gather_field{fm[-1]}") if gather else "spread"
    traffic[key] = tobytes(*vals["dram__bytes_read.sum"]) + tobytes(*vals["dram__bytes_write.sum"])
json.dump({**traffic, "source": rep, "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, C5"},
          open(f"{OUT}/traffic.json", "w"), indent=1)
print(open(f"{OUT}/{tag}_launches_C5_summary.txt").read()[:1800])
print(open(f"{OUT}/{tag}_ncu_kernels_C5.txt").read())
print(json.dumps(traffic))
