"""Write the committed profile summaries (profiles/) from raw captures in gpurun_out/.

    python tools/summarize_profiles.py <launches.csv> <tiles.ncu-rep> <tag>

Writes profiles/<tag>_launches_C5_summary.txt (per-kernel share of the step from the
ncu launch list), profiles/<tag>_ncu_tiles_C5.txt (key metrics of the two tile kernels from a
--set full capture) and profiles/traffic.json (dram read+write bytes per launch of the tile
kernels, read by bench.py for the roofline "traffic" field)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]

rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
# plan-time kernels (run once per plan, outside every timed step) and the one-off input check
PLAN = ("k_kern_a", "k_kern_b", "k_fft_rows_inplace", "k_transpose", "k_transpose_scale_real", "k_check")
step_tot = sum(sum(v) for k, v in d.items() if k.split()[-1].split("<")[0] not in PLAN)
with open(f"profiles/{tag}_launches_C5_summary.txt", "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py (C5)\n")
    f.write("cold-cache serialised launch times over every call of the run (plan, warm-up, timed, profiled, e2e);\n")
    f.write("'step share' leaves out the plan-time kernels (marked *) -- compare it with bench.py's stages_ms\n")
    f.write(f"{'total ms':>9} {'n':>4} {'avg ms':>8} {'share':>6} {'step share':>10}  kernel\n")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        plan = k.split()[-1].split("<")[0] in PLAN
        ss = "" if plan else f"{100*sum(v)/step_tot:9.1f}%"
        f.write(f"{sum(v)/1e6:9.3f} {len(v):4d} {sum(v)/len(v)/1e6:8.3f} {100*sum(v)/tot:5.1f}% {ss:>10}  {k}{' *' if plan else ''}\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
traffic = {}
with open(f"profiles/{tag}_ncu_tiles_C5.txt", "w") as f:
    f.write(f"ncu --set full --clock-control none --import-source on -k regex:k_tiles -c 2 python tools/profile_one.py C5 1\n")
    for row in r[2:]:
        name = row[h.index("Kernel Name")]
        f.write(f"---- {name}\n")
        vals = {}
        for i, n in enumerate(h):
            if n in want:
                f.write(f"  {n} = {row[i]} {units[i]}\n")
                vals[n] = (row[i], units[i])

        def tobytes(v):
            x, u = float(v[0].replace(",", "")), v[1]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        import re
        targs = re.search(r"k_tiles<([^>]*)>", name)
        args = [t.strip() for t in targs.group(1).split(",")] if targs else []
        gather = len(args) > 1 and args[1] in ("1", "true", "(bool)1")
        field = len(args) > 2 and args[2] in ("1", "true", "(bool)1")
        key = ("gather_field" if field else "gather") if gather else "spread"
        traffic[key] = tobytes(vals["dram__bytes_read.sum"]) + tobytes(vals["dram__bytes_write.sum"])
json.dump({**traffic, "source": rep, "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, C5"},
          open("profiles/traffic.json", "w"), indent=1)
print(open(f"profiles/{tag}_launches_C5_summary.txt").read()[:1500])
print(json.dumps(traffic))
