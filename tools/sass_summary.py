"""Static SASS opcode counts per kernel of the product library (cuobjdump -sass), for the opcodes
that show which hardware paths each kernel uses: DMMA (FP64 tensor-core MMA), UBLKCP (bulk async
copy, cp.async.bulk), SYNCS (mbarrier), LDGSTS (cp.async), SHFL, BAR, DFMA/DMUL/DADD, LDS/STS,
LDG/STG.  python tools/sass_summary.py [lib] > profiles/rNN_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1611_09538_b200", "_lib", "libse1p.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
dem = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
KEYS = ["DMMA", "UBLKCP", "SYNCS", "LDGSTS", "SHFL", "BAR", "DFMA", "DMUL", "DADD", "LDS", "STS", "LDG", "STG",
        "ATOMS", "ATOMG", "RED", "MUFU"]
funcs, cur = collections.OrderedDict(), None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        op = m.group(1)
        funcs[cur]["total"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "") and k in ("SYNCS", "UBLKCP"):
                funcs[cur][k] += 1
print(f"# static SASS instruction counts per kernel, {os.path.basename(lib)} (sm_100a), cuobjdump -sass")
print(f"{'kernel':70s} {'total':>6s} " + " ".join(f"{k:>6s}" for k in KEYS))
for f, c in funcs.items():
    name = dem(f)
    name = re.sub(r"\(.*\)$", "", name)[:70]
    print(f"{name:70s} {c['total']:6d} " + " ".join(f"{c[k]:6d}" for k in KEYS))
