"""Graph-mode stress: replay the C5 (or given config) k-space graph many times and check every
result bitwise against the first (intermittent-fault hunt).   python tools/stress_graph.py C5 500"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
out = torch.empty(cfg.N, dtype=torch.float64, device="cuda")
kw = kspace_kwargs(cfg)
ref = se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, **kw).clone()
bad = 0
for r in range(reps):
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, out=out, graph=True, skip_checks=True, **kw)
    if r % 50 == 49 or r == reps - 1:
        torch.cuda.synchronize()
        if not torch.equal(out, ref):
            bad += 1
            print(f"rep {r}: differs by {float((out - ref).abs().max()):.3e}")
print(f"{reps} graph replays, {bad} mismatching checks")
