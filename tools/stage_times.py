"""Per-stage device times of the k-space path for one config (CUDA events inside the library).
    python tools/stage_times.py C5 [field]   (field: the field (force) variant of the gather)"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
field = len(sys.argv) > 2 and sys.argv[2] == "field"
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = kspace_kwargs(cfg)
acc = {}
for r in range(6):
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, skip_checks=True, profile=True, field=field, **kw)
    if r >= 2:
        for k, v in se1p.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v / 4
print(cfg.name, "field" if field else "sweep", " ".join(f"{k}={v:.3f}" for k, v in acc.items()), f"total={sum(acc.values()):.3f} ms", flush=True)
