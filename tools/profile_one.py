"""Run the k-space path of one config a few times (for ncu / compute-sanitizer captures)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
field = len(sys.argv) > 3 and sys.argv[3] == "field"
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
for _ in range(reps):
    phi = se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, skip_checks=True, field=field, **kspace_kwargs(cfg))
    phi = phi[0] if field else phi
torch.cuda.synchronize()
print("ok", float(phi.abs().max()))
