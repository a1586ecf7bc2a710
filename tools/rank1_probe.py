import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p
from paper_1611_09538_b200 import dist as sdist
from se1p_synth import CONFIGS, kspace_kwargs, make_system
cfg = CONFIGS["C5"]
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = kspace_kwargs(cfg)
info = se1p.plan_info(cfg.L, cfg.xi, cfg.M, cfg.P, **kw)
be = sdist.CudaBackend(cfg.L, cfg.xi, cfg.M, cfg.P, **kw)
plan = sdist.make_plan(info, 8)
r = 1
lo, hi = plan.bounds[r], plan.bounds[r + 1]
for _ in range(2):
    slab = be.forward(xd, qd, lo, hi, plan.order)
    split = torch.zeros(2 * plan.count(r) * plan.Mt * plan.Mt, dtype=torch.float64, device="cuda")
    be.modes(split, plan.owned[r], plan.bounds)
    be.backward(slab, cfg.N, lo, hi, plan.order)
torch.cuda.synchronize()
print("ok")
