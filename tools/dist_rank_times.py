"""Per-rank device time of the mode-sharded path, emulated on one GPU (each rank's three stages
timed in turn; the transposes are not included):  python tools/dist_rank_times.py [C5]"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from paper_1611_09538_b200 import dist as sdist  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = kspace_kwargs(cfg)
info = se1p.plan_info(cfg.L, cfg.xi, cfg.M, cfg.P, **kw)
be = sdist.CudaBackend(cfg.L, cfg.xi, cfg.M, cfg.P, **kw)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


single = min(timed(lambda: se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, skip_checks=True, **kw))[1] for _ in range(3))
print(f"{cfg.name} single GPU {single:.3f} ms")
for R in (2, 4, 8):
    plan = sdist.make_plan(info, R)
    worst = 0.0
    for r in range(R):
        lo, hi = plan.bounds[r], plan.bounds[r + 1]
        for _ in range(2):   # second pass timed (plans and workspace warm)
            slab, tf = timed(lambda: be.forward(xd, qd, lo, hi, plan.order))
            split = torch.zeros(2 * plan.count(r) * plan.Mt * plan.Mt, dtype=torch.float64, device="cuda")
            _, tm = timed(lambda: be.modes(split, plan.owned[r], plan.bounds))
            _, tb = timed(lambda: be.backward(slab, cfg.N, lo, hi, plan.order))
        worst = max(worst, tf + tm + tb)
        print(f"  R={R} rank {r}: rows [{lo},{hi}) forward {tf:.3f} modes {tm:.3f} backward {tb:.3f} ms", flush=True)
    print(f"R={R}: slowest rank {worst:.3f} ms (compute only) -> speedup {single / worst:.2f}, "
          f"efficiency {single / worst / R:.2f}", flush=True)
