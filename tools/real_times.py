"""Device time of the real-space sum (and its field) at the configs' cutoffs.  python tools/real_times.py"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, make_system  # noqa: E402

for name in ["C3", "C4", "C5"]:
    c = CONFIGS[name]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    for field in (False, True):
        se1p.real(xd, qd, c.L, c.xi, c.rc, field=field)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            se1p.real(xd, qd, c.L, c.xi, c.rc, field=field, skip_checks=True, sync=False)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} rc={c.rc} field={field}: {e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
