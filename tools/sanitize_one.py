"""Small run of every device entry for compute-sanitizer (one tool per gpurun call):
    compute-sanitizer --tool memcheck python tools/sanitize_one.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

for name in ("C1", "C2"):
    c = CONFIGS[name]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = kspace_kwargs(c)
    phi = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
    _, E = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, field=True, **kw)
    r, Er = se1p.real(xd, qd, c.L, c.xi, c.rc, field=True)
    p3 = se1p.kspace3p(xd, qd, c.L, c.xi, c.M, c.P if c.P % 2 == 0 else c.P + 1)
    torch.cuda.synchronize()
    print(name, float(phi.abs().max()), float(E.abs().max()), float(r.abs().max()), float(p3.abs().max()),
          flush=True)
print("sanitize run ok")
