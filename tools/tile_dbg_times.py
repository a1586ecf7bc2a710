"""Stage times of the C5 k-space call under SE1P_TILE_DBG experiment bits (timing only)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_09538_b200 as se1p
from se1p_synth import CONFIGS, kspace_kwargs, make_system
c = CONFIGS["C5"]
x, q = make_system(c.N, c.L, c.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = kspace_kwargs(c)
for _ in range(3):
    se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, profile=True, **kw)
g = []
for _ in range(5):
    se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, profile=True, **kw)
    g.append(se1p.stage_times())
print(os.environ.get("SE1P_TILE_DBG", "0"), "spread %.3f gather %.3f" % (np.median([t["spread"] for t in g]), np.median([t["gather"] for t in g])))
