"""Real-space sum of one config a few times (for ncu captures).  python tools/real_one.py C5 [rc]"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, make_system  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
rc = float(sys.argv[2]) if len(sys.argv) > 2 else c.rc
x, q = make_system(c.N, c.L, c.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
for _ in range(2):
    se1p.real(xd, qd, c.L, c.xi, rc, skip_checks=True)
torch.cuda.synchronize()
print("ok")
