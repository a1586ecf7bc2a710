"""Stage times of one config with a library variant (tools/build_variant.py).
    python tools/variant_times.py <name|product> C5 [field]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

name = sys.argv[1]
if name != "product":
    se1p.LIB_PATH = os.path.join(os.path.dirname(se1p.LIB_PATH), f"libse1p_{name}.so")
se1p.load(build_if_needed=False)
cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C5"]
field = len(sys.argv) > 3 and sys.argv[3] == "field"
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = kspace_kwargs(cfg)
acc = {}
for r in range(6):
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, skip_checks=True, profile=True, field=field, **kw)
    if r >= 2:
        for k, v in se1p.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v / 4
print(name, cfg.name, "field" if field else "", " ".join(f"{k}={v:.3f}" for k, v in acc.items()),
      f"total={sum(acc.values()):.3f} ms", flush=True)
