"""Real-space device time with a library variant (tools/build_variant.py).
    python tools/real_variant.py NAME [C4,C5] [field]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, make_system  # noqa: E402

if sys.argv[1] != "product":
    se1p.LIB_PATH = os.path.join(os.path.dirname(se1p.LIB_PATH), f"libse1p_{sys.argv[1]}.so")
for name in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["C4", "C5"]):
    c = CONFIGS[name]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    field = len(sys.argv) > 3 and sys.argv[3] == "field"
    se1p.real(xd, qd, c.L, c.xi, c.rc, field=field)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        se1p.real(xd, qd, c.L, c.xi, c.rc, skip_checks=True, sync=False, field=field)
    e1.record()
    torch.cuda.synchronize()
    print(sys.argv[1], name, "field" if field else "", f"{e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
