"""Per-part device time of the real-space sum split over R emulated ranks (se1p.real part=(r, R)),
the load balance dist.real gets: python tools/real_parts_times.py [C5]"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, make_system  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
x, q = make_system(c.N, c.L, c.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
out = torch.empty(c.N, dtype=torch.float64, device="cuda")


def timed(part):
    se1p.real(xd, qd, c.L, c.xi, c.rc, out=out, part=part, skip_checks=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        se1p.real(xd, qd, c.L, c.xi, c.rc, out=out, part=part, skip_checks=True, sync=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3


t1 = timed(None)
print(f"{c.name} whole: {t1:.3f} ms", flush=True)
for R in (2, 4, 8):
    ts = [timed((r, R)) for r in range(R)]
    print(f"{c.name} R={R}: parts {' '.join(f'{t:.3f}' for t in ts)} ms; max {max(ts):.3f}; "
          f"efficiency t1/(R max) = {t1 / (R * max(ts)):.3f}", flush=True)
