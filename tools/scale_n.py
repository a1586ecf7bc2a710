"""k-space at C5 parameters with N = 2e6 .. 3.2e7 (denser systems; the grid is unchanged): device
time per call and throughput, plus sampled parity against the exact oracle at the largest N.
    python tools/scale_n.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

c = CONFIGS["C5"]
kw = kspace_kwargs(c)
for N in (2_000_000, 8_000_000, 32_000_000):
    x, q = make_system(N, c.L, 77)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, out=out, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, out=out, skip_checks=True, sync=False, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"N={N:9d}: {ms:8.3f} ms  {N / ms * 1e3:.3e} particles/s  (free {torch.cuda.mem_get_info()[0] / 1e9:.0f} GB)",
          flush=True)
    if N == 32_000_000:
        import oracle
        t = np.arange(0, N, N // 8)
        phir = se1p.real(xd, qd, c.L, c.xi, c.rc).cpu().numpy()
        ref = oracle.phi_exact(x, q, c.L, t)
        conv = oracle.phi_real(x, q, c.L, c.xi, None, t)
        trunc = oracle.phi_real(x, q, c.L, c.xi, c.rc, t)
        got = out.cpu().numpy()[t] + phir[t]
        print("rel rms vs exact (same truncated real space, R-13):", oracle.rel_rms(got, ref - conv + trunc), flush=True)
