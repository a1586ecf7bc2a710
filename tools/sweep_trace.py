"""CTA 0's per-batch pipeline timeline of the sweep kernels (build: tools/build_variant.py trace
-DSE1P_SWEEP_TRACE=1; TRACE_LIB picks another variant).  python tools/sweep_trace.py [C5]
Fields per batch: 0 producer post, 1 expander sees records, 2 slot free, 3 full, 4 consumer warp 0
sees it, 8 after header/flush, 9 after its list, 10 after k-steps, 11 after carry/frame store,
5 arrive; 6 its k-steps, 7 batch size."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402

se1p.LIB_PATH = os.path.join(os.path.dirname(se1p.LIB_PATH), os.environ.get("TRACE_LIB", "libse1p_trace.so"))
se1p.load(build_if_needed=False)
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
x, q = make_system(cfg.N, cfg.L, cfg.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = kspace_kwargs(cfg)
for _ in range(3):
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, skip_checks=True, **kw)
torch.cuda.synchronize()
lib = ctypes.CDLL(se1p.LIB_PATH)
buf = np.zeros((2, 8192, 12), dtype=np.int64)
assert lib.se1p_sweep_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
print(os.environ.get("TRACE_LIB", "libse1p_trace.so"))
for gi, name in enumerate(["gridding", "gather"]):
    t = buf[gi].astype(np.float64)
    ok = (t[:, 5] > 0) & (t[:, 4] > 0) & (t[:, 0] > 0) & (t[:, 10] > 0)
    idx = np.nonzero(ok)[0]
    t = t[idx]
    n = len(idx)
    med = lambda a, b: np.median(t[:, b] - t[:, a])
    mean = lambda a, b: np.mean(t[:, b] - t[:, a])
    span = t[-1, 5] - t[0, 4]
    print(f"== {name}: {n} batches traced, consumer span {span:.0f} cyc = {span / n:.0f} cyc/batch")
    print(f"  pipeline (median): post->records {med(0, 1):.0f}, ->slot free {med(1, 2):.0f}, ->full {med(2, 3):.0f},"
          f" ->cons sees {med(3, 4):.0f}, ->done {med(4, 5):.0f}")
    print(f"  consumer warp 0 (mean): header/flush {mean(4, 8):.0f}, list {mean(8, 9):.0f}, k-steps {mean(9, 10):.0f},"
          f" carry/store {mean(10, 11):.0f}, arrive {mean(11, 5):.0f}, gap to next {np.mean(t[1:, 4] - t[:-1, 5]):.0f}")
    ks = t[:, 6]
    for kk in range(0, 7):
        sel = ks == kk
        if sel.sum() > 5:
            print(f"    k-steps={kk}: {sel.sum():5d} batches, k-step phase mean {np.mean(t[sel, 10] - t[sel, 9]):.0f}")
    print(f"  k-steps/batch {np.mean(ks):.2f}, candidates/batch {np.mean(t[:, 7]):.1f}")
