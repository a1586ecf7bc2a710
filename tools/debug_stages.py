"""Stage-by-stage comparison of the CUDA path with the numpy Alg. 1 oracle (debug tool)."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p
from oracle import se1p_discrete as sd
from se1p_synth import make_system

N, L, xi, M, P, n_l, S0, SI, SJ = 100, (1.0, 1.0, 1.0), 4.0, 16, 16, 2, 110, 64, 32
if len(sys.argv) > 1:
    N, M, P, n_l, S0, SI, SJ = [int(v) for v in sys.argv[1:8]]
x, q = make_system(N, L, 1)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
kw = dict(n_local=n_l, S0=S0, SI=SI, Ntilde=SJ)
d = sd.derived(L, xi, M, P)
pref = (2 * xi ** 2 / (math.pi * d["eta"])) ** 1.5
H = sd.gridding(x, q, xi, d["h"], P, M, d["Mt1"], d["Mt2"], d["eta"]) / pref
g1 = se1p.debug_stage(xd, qd, L, xi, M, P, 1, **kw)
print("spread  max|d| %.3e  max|H| %.3e" % (np.abs(g1 - H).max(), np.abs(H).max()))
Hz = np.fft.fft(H, axis=2)[:, :, : M // 2 + 1].transpose(2, 0, 1)
g2 = se1p.debug_stage(xd, qd, L, xi, M, P, 2, **kw)
print("zfft    max|d| %.3e  max %.3e" % (np.abs(g2 - Hz).max(), np.abs(Hz).max()))
# mode stage reference: per plane as the oracle does, with constants folded like the GPU
phi, allv = sd.se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ, return_all=True)
Ht = allv["Htilde"]
C = 4 * math.pi * d["h"] ** 3 * pref * pref
Hk_ref = np.fft.fft(Ht, axis=2)[:, :, : M // 2 + 1].transpose(2, 0, 1) * C / (M * pref)
g3 = se1p.debug_stage(xd, qd, L, xi, M, P, 3, **kw)
for n in range(M // 2 + 1):
    print("modes plane %2d max|d| %.3e max %.3e ratio %.6f" % (n, np.abs(g3[n] - Hk_ref[n]).max(), np.abs(Hk_ref[n]).max(),
          (np.vdot(Hk_ref[n], g3[n]) / np.vdot(Hk_ref[n], Hk_ref[n])).real))
g4 = se1p.debug_stage(xd, qd, L, xi, M, P, 4, **kw)
ref4 = Ht / pref * C
print("izfft   max|d| %.3e  max %.3e" % (np.abs(g4 - ref4).max(), np.abs(ref4).max()))
got = se1p.kspace(xd, qd, L, xi, M, P, **kw).cpu().numpy()
print("phi     max|d| %.3e  max %.3e" % (np.abs(got - phi).max(), np.abs(phi).max()))
