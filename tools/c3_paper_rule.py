"""C3 at the paper's literal upsampling rule against the exact oracle: s_l with
e^{-2 pi s_l} < E = 1e-10, n_l ~ M/10, s0 ~ 2.4, J modes at the paper's
extent M~ = M_free + P.  Prints the relative rms of phi^F + phi^R + phi^self on C3's oracle set.
    python tools/c3_paper_rule.py"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, edge_targets, make_system, sample_targets  # noqa: E402

c = CONFIGS["C3"]
x, q = make_system(c.N, c.L, c.seed)
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
h = c.L[2] / c.M
Mt = int(round(c.L[0] / h)) + c.P
s_l = math.log(1e10) / (2 * math.pi)
rows = []
for name, kw in [("paper rule (n_l=M/10, s_l=3.66, s0=2.4, Ntilde=M~)",
                  dict(n_local=round(c.M / 10), sf=s_l, s0=2.4, Ntilde=Mt)),
                 ("paper rule, n_l=M/10, Ntilde=M~, S0=SI=8M~", dict(n_local=round(c.M / 10), S0=8 * Mt, SI=8 * Mt,
                                                                   Ntilde=Mt)),
                 ("build default (se1p_synth C3)", dict(n_local=c.n_local, S0=c.S0, SI=c.SI, Ntilde=c.Ntilde))]:
    phik = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw).cpu().numpy()
    phir = se1p.real(xd, qd, c.L, c.xi, c.rc).cpu().numpy()
    tg = np.unique(np.concatenate([sample_targets(c.N, c.oracle_targets, c.seed),
                                   edge_targets(x, c.L, c.P * h, c.oracle_edge, c.seed)]))
    ref = oracle.phi_exact(x, q, c.L, tg)
    err = oracle.rel_rms(phik[tg] + phir[tg], ref)
    info = se1p.plan_info(c.L, c.xi, c.M, c.P, **kw)
    print(f"{name}: S0={info['S0']} SI={info['SI']} n_l={info['n_local']} Ntilde={info['Ntilde']}  rel rms {err:.3e}",
          flush=True)
