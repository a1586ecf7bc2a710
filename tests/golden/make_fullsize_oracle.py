"""Writes tests/golden/fullsize_<C>.npz: the exact Ewald1P potential (oracle/, Eqs. (2)-(6),
P:80-92) of BASELINE.json's C4 and C5 systems on the oracle evaluation sets of SURVEY.md 8(c)
step 7 -- C4: 2048 seeded targets + 256 within 2w of a free face, C5: 512 + 256 -- each against
all N sources.  For C5 also the converged real-space term and the real-space term truncated at
the config's rc = 0.1 (reading R-13).  Calls only oracle/ and the seeded input generator.

    python tests/golden/make_fullsize_oracle.py [C4 C5]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from se1p_synth import CONFIGS, edge_targets, make_system, sample_targets  # noqa: E402

SETS = {"C4": (2048, 256), "C5": (512, 256)}


def targets(cfg, x):
    m, me = SETS[cfg.name]
    h = cfg.L[2] / cfg.M
    t = sample_targets(cfg.N, m, cfg.seed + 31)
    e = edge_targets(x, cfg.L, cfg.P * h, me, cfg.seed + 31)
    return np.unique(np.concatenate([t, e]))


def main(names):
    for name in names:
        cfg = CONFIGS[name]
        x, q = make_system(cfg.N, cfg.L, cfg.seed)
        tg = targets(cfg, x)
        t0 = time.time()
        exact = oracle.phi_exact(x, q, cfg.L, tg)
        out = dict(targets=tg, exact=exact)
        if name == "C5":
            out["real_conv"] = oracle.phi_real(x, q, cfg.L, cfg.xi, None, tg)
            out["real_trunc"] = oracle.phi_real(x, q, cfg.L, cfg.xi, cfg.rc, tg)
        np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), f"fullsize_{name}.npz"), **out)
        print(name, tg.size, "targets", f"{time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C4", "C5"])
