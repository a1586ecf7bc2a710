"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the SE1P method: it only draws particle systems and
records the workload configurations named in BASELINE.json.  Both sides (the CPU oracle
under ``oracle/`` and the CUDA path under ``paper_1611_09538_b200/``) receive the same
arrays from here and nothing else is shared between them.

Recipe: positions uniform in the box [0,L1)x[0,L2)x[0,L3)
(the paper's "randomly/uniformly distributed particles"),
charges uniform in [-1,1] shifted to zero sum (BASELINE.json config 1; charge neutrality
is required by Eq. (1)).  The third axis is the periodic one.
"""
from __future__ import annotations

import dataclasses

import numpy as np


def make_system(N: int, L, seed: int):
    """Return (x [N,3] float64, q [N] float64) for a neutral uniform random system."""
    L = np.asarray(L, dtype=np.float64)
    rng = np.random.default_rng(seed)
    x = rng.random((N, 3)) * L
    # guard against x == L after the multiply (cannot happen for L=1,2 but keep the box half-open)
    x = np.where(x >= L, np.nextafter(L, 0.0), x)
    q = rng.uniform(-1.0, 1.0, N)
    q -= q.mean()
    return np.ascontiguousarray(x), np.ascontiguousarray(q)


def sample_targets(N: int, m: int, seed: int):
    """Seeded subset of target indices (sorted, unique) for oracle checks at large N."""
    if m >= N:
        return np.arange(N, dtype=np.int64)
    rng = np.random.default_rng(seed + 7919)
    return np.sort(rng.choice(N, size=m, replace=False)).astype(np.int64)


def edge_targets(x: np.ndarray, L, width: float, m: int, seed: int):
    """Targets within `width` of a free (x or y) face: where aliasing error concentrates."""
    L = np.asarray(L, dtype=np.float64)
    d = np.minimum.reduce([x[:, 0], L[0] - x[:, 0], x[:, 1], L[1] - x[:, 1]])
    idx = np.nonzero(d < width)[0]
    if idx.size > m:
        rng = np.random.default_rng(seed + 104729)
        idx = np.sort(rng.choice(idx, size=m, replace=False))
    return idx.astype(np.int64)


@dataclasses.dataclass(frozen=True)
class Config:
    """A BASELINE.json workload.  Method parameters are data here (no arithmetic)."""

    name: str
    N: int
    L: tuple
    xi: float
    M: int            # grid points on the periodic axis (h = L3/M)
    P: int            # Gaussian support points per dimension
    n_local: int      # n_l: number of upsampled |k3| modes (Eq. (I))
    Ntilde: int       # FFT extent of the free axes for the J modes (>= M_free + P)
    S0: int           # padded extent of the k3 = 0 plane (0 -> from s0)
    SI: int           # padded extent of the I planes (0 -> from sf)
    s0: float         # paper's factors when the config fixes them (BASELINE config 1)
    sf: float
    rc: float         # real-space cutoff
    seed: int
    oracle_targets: int   # seeded target subset for the exact oracle (all N if >= N)
    oracle_edge: int      # extra targets near a free face


# Parameters: BASELINE.json configs + the readings in DESIGN.md ("Parameter choices").
# C1 keeps the config's own s0 = 2+sqrt(2), s_l = 2 on |k3| <= 2 and the paper's M~ extent.
CONFIGS = {
    "C1": Config("C1", 100, (1.0, 1.0, 1.0), 4.0, 16, 16, 2, 32, 0, 0, 2.0 + 2.0 ** 0.5, 2.0, 1.158, 1, 100, 0),
    "C2": Config("C2", 2000, (1.0, 1.0, 1.0), 8.0, 32, 20, 3, 64, 416, 416, 0.0, 0.0, 0.594, 2, 2000, 0),
    "C3": Config("C3", 20000, (1.0, 1.0, 2.0), 12.0, 96, 24, 7, 96, 576, 576, 0.0, 0.0, 0.401, 3, 1024, 128),
    "C4": Config("C4", 200000, (1.0, 1.0, 1.0), 20.0, 128, 24, 4, 224, 1216, 1216, 0.0, 0.0, 0.247, 4, 512, 128),
    "C5": Config("C5", 2000000, (2.0, 2.0, 2.0), 30.0, 256, 24, 16, 320, 2240, 2240, 0.0, 0.0, 0.1, 5, 256, 64),
}


def kspace_kwargs(c: Config) -> dict:
    """Keyword arguments of paper_1611_09538_b200.kspace for a config (data only)."""
    kw = dict(n_local=c.n_local, Ntilde=c.Ntilde)
    if c.S0:
        kw.update(S0=c.S0, SI=c.SI)
    else:
        kw.update(s0=c.s0, sf=c.sf)
    return kw
