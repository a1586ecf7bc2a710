"""SE3P k-space (the triply periodic Spectral Ewald baseline of SURVEY 8(f) NEXT-4), step by step
in plain numpy.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's Ex. 5 compares SE1P with SE3P [Lindbo2011]; SE3P is Alg. 1 with every
direction periodic, so each step is the SE1P step with the free-axis machinery removed:

  step 1  h = L3/M, M_d = L_d/h, eta = P xi^2 h^2/(c^2 pi), c = 0.95   (as Alg. 1 step 1)
  step 2  gridding H on the periodic M1 x M2 x M grid: the Gaussians of Eq. (spread_1p)
          with the periodic-axis stencil of reading R-3 on all three axes (P even: the node set
          is then the same as the free-axis rule of the SE1P grid shifted by P/2 nodes)
  step 3  3D FFT (all axes periodic: no padding, no upsampling)
  step 4  scaling by e^{-(1-eta) k^2/4xi^2} / k^2, k != 0, and 0 at k = 0 (neutral, tin-foil):
          the 3P Green's function in place of Eq. (G_kappa_k)
  step 5  3D IFFT
  step 6  gather with the constant 4 pi h^3 (2xi^2/(pi eta))^{3/2} of reading R-1 (the 3P sum
          (4 pi/V) sum_k and the 1P mode sum share it: (1/L3)(dk/2pi)^2 sum = 1/V sum for
          dk = 2 pi/L_d).
"""
from __future__ import annotations

import math

import numpy as np

C_ETA = 0.95


def _axis_stencil(xc, h, P, M):
    """Periodic-axis rule (reading R-3): nodes l with l h in (x - w, x + w], l mod M."""
    t = np.arange(P)
    l = np.floor(xc / h - P / 2.0).astype(np.int64)[:, None] + 1 + t
    return l % M, l * h - xc[:, None]


def se3p_kspace(x, q, L, xi, M, P, eta=None):
    x = np.asarray(x, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    L1, L2, L3 = (float(v) for v in L)
    h = L3 / M
    M1, M2 = int(round(L1 / h)), int(round(L2 / h))
    if abs(M1 * h - L1) > 1e-12 * L1 or abs(M2 * h - L2) > 1e-12 * L2:
        raise ValueError("L1/h and L2/h must be integers")
    if eta is None or eta <= 0:
        eta = P * xi ** 2 * h ** 2 / (C_ETA ** 2 * math.pi)
    alpha = 2.0 * xi ** 2 / eta
    pref = (2.0 * xi ** 2 / (math.pi * eta)) ** 1.5
    dims = (M1, M2, M)
    # step 2: gridding
    H = np.zeros(M1 * M2 * M)
    st = [_axis_stencil(x[:, d], h, P, dims[d]) for d in range(3)]
    w = [np.exp(-alpha * st[d][1] ** 2) for d in range(3)]
    val = pref * q[:, None, None, None] * w[0][:, :, None, None] * w[1][:, None, :, None] * w[2][:, None, None, :]
    idx = (st[0][0][:, :, None, None] * M2 + st[1][0][:, None, :, None]) * M + st[2][0][:, None, None, :]
    H += np.bincount(idx.ravel(), weights=val.ravel(), minlength=H.size)
    H = H.reshape(dims)
    # steps 3-5: FFT, scaling, IFFT
    k = [2.0 * math.pi * np.fft.fftfreq(n, d=h) for n in dims]
    k2 = k[0][:, None, None] ** 2 + k[1][None, :, None] ** 2 + k[2][None, None, :] ** 2
    G = np.zeros(dims)
    nz = k2 > 0
    G[nz] = np.exp(-(1.0 - eta) * k2[nz] / (4.0 * xi ** 2)) / k2[nz]
    Ht = np.fft.ifftn(G * np.fft.fftn(H)).real
    # step 6: gather
    C = 4.0 * math.pi * h ** 3 * pref
    Hs = Ht.ravel()[idx]
    return C * np.einsum("ni,nj,nk,nijk->n", w[0], w[1], w[2], Hs)
