"""Algorithm 1 of PAPER.md (SE1P k-space), step by step, in plain numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  This is the discrete quantity the CUDA
path computes; it follows the paper's order and notation with library FFTs as the only
primitives and no blocking, fusion or reordering:

  step 1  h = L3/M, M~ = M+P, L~ = M~ h, eta = P xi^2 h^2 / (c^2 pi), c = 0.95
  step 2  gridding H on the M~ x M~ x M grid, Eq. (spread_1p)
  step 3  AFT (Alg. 2): 1D FFT in z, then per-k3 2D FFTs zero-padded to S x S
  step 4  scaling by e^{-(1-eta)(kappa^2+k3^2)/4xi^2} Ghat(kappa,k3), Eq. (G_kappa_k)
  step 5  AIFT (Alg. 3): 2D IFFTs restricted to the M~ x M~ block, then 1D IFFT in z
  step 6  gather, Eq. (se1p_complete_discretized) with the constant of reading R-1

Readings of the paper taken here (DESIGN.md lists them):
  R-1  gather constant: phi = 4 pi h^3 (2xi^2/(pi eta))^{3/2} sum H~ W, with H~ the normalised
       inverse transform of the scaled unnormalised transform of H.  Derived from Eq. (4a)
       and the split; the printed 2/L3 differs by 2 pi.
  R-3  stencil: free axes use nodes j with grid coordinate (j - P/2) h inside (x - w, x + w],
       w = P h/2, i.e. j = floor(x/h)+1 .. floor(x/h)+P; the periodic axis uses nodes l with
       l h in (z - w, z + w], distances unwrapped (closest periodic distance), l mod M.
  R-4  AIFT restricts to the M~ x M~ extended block (P:767-768 say "M"; the gather needs M~).
  R-5  padded extents are explicit integers S0 (k3 = 0), SI (0 < |k3| <= 2 pi n_l / L3) and
       SJ (the rest); the paper's s0, s_l map to S = ceil(s M~) ("s M~ integer").
  R-6  R = sqrt(L~1^2 + L~2^2) (= sqrt(2) L~, for the square cross-sections used here).
"""
from __future__ import annotations

import math

import numpy as np
from scipy import special

C_ETA = 0.95


def derived(L, xi, M, P, eta=None):
    """Step 1 of Alg. 1."""
    L1, L2, L3 = (float(v) for v in L)
    h = L3 / M
    M1 = int(round(L1 / h))
    M2 = int(round(L2 / h))
    if abs(M1 * h - L1) > 1e-12 * L1 or abs(M2 * h - L2) > 1e-12 * L2:
        raise ValueError("L1/h and L2/h must be integers")
    Mt1, Mt2 = M1 + P, M2 + P
    if eta is None or eta <= 0:
        eta = P * xi ** 2 * h ** 2 / (C_ETA ** 2 * math.pi)          # Eq. (comp_eta)
    return dict(h=h, M1=M1, M2=M2, Mt1=Mt1, Mt2=Mt2, Lt1=Mt1 * h, Lt2=Mt2 * h, eta=eta)


def _stencils(x, h, P, M):
    """Reading R-3: node indices and signed distances (node - particle) per axis."""
    t = np.arange(P)
    jx = np.floor(x[:, 0] / h).astype(np.int64)[:, None] + 1 + t          # free axis 1
    jy = np.floor(x[:, 1] / h).astype(np.int64)[:, None] + 1 + t          # free axis 2
    dx = (jx - P / 2.0) * h - x[:, 0:1]
    dy = (jy - P / 2.0) * h - x[:, 1:2]
    lz = np.floor(x[:, 2] / h - P / 2.0).astype(np.int64)[:, None] + 1 + t  # periodic axis
    dz = lz * h - x[:, 2:3]
    return jx, jy, lz % M, dx, dy, dz


def gridding(x, q, xi, h, P, M, Mt1, Mt2, eta, chunk=2048):
    """Step 2: H(r,z) = (2xi^2/(pi eta))^{3/2} sum_n q_n e^{-2xi^2|r-r_n|^2/eta} e^{-2xi^2 (z-z_n)_*^2/eta}
    on the M~1 x M~2 x M grid, each Gaussian truncated to its P^3 support (Eq. spread_1p)."""
    alpha = 2.0 * xi ** 2 / eta
    pref = (2.0 * xi ** 2 / (math.pi * eta)) ** 1.5
    H = np.zeros(Mt1 * Mt2 * M)
    for s in range(0, q.size, chunk):
        xs, qs = x[s:s + chunk], q[s:s + chunk]
        jx, jy, lz, dx, dy, dz = _stencils(xs, h, P, M)
        wx, wy, wz = np.exp(-alpha * dx ** 2), np.exp(-alpha * dy ** 2), np.exp(-alpha * dz ** 2)
        val = pref * qs[:, None, None, None] * wx[:, :, None, None] * wy[:, None, :, None] * wz[:, None, None, :]
        idx = (jx[:, :, None, None] * Mt2 + jy[:, None, :, None]) * M + lz[:, None, None, :]
        H += np.bincount(idx.ravel(), weights=val.ravel(), minlength=H.size)
    return H.reshape(Mt1, Mt2, M)


def ghat(kappa2, k3, R):
    """Eq. (G_kappa_k): 1/(kappa^2+k3^2) for k3 != 0; truncated free-space kernel
    (Vico) for k3 = 0, Eqs. (g_zeromod), (g_zeromod0)."""
    if k3 != 0.0:
        return 1.0 / (kappa2 + k3 * k3)
    kappa = np.sqrt(kappa2)
    out = np.empty_like(kappa)
    nz = kappa > 0
    kn = kappa[nz]
    out[nz] = (1.0 - special.j0(R * kn)) / kn ** 2 - R * math.log(R) * special.j1(R * kn) / kn
    out[~nz] = R ** 2 / 4.0 * (1.0 - 2.0 * math.log(R))
    return out


def mode_extent(nprime, n_l, S0, SI, SJ):
    """Adaptive upsampling, Eq. (upsamplings), as padded extents (reading R-5).
    SI may be a sequence: the extent of |n| = 1..n_l (multi-tier)."""
    if nprime == 0:
        return S0
    if abs(nprime) <= n_l:
        return SI[abs(nprime) - 1] if hasattr(SI, "__len__") else SI
    return SJ


def se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ, eta=None, return_all=False, return_field=False):
    """phi^F(x_m) = phi^{F,k3!=0} + phi^{F,k3=0} by Alg. 1; with return_field also the
    k-space field E^F = -grad phi^F at the particles (the SE force is the gradient of the gather,
    Eq. (force_se1p); the constant follows reading R-1)."""
    x = np.asarray(x, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    d = derived(L, xi, M, P, eta)
    h, Mt1, Mt2, eta = d["h"], d["Mt1"], d["Mt2"], d["eta"]
    if Mt1 != Mt2:
        raise ValueError("square free cross-section required (M1 == M2)")
    L3 = float(L[2])
    R = math.hypot(d["Lt1"], d["Lt2"])                                   # reading R-6
    for S in (S0, SJ, *(SI if hasattr(SI, "__len__") else (SI,))):
        if S < Mt1:
            raise ValueError("padded extents must be >= M~")

    # step 2: gridding
    H = gridding(x, q, xi, h, P, M, Mt1, Mt2, eta)

    # step 3: AFT, Alg. 2.  Step 1: 1D FFT along z.
    Hz = np.fft.fft(H, axis=2)
    Ht = np.zeros_like(Hz)
    for n in range(M):
        nprime = n if n < M // 2 else n - M          # k3 index in {-M/2, ..., M/2-1}
        k3 = 2.0 * math.pi * nprime / L3
        S = mode_extent(nprime, n_l, S0, SI, SJ)
        # steps 2-4 of Alg. 2: zero-pad to S x S and 2D FFT
        F = np.fft.fft2(Hz[:, :, n], s=(S, S))
        # step 4 of Alg. 1: scale, Eq. (scale_1p); kappa = 2 pi a'/(S h), a' in {-S/2..S/2-1}
        kap = 2.0 * math.pi * np.fft.fftfreq(S, d=h)
        kappa2 = kap[:, None] ** 2 + kap[None, :] ** 2
        F *= np.exp(-(1.0 - eta) * (kappa2 + k3 ** 2) / (4.0 * xi ** 2)) * ghat(kappa2, k3, R)
        # step 5: AIFT, Alg. 3 steps 1-3: 2D IFFT, restrict to the M~ x M~ block (reading R-4)
        Ht[:, :, n] = np.fft.ifft2(F)[:Mt1, :Mt2]
    # Alg. 3 steps 4-5: merge and 1D IFFT along z
    Htil = np.fft.ifft(Ht, axis=2).real

    # step 6: gather (reading R-1 for the constant)
    phi, E = _gather(x, Htil, xi, d["h"], P, M, Mt2, eta, field=return_field)
    if return_field:
        return (phi, E, dict(H=H, Htilde=Htil, derived=d, R=R)) if return_all else (phi, E)
    if return_all:
        return phi, dict(H=H, Htilde=Htil, derived=d, R=R)
    return phi


def _gather(x, Htil, xi, h, P, M, Mt2, eta, field=False):
    """Step 6: phi(x_m) = C sum H~ wx wy wz (Eq. (se1p_complete_discretized), reading R-1), and with
    `field` the electric field E = -grad phi: d/dx_m e^{-alpha (node - x_m)^2} = 2 alpha (node - x_m) w."""
    alpha = 2.0 * xi ** 2 / eta
    pref = (2.0 * xi ** 2 / (math.pi * eta)) ** 1.5
    C = 4.0 * math.pi * h ** 3 * pref
    phi = np.empty(x.shape[0])
    E = np.empty((x.shape[0], 3)) if field else None
    flat = Htil.ravel()
    for s in range(0, x.shape[0], 2048):
        xs = x[s:s + 2048]
        jx, jy, lz, dx, dy, dz = _stencils(xs, h, P, M)
        wx, wy, wz = np.exp(-alpha * dx ** 2), np.exp(-alpha * dy ** 2), np.exp(-alpha * dz ** 2)
        idx = (jx[:, :, None, None] * Mt2 + jy[:, None, :, None]) * M + lz[:, None, None, :]
        Hs = flat[idx]
        phi[s:s + 2048] = C * np.einsum("ni,nj,nk,nijk->n", wx, wy, wz, Hs)
        if field:
            gx, gy, gz = 2 * alpha * dx * wx, 2 * alpha * dy * wy, 2 * alpha * dz * wz
            E[s:s + 2048, 0] = -C * np.einsum("ni,nj,nk,nijk->n", gx, wy, wz, Hs)
            E[s:s + 2048, 1] = -C * np.einsum("ni,nj,nk,nijk->n", wx, gy, wz, Hs)
            E[s:s + 2048, 2] = -C * np.einsum("ni,nj,nk,nijk->n", wx, wy, gz, Hs)
    return phi, E


def extents_from_factors(Mt, s0, sl, SJ=None):
    """Paper's factors -> integer extents, rounding s M~ up (reading R-5)."""
    S0 = int(math.ceil(s0 * Mt - 1e-9))
    SI = int(math.ceil(sl * Mt - 1e-9))
    return S0, SI, (Mt if SJ is None else SJ)
