"""CPU oracle for the SE1P k-space path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_1611_09538_b200`` never imports it and shares no code with it.

Two layers:

* ``ewald1p.c`` (compiled to ``liborc.so``): the plain definition of the singly periodic
  Coulomb potential through the Ewald1P formulas, Eqs. (1)-(6) of PAPER.md, with
  the special functions of Appendix A.  This is the exact answer the fast
  method approximates.
* ``se1p_discrete.py``: Algorithm 1 with the AFT/AIFT of Algorithms 2/3
   written out step by step in numpy -- the discrete quantity the CUDA path
  computes, used for element-wise parity at tight tolerance.

Pins (tests/test_oracle_*.py) tie both to things other than themselves: brute-force image
sums, the coaxial-pair digamma closed form, xi-invariance, scipy/mpmath special
functions, the Kolafa-Perram estimates and the exact Ewald sum within the
error bounds of Theorem 1.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ewald1p.c")
_SRCS = [_SRC, os.path.join(_HERE, "ewald3p.c")]
_LIB = os.path.join(_HERE, "liborc.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
               "-o", _LIB, *_SRCS, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        lib.orc_e1.restype = d
        lib.orc_e1.argtypes = [d]
        lib.orc_g.restype = d
        lib.orc_g.argtypes = [d]
        lib.orc_k0.restype = d
        lib.orc_k0.argtypes = [d]
        lib.orc_K0inc.restype = d
        lib.orc_K0inc.argtypes = [d, d]
        lib.orc_gauss_legendre.argtypes = [i32, P, P]
        lib.orc_phi_real.argtypes = [P, P, i64, P, d, d, P, i64, P]
        lib.orc_phi_k3nz.argtypes = [P, P, i64, P, d, i32, P, i64, P]
        lib.orc_phi_k30.argtypes = [P, P, i64, P, d, P, i64, P]
        lib.orc_phi_self.argtypes = [P, d, P, i64, P]
        lib.orc_phi_exact.argtypes = [P, P, i64, P, d, P, i64, P, P]
        lib.orc_phi_brute.argtypes = [P, P, i64, P, i64, P, i64, P]
        lib.orc_dK0db.restype = d
        lib.orc_dK0db.argtypes = [d, d]
        lib.orc_field_real.argtypes = [P, P, i64, P, d, d, P, i64, P]
        lib.orc_field_k3nz.argtypes = [P, P, i64, P, d, i32, P, i64, P]
        lib.orc_field_k30.argtypes = [P, P, i64, P, d, P, i64, P]
        lib.orc_field_exact.argtypes = [P, P, i64, P, d, P, i64, P, P]
        lib.orc_field_brute.argtypes = [P, P, i64, P, i64, P, i64, P]
        lib.orc3_phi_real.argtypes = [P, P, i64, P, d, d, P, i64, P]
        lib.orc3_phi_kspace.argtypes = [P, P, i64, P, d, i32, P, i64, P]
        lib.orc3_phi_exact.argtypes = [P, P, i64, P, d, P, i64, P]
        lib.orc3_rc_converged.restype = d
        lib.orc3_rc_converged.argtypes = [d]
        lib.orc3_kmax_converged.restype = i32
        lib.orc3_kmax_converged.argtypes = [d, P]
        lib.orc_modes_needed.restype = i32
        lib.orc_modes_needed.argtypes = [d, d]
        lib.orc_rc_converged.restype = d
        lib.orc_rc_converged.argtypes = [d]
        lib.orc_threads.restype = i32
        lib.orc_threads.argtypes = []
        _lib = lib
    return _lib


def threads_used(N, m):
    """OpenMP threads the source sums of phi_exact keep busy for m targets of an N-particle
    system: the work items are (target, source block) pairs (ewald1p.c, orc_src_blocks)."""
    blocks = 1 if N < 65536 else 64
    return int(min(_load().orc_threads(), m * blocks))


def _prep(x, q, L, targets):
    x = np.ascontiguousarray(x, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    L = np.ascontiguousarray(L, dtype=np.float64)
    N = q.shape[0]
    if targets is None:
        targets = np.arange(N, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.int64)
    out = np.zeros(targets.shape[0], dtype=np.float64)
    return x, q, L, N, targets, out


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- special functions
def e1(v):
    return _load().orc_e1(float(v))


def g(u):
    """gamma + log u + E1(u)."""
    return _load().orc_g(float(u))


def k0(v):
    return _load().orc_k0(float(v))


def K0inc(a, b):
    """Incomplete modified Bessel function K0(a,b) (App. A)."""
    return _load().orc_K0inc(float(a), float(b))


def gauss_legendre():
    xs = np.zeros(32)
    ws = np.zeros(32)
    _load().orc_gauss_legendre(32, _p(xs), _p(ws))
    return xs, ws


# ---------------------------------------------------------------- Ewald1P terms
def phi_real(x, q, L, xi, rc, targets=None):
    """phi^R, Eq. (3), truncated at d <= rc.  rc=None -> converged (erfc(6.6) ~ 1e-20)."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    if rc is None:
        rc = lib.orc_rc_converged(float(xi))
    lib.orc_phi_real(_p(x), _p(q), N, _p(L), float(xi), float(rc), _p(targets), targets.size, _p(out))
    return out


def phi_k3nz(x, q, L, xi, J=None, targets=None):
    """phi^{F,k3!=0}, Eq. (4b) P:88 (modes |j| <= J)."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    if J is None:
        J = lib.orc_modes_needed(float(xi), float(L[2]))
    lib.orc_phi_k3nz(_p(x), _p(q), N, _p(L), float(xi), int(J), _p(targets), targets.size, _p(out))
    return out


def phi_k30(x, q, L, xi, targets=None):
    """phi^{F,k3=0}, Eq. (5) P:89."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    lib.orc_phi_k30(_p(x), _p(q), N, _p(L), float(xi), _p(targets), targets.size, _p(out))
    return out


def phi_self(q, xi, targets=None):
    """phi^self, Eq. (6) P:90."""
    lib = _load()
    q = np.ascontiguousarray(q, dtype=np.float64)
    if targets is None:
        targets = np.arange(q.size, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.int64)
    out = np.zeros(targets.size)
    lib.orc_phi_self(_p(q), float(xi), _p(targets), targets.size, _p(out))
    return out


def phi_exact(x, q, L, targets=None, xi_o=0.0, components=False):
    """Full potential phi(x_m), Eq. (2) at the oracle's own xi_o (default 0.7/L3), converged."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    comps = np.zeros((targets.size, 4)) if components else None
    lib.orc_phi_exact(_p(x), _p(q), N, _p(L), float(xi_o), _p(targets), targets.size, _p(out),
                      _p(comps) if components else None)
    return (out, comps) if components else out


def phi_brute(x, q, L, A, targets=None):
    """Eq. (1) with P_1 images |alpha| <= A, symmetric (no extrapolation)."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    lib.orc_phi_brute(_p(x), _p(q), N, _p(L), int(A), _p(targets), targets.size, _p(out))
    return out


def phi_brute_extrapolated(x, q, L, A=2000, targets=None):
    """Richardson extrapolation of the O(A^-2) tail: (4 S(2A) - S(A)) / 3."""
    s1 = phi_brute(x, q, L, A, targets)
    s2 = phi_brute(x, q, L, 2 * A, targets)
    return (4.0 * s2 - s1) / 3.0


def phi_kspace_reference(x, q, L, xi, targets=None):
    """phi^F(xi) = phi^{F,k3!=0} + phi^{F,k3=0} at the caller's xi, obtained from the exact
    total: phi - phi^R(xi, converged) - phi^self(xi) (Eq. (2)).  Cheap at any xi."""
    tot = phi_exact(x, q, L, targets)
    return tot - phi_real(x, q, L, xi, None, targets) - phi_self(q, xi, targets)


def dK0db(a, b):
    """dK0(a,b)/db = -int_0^1 e^{-a/s - bs} ds (P:95 differentiated)."""
    return _load().orc_dK0db(float(a), float(b))


def _field(fn, x, q, L, targets, *args):
    x, q, L, N, targets, _ = _prep(x, q, L, targets)
    out = np.zeros((targets.size, 3))
    fn(_p(x), _p(q), N, _p(L), *args, _p(targets), targets.size, _p(out))
    return out


def field_real(x, q, L, xi, rc, targets=None):
    """E^R = -grad phi^R at each target (Eq. (3) differentiated), truncated at d <= rc (None: converged)."""
    lib = _load()
    if rc is None:
        rc = lib.orc_rc_converged(float(xi))
    return _field(lib.orc_field_real, x, q, L, targets, float(xi), float(rc))


def field_k3nz(x, q, L, xi, J=None, targets=None):
    lib = _load()
    if J is None:
        J = lib.orc_modes_needed(float(xi), float(np.asarray(L, dtype=float)[2]))
    return _field(lib.orc_field_k3nz, x, q, L, targets, float(xi), int(J))


def field_k30(x, q, L, xi, targets=None):
    return _field(_load().orc_field_k30, x, q, L, targets, float(xi))


def field_exact(x, q, L, targets=None, xi_o=0.0):
    """E = -grad phi at each target (own charge excluded), converged at xi_o; force = q E."""
    lib = _load()
    x, q, L, N, targets, _ = _prep(x, q, L, targets)
    out = np.zeros((targets.size, 3))
    lib.orc_field_exact(_p(x), _p(q), N, _p(L), float(xi_o), _p(targets), targets.size, _p(out), None)
    return out


def field_brute(x, q, L, A, targets=None):
    return _field(_load().orc_field_brute, x, q, L, targets, int(A))


def field_brute_extrapolated(x, q, L, A=2000, targets=None):
    return (4.0 * field_brute(x, q, L, 2 * A, targets) - field_brute(x, q, L, A, targets)) / 3.0


def field_kspace_reference(x, q, L, xi, targets=None):
    """E^F(xi) = E - E^R(xi, converged) (the self term has no gradient)."""
    return field_exact(x, q, L, targets) - field_real(x, q, L, xi, None, targets)


def rel_rms(a, ref):
    """Relative rms error sqrt(sum (a-ref)^2 / sum ref^2) (P:123-126 normalised)."""
    a = np.asarray(a)
    ref = np.asarray(ref)
    return float(np.sqrt(np.sum((a - ref) ** 2) / np.sum(ref ** 2)))


# ---------------------------------------------------------------- triply periodic (NEXT-4)
# ewald3p.c: the classic 3P Ewald sum (tin-foil), the SE3P baseline's exact answer.

def phi3_real(x, q, L, xi, rc=None, targets=None):
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    if rc is None:
        rc = lib.orc3_rc_converged(float(xi))
    lib.orc3_phi_real(_p(x), _p(q), N, _p(L), float(xi), float(rc), _p(targets), targets.size, _p(out))
    return out


def phi3_kspace(x, q, L, xi, K=None, targets=None):
    """(4 pi/V) sum_{k != 0, |j_d| <= K} e^{-k^2/4xi^2}/k^2 sum_n q_n cos(k.(x_m - x_n)); K=None: converged."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    if K is None:
        K = lib.orc3_kmax_converged(float(xi), _p(L))
    lib.orc3_phi_kspace(_p(x), _p(q), N, _p(L), float(xi), int(K), _p(targets), targets.size, _p(out))
    return out


def phi3_exact(x, q, L, targets=None, xi_o=0.0):
    """Triply periodic potential (tin-foil boundary), converged Ewald sum at the oracle's xi_o."""
    lib = _load()
    x, q, L, N, targets, out = _prep(x, q, L, targets)
    lib.orc3_phi_exact(_p(x), _p(q), N, _p(L), float(xi_o), _p(targets), targets.size, _p(out))
    return out
