"""B200-native SE1P k-space path (arXiv:1611.09538) -- Python binding of libse1p.so.

Argument marshalling only: every step of the path runs in the CUDA kernels of
``csrc/`` behind the C ABI of ``include/se1p.h``.  There is no CPU fallback: if the
shared library is missing or fails to load, importing the functions raises.

    import torch, paper_1611_09538_b200 as se1p
    phi_k = se1p.kspace(x, q, L, xi, M, P, s0=..., sf=..., n_local=...)  # x [N,3], q [N] f64 cuda
    phi_r = se1p.real(x, q, L, xi, rc)                                  # phi^R + phi^self
    phi = phi_k + phi_r                                                 # Eq. (2)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = _build.OUT

STATUS = {0: "OK", 1: "EINVAL", 2: "EDOMAIN", 3: "ENONNEUTRAL", 4: "EPARAM", 5: "ENOMEM", 6: "ECUDA", 7: "ENCCL"}
EXPORTS = ["se1p_kspace", "se1p_kspace_ex", "se1p_real", "se1p_real_ex", "se1p_plan_query",
           "se1p_last_stage_times", "se1p_last_launch_count", "se1p_release", "se1p_last_error",
           "se1p_version", "se1p_debug_copy", "se1p_kspace_slab_forward", "se1p_kspace_modes",
           "se1p_kspace_slab_backward", "se1p_kspace_field_ex", "se1p_real_field_ex", "se1p_plan_from_tol",
           "se1p_kspace3p_ex", "se1p_kspace_tiers_ex", "se1p_set_allocator", "se1p_energy_forces",
           "se1p_real_table"]


class SE1PError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"se1p {STATUS.get(code, code)}: {msg}")
        self.code = code


class Opts(ctypes.Structure):
    _fields_ = [("Ntilde", ctypes.c_int), ("S0", ctypes.c_int), ("SI", ctypes.c_int), ("host_io", ctypes.c_int),
                ("skip_checks", ctypes.c_int), ("sync", ctypes.c_int), ("reserved", ctypes.c_int * 10)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("h", ctypes.c_double), ("eta", ctypes.c_double), ("M", ctypes.c_int), ("Mfree", ctypes.c_int),
                ("Mt", ctypes.c_int), ("P", ctypes.c_int), ("n_local", ctypes.c_int), ("Ntilde", ctypes.c_int),
                ("S0", ctypes.c_int), ("SI", ctypes.c_int), ("LK", ctypes.c_int), ("n_kernel_planes", ctypes.c_int),
                ("n_planes", ctypes.c_int), ("grid_points", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("plan_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TolPlan(ctypes.Structure):
    _d, _i = ctypes.c_double, ctypes.c_int
    _fields_ = [("xi", _d), ("tol", _d), ("Q", _d), ("rc", _d), ("kinf", _d), ("M", _i), ("P", _i), ("Mfree", _i),
                ("Mt", _i), ("h", _d), ("eta", _d), ("n_local", _i), ("s_l", _d), ("s0", _d), ("SI", _i), ("S0", _i),
                ("Ntilde", _i), ("est_real", _d), ("est_fourier", _d), ("est_approx", _d)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load(build_if_needed: bool = True):
    """Load libse1p.so (building it in-tree with nvcc if missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_needed and _build.needs_build():
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libse1p.so not found at {LIB_PATH}; run paper_1611_09538_b200/build.py")
    lib = ctypes.CDLL(LIB_PATH)
    d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.se1p_kspace.argtypes = [vp, vp, i64, vp, d, i32, i32, d, d, d, i32, vp]
    lib.se1p_kspace_ex.argtypes = [vp, vp, vp, vp, i64, vp, d, i32, i32, d, d, d, i32, vp]
    lib.se1p_real.argtypes = [vp, vp, i64, vp, d, d, vp]
    lib.se1p_real_ex.argtypes = [vp, vp, vp, vp, i64, vp, d, d, vp]
    lib.se1p_kspace_tiers_ex.argtypes = [vp, vp, vp, vp, i64, vp, d, i32, i32, d, d, i32, vp, vp]
    lib.se1p_kspace3p_ex.argtypes = [vp, vp, vp, vp, i64, vp, d, i32, i32, d, vp]
    lib.se1p_plan_from_tol.argtypes = [vp, d, d, d, vp]
    lib.se1p_kspace_field_ex.argtypes = [vp, vp, vp, vp, i64, vp, d, i32, i32, d, d, d, i32, vp, vp]
    lib.se1p_energy_forces.argtypes = [vp, vp, vp, vp, i64, vp, d, d, i32, i32, d, d, d, i32, vp, vp, vp]
    lib.se1p_energy_forces.restype = i32
    lib.se1p_real_field_ex.argtypes = [vp, vp, vp, vp, i64, vp, d, d, vp, vp]
    lib.se1p_plan_query.argtypes = [vp, vp, d, i32, i32, d, d, d, i32, vp]
    lib.se1p_last_stage_times.argtypes = [vp, i32]
    lib.se1p_last_launch_count.restype = i32
    lib.se1p_last_error.restype = ctypes.c_char_p
    lib.se1p_version.restype = ctypes.c_char_p
    lib.se1p_debug_copy.argtypes = [i32, vp, i64]
    lib.se1p_debug_copy.restype = i32
    lib.se1p_set_allocator.argtypes = [vp, vp, vp]
    lib.se1p_set_allocator.restype = i32
    lib.se1p_real_table.argtypes = [d, d, vp, vp, vp, i32]
    lib.se1p_real_table.restype = i32
    ip = ctypes.POINTER(ctypes.c_int)
    lib.se1p_kspace_slab_forward.argtypes = [vp, vp, vp, vp, i64, vp, d, i32, i32, d, d, d, i32,
                                             i32, i32, ip, vp]
    lib.se1p_kspace_modes.argtypes = [vp, vp, vp, d, i32, i32, d, d, d, i32, i32, ip, i32, ip, vp]
    lib.se1p_kspace_slab_backward.argtypes = [vp, vp, i64, vp, d, i32, i32, d, d, d, i32, i32, i32,
                                              ip, vp, vp]
    for f in ["se1p_kspace", "se1p_kspace_ex", "se1p_real", "se1p_real_ex", "se1p_plan_query", "se1p_last_stage_times",
              "se1p_kspace_slab_forward", "se1p_kspace_modes", "se1p_kspace_slab_backward"]:
        getattr(lib, f).restype = i32
    _lib = lib
    return lib


def _check(code):
    if code != 0:
        raise SE1PError(code, load().se1p_last_error().decode())


def _opts(Ntilde=None, S0=None, SI=None, host_io=False, skip_checks=False, sync=True, profile=False, stop_after=0,
          graph=False, part=None):
    o = Opts()
    o.Ntilde = int(Ntilde or 0)
    o.S0 = int(S0 or 0)
    o.SI = int(SI or 0)
    o.host_io = int(bool(host_io))
    o.skip_checks = int(bool(skip_checks))
    o.sync = int(bool(sync))
    o.reserved[0] = 1 if profile else 0
    o.reserved[1] = int(stop_after)
    o.reserved[3] = 1 if graph else 0
    if part is not None:   # (r, R): part r of R of the real-space sum (include/se1p.h)
        o.reserved[5], o.reserved[4] = int(part[0]), int(part[1])
    return o


_graph_streams = {}


def _graph_stream(x):
    """A per-device side stream for graph capture (the legacy default stream cannot be captured)."""
    import torch
    dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    if dev not in _graph_streams:
        _graph_streams[dev] = torch.cuda.Stream(device=dev)
    return _graph_streams[dev]


def _Larr(L):
    return (ctypes.c_double * 3)(*[float(v) for v in L])


def _args(x, q):
    """(x_ptr, q_ptr, N, host_io, keepalive).  torch CUDA tensors -> device pointers;
    numpy arrays -> host pointers (the library copies them)."""
    if isinstance(x, np.ndarray):
        xa = np.ascontiguousarray(x, dtype=np.float64)
        qa = np.ascontiguousarray(q, dtype=np.float64)
        return xa.ctypes.data, qa.ctypes.data, qa.shape[0], True, (xa, qa)
    import torch
    if not (x.is_cuda and q.is_cuda):
        raise TypeError("x and q must both be CUDA tensors (or both numpy arrays for host I/O)")
    if x.dtype != torch.float64 or q.dtype != torch.float64:
        raise TypeError("x and q must be float64")
    xc, qc = x.contiguous(), q.contiguous()
    if xc.dim() != 2 or xc.shape[1] != 3 or qc.shape[0] != xc.shape[0]:
        raise ValueError("x must be [N,3] and q [N]")
    return xc.data_ptr(), qc.data_ptr(), qc.shape[0], False, (xc, qc)


def _stream_ptr(stream, x):
    if isinstance(x, np.ndarray):
        return None
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    return ctypes.c_void_p(s.cuda_stream)


def _neg(v, default=-1.0):
    return default if v is None else float(v)


def _outputs(x, N, field, out, field_out):
    """Output buffers on the inputs' side (numpy for host I/O, CUDA tensors otherwise)."""
    if isinstance(x, np.ndarray):
        out = np.zeros(N) if out is None else out
        fo = (np.zeros((N, 3)) if field_out is None else field_out) if field else None
        return out, fo, out.ctypes.data, (fo.ctypes.data if field else None)
    import torch
    out = torch.empty(N, dtype=torch.float64, device=x.device) if out is None else out
    fo = (torch.empty(N, 3, dtype=torch.float64, device=x.device) if field_out is None else field_out) if field else None
    return out, fo, out.data_ptr(), (fo.data_ptr() if field else None)


def kspace(x, q, L, xi, M, P, eta=None, s0=None, sf=None, n_local=None, Ntilde=None, S0=None, SI=None,
           out=None, stream=None, sync=True, skip_checks=False, profile=False, stop_after=0,
           field=False, field_out=None, graph=False, S_modes=None):
    """phi^F = phi^{F,k3!=0} + phi^{F,k3=0} at every particle (Alg. 1).
    field=True returns (phi^F, E^F) with E^F = -grad phi^F, [N,3] (forces q E).
    graph=True captures the device stages as a CUDA graph on the first call and replays it on later
    calls with the same parameters and buffers (pass `out`/`field_out` to keep the buffers fixed).
    S_modes: multi-tier upsampling, padded extent of modes |k3| = 2 pi n/L3, n = 1..n_local
    (needs n_local; potential only)."""
    lib = load()
    xp, qp, N, host, keep = _args(x, q)
    out, fo, optr, fptr = _outputs(x, N, field, out, field_out)
    if S_modes is not None:
        if field or n_local is None or len(S_modes) != int(n_local):
            raise ValueError("S_modes needs n_local = len(S_modes) and the potential (field=False)")
        o = _opts(Ntilde, S0, None, host, skip_checks, sync, profile, stop_after, graph)
        tiers = (ctypes.c_int * len(S_modes))(*[int(s) for s in S_modes])
        _check(lib.se1p_kspace_tiers_ex(ctypes.addressof(o), _stream_ptr(stream, x), xp, qp, N, _Larr(L), float(xi),
                                        int(M), int(P), _neg(eta, 0.0), _neg(s0), int(n_local), tiers, optr))
        return out
    o = _opts(Ntilde, S0, SI, host, skip_checks, sync, profile, stop_after, graph)
    side = None
    if graph and not host and stream is None:
        import torch
        side, cur = _graph_stream(x), torch.cuda.current_stream(x.device)
        side.wait_stream(cur)
        stream = side
    args = (ctypes.addressof(o), _stream_ptr(stream, x), xp, qp, N, _Larr(L), float(xi), int(M), int(P),
            _neg(eta, 0.0), _neg(s0), _neg(sf), -1 if n_local is None else int(n_local), optr)
    if field:
        _check(lib.se1p_kspace_field_ex(*args, fptr))
    else:
        _check(lib.se1p_kspace_ex(*args))
    if side is not None:
        cur.wait_stream(side)
    return (out, fo) if field else out


def kspace3p(x, q, L, xi, M, P, eta=None, out=None, stream=None, sync=True, skip_checks=False, profile=False):
    """SE3P baseline (NEXT-4): k-space part of the triply periodic Ewald sum (tin-foil), same
    gridding/gather as kspace() with a plain 3D FFT; P even (see se1p.h)."""
    lib = load()
    xp, qp, N, host, keep = _args(x, q)
    out, _, optr, _ = _outputs(x, N, False, out, None)
    o = _opts(host_io=host, skip_checks=skip_checks, sync=sync, profile=profile)
    _check(lib.se1p_kspace3p_ex(ctypes.addressof(o), _stream_ptr(stream, x), xp, qp, N, _Larr(L), float(xi), int(M),
                                int(P), _neg(eta, 0.0), optr))
    return out


def real(x, q, L, xi, rc, out=None, stream=None, sync=True, skip_checks=False, field=False, field_out=None,
         part=None):
    """phi^R + phi^self (Eq. (3) truncated at rc, Eq. (6)).
    field=True returns (phi^R + phi^self, E^R), E^R = -grad phi^R, [N,3].
    part=(r, R): only part r of R of the targets, the other entries 0 (the R parts sum exactly)."""
    lib = load()
    xp, qp, N, host, keep = _args(x, q)
    out, fo, optr, fptr = _outputs(x, N, field, out, field_out)
    o = _opts(host_io=host, skip_checks=skip_checks, sync=sync, part=part)
    args = (ctypes.addressof(o), _stream_ptr(stream, x), xp, qp, N, _Larr(L), float(xi), float(rc), optr)
    if field:
        _check(lib.se1p_real_field_ex(*args, fptr))
        return out, fo
    _check(lib.se1p_real_ex(*args))
    return out


def _tol_params(q, L, xi, tol):
    """(rc, M, P, kspace kwargs) from plan_from_tol for this system's Q = sum q^2."""
    Q = float((q * q).sum())
    plan = plan_from_tol(L, Q, xi, tol)
    M, P, kw = kspace_args(plan)
    return plan["rc"], M, P, kw


def potential(x, q, L, xi, rc=None, M=None, P=None, tol=None, **kw):
    """Full singly periodic potential phi = phi^F + phi^R + phi^self (Eq. (2)).
    Either rc, M, P (and kspace keywords) or tol: the parameters from plan_from_tol (NEXT-2)."""
    if tol is not None:
        rc, M, P, kw2 = _tol_params(q, L, xi, tol)
        kw = {**kw2, **kw}
    if rc is None or M is None or P is None:
        raise ValueError("give rc, M, P or tol")
    return kspace(x, q, L, xi, M, P, **kw) + real(x, q, L, xi, rc)


def energy_forces(x, q, L, xi, rc=None, M=None, P=None, tol=None, stream=None, sync=True, skip_checks=False,
                  eta=None, s0=None, sf=None, n_local=None, Ntilde=None, S0=None, SI=None):
    """(U, phi, F) from se1p_energy_forces: the electrostatic energy U = 1/2 sum_n q_n phi_n, the
    potentials phi = phi^F + phi^R + phi^self and the forces F_n = q_n E_n, E = E^F + E^R (Eq. (2)
    and its gradient), all computed in the library.  rc, M, P or tol as in potential().
    CUDA tensors in -> CUDA tensors out (U a 0-d tensor); numpy in -> numpy out (U a float)."""
    if tol is not None:
        rc, M, P, kw2 = _tol_params(q, L, xi, tol)
        eta, n_local, S0, SI, Ntilde = kw2["eta"], kw2["n_local"], kw2["S0"], kw2["SI"], kw2["Ntilde"]
    if rc is None or M is None or P is None:
        raise ValueError("give rc, M, P or tol")
    lib = load()
    xp, qp, N, host, keep = _args(x, q)
    phi, F, pptr, fptr = _outputs(x, N, True, None, None)
    if host:
        U = np.zeros(1)
        uptr = U.ctypes.data
    else:
        import torch
        U = torch.zeros((), dtype=torch.float64, device=x.device)
        uptr = U.data_ptr()
    o = _opts(Ntilde, S0, SI, host, skip_checks, sync)
    _check(lib.se1p_energy_forces(ctypes.addressof(o), _stream_ptr(stream, x), xp, qp, N, _Larr(L), float(xi),
                                  float(rc), int(M), int(P), _neg(eta, 0.0), _neg(s0), _neg(sf),
                                  -1 if n_local is None else int(n_local), uptr, pptr, fptr))
    return (float(U[0]) if host else U), phi, F


def _ints(v):
    v = [int(a) for a in v]
    return (ctypes.c_int * max(1, len(v)))(*v)


def slab_forward(x, q, L, xi, M, P, x_lo, x_hi, plane_order, out=None, stream=None, sync=False,
                 skip_checks=False, eta=None, s0=None, sf=None, n_local=None, Ntilde=None, S0=None, SI=None):
    """Distributed path, rank stage 1 (include/se1p.h): grid the slab rows [x_lo, x_hi) and
    z-transform them.  Returns the slab buffer, float64 [M/2+1, x_hi-x_lo, M~, 2] (re, im)."""
    import torch
    lib = load()
    xp, qp, N, host, keep = _args(x, q)
    if host:
        raise TypeError("the distributed entries take CUDA tensors")
    n_planes = int(M) // 2 + 1
    info = plan_info(L, xi, M, P, eta=eta, s0=s0, sf=sf, n_local=n_local, Ntilde=Ntilde, S0=S0, SI=SI)
    if out is None:
        out = torch.empty((n_planes, x_hi - x_lo, info["Mt"], 2), dtype=torch.float64, device=x.device)
    o = _opts(Ntilde, S0, SI, False, skip_checks, sync)
    _check(lib.se1p_kspace_slab_forward(ctypes.addressof(o), _stream_ptr(stream, x), xp, qp, N, _Larr(L), float(xi),
                                        int(M), int(P), _neg(eta, 0.0), _neg(s0), _neg(sf),
                                        -1 if n_local is None else int(n_local), int(x_lo), int(x_hi),
                                        _ints(plane_order), out.data_ptr()))
    return out


def modes(planes, L, xi, M, P, plane_ids, slab_lo, stream=None, sync=False, eta=None, s0=None, sf=None,
          n_local=None, Ntilde=None, S0=None, SI=None):
    """Distributed path, rank stage 2: the mode stage on the owner's split buffer (in place)."""
    lib = load()
    o = _opts(Ntilde, S0, SI, False, False, sync)
    _check(lib.se1p_kspace_modes(ctypes.addressof(o), _stream_ptr(stream, planes), _Larr(L), float(xi), int(M), int(P),
                                 _neg(eta, 0.0), _neg(s0), _neg(sf), -1 if n_local is None else int(n_local),
                                 len(plane_ids), _ints(plane_ids), len(slab_lo) - 1, _ints(slab_lo),
                                 planes.data_ptr()))
    return planes


def slab_backward(planes, N, L, xi, M, P, x_lo, x_hi, plane_order, out=None, stream=None, sync=False, eta=None,
                  s0=None, sf=None, n_local=None, Ntilde=None, S0=None, SI=None):
    """Distributed path, rank stage 3: inverse z-transform of the slab rows and the gather over the
    slab's tiles.  Returns phi_partial [N] (user order)."""
    import torch
    lib = load()
    if out is None:
        out = torch.empty(int(N), dtype=torch.float64, device=planes.device)
    o = _opts(Ntilde, S0, SI, False, False, sync)
    _check(lib.se1p_kspace_slab_backward(ctypes.addressof(o), _stream_ptr(stream, planes), int(N), _Larr(L), float(xi),
                                         int(M), int(P), _neg(eta, 0.0), _neg(s0), _neg(sf),
                                         -1 if n_local is None else int(n_local), int(x_lo), int(x_hi),
                                         _ints(plane_order), planes.data_ptr(), out.data_ptr()))
    return out


def plan_info(L, xi, M, P, eta=None, s0=None, sf=None, n_local=None, Ntilde=None, S0=None, SI=None):
    lib = load()
    info = PlanInfo()
    o = _opts(Ntilde, S0, SI)
    _check(lib.se1p_plan_query(ctypes.addressof(o), _Larr(L), float(xi), int(M), int(P), _neg(eta, 0.0), _neg(s0),
                               _neg(sf), -1 if n_local is None else int(n_local), ctypes.addressof(info)))
    return info.as_dict()


def plan_from_tol(L, Q, xi, tol):
    """Parameters for an absolute rms error tolerance by the paper's recipe (host
    only).  Returns a dict: rc, kinf, M, P, eta, n_local, s_l, s0, extents SI, S0, Ntilde and the
    three error estimates.  `kspace_args(plan)` turns it into kspace() keyword arguments."""
    lib = load()
    out = TolPlan()
    _check(lib.se1p_plan_from_tol(_Larr(L), float(Q), float(xi), float(tol), ctypes.addressof(out)))
    return out.as_dict()


def real_table(xi, rc):
    """(degree, intervals, coefficients [degree + 1, intervals]) of the real-space kernel's erfc
    table (host only; include/se1p.h se1p_real_table); degree 0: fallback kernel, no table."""
    import numpy as np
    lib = load()
    deg, K = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib.se1p_real_table(ctypes.c_double(xi), ctypes.c_double(rc), ctypes.byref(deg), ctypes.byref(K), None, 0))
    c = np.zeros((deg.value + 1) * K.value if deg.value > 0 else 0)
    if deg.value > 0:
        _check(lib.se1p_real_table(ctypes.c_double(xi), ctypes.c_double(rc), ctypes.byref(deg), ctypes.byref(K),
                                   c.ctypes.data_as(ctypes.c_void_p), int(c.size)))
    return deg.value, K.value, c.reshape(deg.value + 1, K.value) if deg.value > 0 else c


def kspace_args(plan):
    """(M, P, kwargs) of kspace() for a plan_from_tol() result."""
    return plan["M"], plan["P"], dict(eta=plan["eta"], n_local=plan["n_local"], S0=plan["S0"], SI=plan["SI"],
                                      Ntilde=plan["Ntilde"])


def stage_times():
    """Per-stage device ms of the last profiled call (CUDA events on the call's stream):
    bin, records, spread, zfft, modes, izfft, gather, finish."""
    buf = (ctypes.c_double * 10)()
    n = load().se1p_last_stage_times(buf, 10)
    names = ["bin", "records", "spread", "zfft", "modes", "izfft", "gather", "finish"]
    return {names[i]: buf[i] for i in range(n)}


def launch_count():
    return load().se1p_last_launch_count()


def debug_stage(x, q, L, xi, M, P, stage, **kw):
    """Testing hook: run the k-space path up to `stage` (1 gridding, 2 z-FFT, 3 modes, 4 inverse
    z-FFT) and return the workspace buffer (real grid [Mt,Mt,M] or planes [M/2+1,Mt,Mt] complex)."""
    info = plan_info(L, xi, M, P, **{k: kw.get(k) for k in ("eta", "s0", "sf", "n_local", "Ntilde", "S0", "SI")})
    kspace(x, q, L, xi, M, P, stop_after=stage, **kw)
    Mt, Mz = info["Mt"], info["M"]
    if stage in (1, 4):
        buf = np.zeros(Mt * Mt * Mz)
        _check(load().se1p_debug_copy(0, buf.ctypes.data, buf.size))
        return buf.reshape(Mt, Mt, Mz)
    buf = np.zeros(2 * (Mz // 2 + 1) * Mt * Mt)
    _check(load().se1p_debug_copy(1, buf.ctypes.data, buf.size))
    return buf.view(np.complex128).reshape(Mz // 2 + 1, Mt, Mt)


def release():
    load().se1p_release()


_ALLOC_T = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_RELEASE_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)
_allocator_refs = None   # the installed callbacks (kept alive while the library may call them)


def _torch_alloc(nbytes, _ctx):
    try:
        import torch
        return torch.cuda.caching_allocator_alloc(int(nbytes))
    except Exception:   # noqa: BLE001 -- NULL tells the library (SE1P_ENOMEM)
        return None


def _torch_release(ptr, _ctx):
    import torch
    torch.cuda.caching_allocator_delete(int(ptr))


def use_torch_allocator(enable: bool = True):
    """Route the library's device memory (plans, workspaces, tables) through torch's caching
    allocator (include/se1p.h se1p_set_allocator; SURVEY.md 8(b) "Ownership"), or back to
    cudaMalloc with enable=False.  Frees everything the library holds first."""
    global _allocator_refs
    lib = load()
    if enable:
        refs = (_ALLOC_T(_torch_alloc), _RELEASE_T(_torch_release))
        _check(lib.se1p_set_allocator(ctypes.cast(refs[0], ctypes.c_void_p), ctypes.cast(refs[1], ctypes.c_void_p),
                                      None))
        _allocator_refs = refs
    else:
        _check(lib.se1p_set_allocator(None, None, None))
        _allocator_refs = None


def version():
    return load().se1p_version().decode()
