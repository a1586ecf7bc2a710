"""CPU tests of the mode-sharded distributed path (paper_1611_09538_b200/dist.py).

The index bookkeeping (slab bounds, LPT plane ownership, plane order, all-to-all split sizes)
and the SPMD orchestration run here over torch.distributed with the gloo backend (world size
2 and 3, 127.0.0.1).  The per-rank stages are a numpy test double that follows Alg. 1 with the
same slab/plane decomposition (gridding of the slab rows, z-FFT, per-plane adaptive 2D
transform and scaling, inverse z-FFT of the slab rows, gather restricted to the slab rows);
the assembled result must equal the single-process Alg. 1 oracle.  The CUDA stages themselves
are covered on the GPU by tests/test_gpu_dist.py.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import se1p_discrete as sd
from paper_1611_09538_b200 import dist as sdist
from se1p_synth import make_system

CASE = dict(N=40, L=(1.0, 1.0, 1.0), xi=4.0, M=16, P=8, n_l=2, S0=72, SI=60, SJ=30, seed=3)


class NumpyStages:
    """Test double of the three per-rank stages (include/se1p.h distributed entries)."""

    def __init__(self, L, xi, M, P, n_l, S0, SI, SJ):
        self.L, self.xi, self.M, self.P = L, xi, M, P
        self.n_l, self.S0, self.SI, self.SJ = n_l, S0, SI, SJ
        d = sd.derived(L, xi, M, P)
        self.d = d
        self.Mt = d["Mt1"]
        self.n_planes = M // 2 + 1
        self.R_vico = math.hypot(d["Lt1"], d["Lt2"])

    def forward(self, x, q, x_lo, x_hi, order):
        d = self.d
        self.x = x.numpy()   # the particles a later backward gathers (the device keeps them the same way)
        H = sd.gridding(x.numpy(), q.numpy(), self.xi, d["h"], self.P, self.M, self.Mt, self.Mt, d["eta"])
        Hz = np.fft.fft(H, axis=2)[:, :, :self.n_planes]
        slab = np.ascontiguousarray(np.stack([Hz[x_lo:x_hi, :, n] for n in order]))   # [slot][W][Mt]
        out = np.empty(slab.shape + (2,))
        out[..., 0], out[..., 1] = slab.real, slab.imag
        return torch.from_numpy(out)

    def _plane(self, F, n):
        d, h = self.d, self.d["h"]
        S = sd.mode_extent(n, self.n_l, self.S0, self.SI, self.SJ)
        k3 = 2.0 * math.pi * n / self.L[2]
        G = np.fft.fft2(F, s=(S, S))
        kap = 2.0 * math.pi * np.fft.fftfreq(S, d=h)
        k2 = kap[:, None] ** 2 + kap[None, :] ** 2
        G *= np.exp(-(1.0 - d["eta"]) * (k2 + k3 ** 2) / (4.0 * self.xi ** 2)) * sd.ghat(k2, k3, self.R_vico)
        return np.fft.ifft2(G)[:self.Mt, :self.Mt]

    def modes(self, buf, plane_ids, bounds):
        Mt, nown = self.Mt, len(plane_ids)
        if nown == 0:
            return buf
        c = buf.numpy().reshape(-1).view(np.complex128)
        planes = np.zeros((nown, Mt, Mt), dtype=np.complex128)
        off = 0
        for r in range(len(bounds) - 1):
            W = bounds[r + 1] - bounds[r]
            blk = c[off:off + nown * W * Mt].reshape(nown, W, Mt)
            planes[:, bounds[r]:bounds[r + 1], :] = blk
            off += nown * W * Mt
        out = np.stack([self._plane(planes[i], n) for i, n in enumerate(plane_ids)])
        off = 0
        for r in range(len(bounds) - 1):
            W = bounds[r + 1] - bounds[r]
            c[off:off + nown * W * Mt] = out[:, bounds[r]:bounds[r + 1], :].reshape(-1)
            off += nown * W * Mt
        return buf

    def backward(self, buf, N, x_lo, x_hi, order):
        self_ = self
        M, Mt, d = self.M, self.Mt, self.d
        flat = buf.numpy().reshape(-1)
        slab = (flat[0::2] + 1j * flat[1::2]).reshape(self.n_planes, x_hi - x_lo, Mt)
        spec = np.zeros((x_hi - x_lo, Mt, M), dtype=np.complex128)
        for i, n in enumerate(order):
            spec[:, :, n] = slab[i]
            if 0 < n < M - n:
                spec[:, :, M - n] = np.conj(slab[i])
        Ht = np.zeros((Mt, Mt, M))
        Ht[x_lo:x_hi] = np.fft.ifft(spec, axis=2).real
        # gather over the slab rows only (reading R-1 constant)
        x, alpha = self_.x, 2.0 * self.xi ** 2 / d["eta"]
        pref = (2.0 * self.xi ** 2 / (math.pi * d["eta"])) ** 1.5
        C = 4.0 * math.pi * d["h"] ** 3 * pref
        t = np.arange(self.P)
        h = d["h"]
        phi = np.zeros(N)
        for m in range(N):
            jx = int(math.floor(x[m, 0] / h)) + 1 + t
            jy = int(math.floor(x[m, 1] / h)) + 1 + t
            lz = int(math.floor(x[m, 2] / h - self.P / 2.0)) + 1 + t
            wx = np.exp(-alpha * ((jx - self.P / 2.0) * h - x[m, 0]) ** 2) * ((jx >= x_lo) & (jx < x_hi))
            wy = np.exp(-alpha * ((jy - self.P / 2.0) * h - x[m, 1]) ** 2)
            wz = np.exp(-alpha * (lz * h - x[m, 2]) ** 2)
            blk = Ht[np.ix_(jx, jy, lz % M)]
            phi[m] = C * np.einsum("i,j,k,ijk->", wx, wy, wz, blk)
        return torch.from_numpy(phi)


def _stages(x):
    c = CASE
    s = NumpyStages(c["L"], c["xi"], c["M"], c["P"], c["n_l"], c["S0"], c["SI"], c["SJ"])
    s.x = x
    return s


def _info(s):
    return {"Mt": s.Mt, "n_planes": s.n_planes, "n_kernel_planes": s.n_l + 1, "LK": 2 * s.Mt, "Ntilde": s.SJ,
            "P": s.P}


def _reference():
    c = CASE
    x, q = make_system(c["N"], c["L"], c["seed"])
    return x, q, sd.se1p_kspace(x, q, c["L"], c["xi"], c["M"], c["P"], c["n_l"], c["S0"], c["SI"], c["SJ"])


def test_slab_bounds_and_lpt():
    assert sdist.slab_bounds(152, 1) == [0, 152]
    b = sdist.slab_bounds(152, 4)                  # 10 tiles -> 3, 3, 2, 2
    assert b == [0, 48, 96, 128, 152]
    b = sdist.slab_bounds(40, 4)                   # 3 tiles over 4 ranks: one empty slab
    assert b[0] == 0 and b[-1] == 40 and all(v % 16 == 0 or v == 40 for v in b)
    assert all(b2 >= b1 for b1, b2 in zip(b, b[1:]))
    # tile-work-weighted split (boundary tiles are light): C5's 18 tiles over 8 ranks
    w = sdist.tile_weights(280, 24)
    assert len(w) == 18 and w[2] == 16 * 24 and w[0] < w[2] and w[17] < w[16] < w[2]
    assert sum(w) == 256 * 24                      # every (particle column, stencil row) once
    b = sdist.slab_bounds(280, 8, 24)
    loads = [sum(w[b[i] // 16:(b[i + 1] + 15) // 16]) for i in range(8)]
    assert b[0] == 0 and b[-1] == 280 and all(v % 16 == 0 for v in b[:-1])
    assert max(loads) <= 2.25 * 16 * 24 < max(sum(w[c // 16:(d + 15) // 16]) for c, d in
                                               zip(sdist.slab_bounds(280, 8), sdist.slab_bounds(280, 8)[1:]))
    assert sdist.slab_bounds(152, 1, 24) == [0, 152]
    costs = [10.0, 9.0, 1.0, 1.0, 1.0, 1.0, 1.0]
    owned = sdist.assign_planes(costs, 2)
    assert sorted(sum(owned, [])) == list(range(7))
    assert owned == [[0, 3, 5], [1, 2, 4, 6]]       # LPT: 10 | 9, then ones to the lighter rank (ties: rank 0)
    info = {"Mt": 152, "n_planes": 65, "n_kernel_planes": 5, "LK": 304, "Ntilde": 224}
    plan = sdist.make_plan(info, 8)
    assert sorted(plan.order) == list(range(65))
    loads = [sum(sdist.plane_costs(info)[n] for n in o) for o in plan.owned]
    assert max(loads) / min(loads) < 1.3
    for r in range(8):   # all-to-all split sizes are consistent between sender and receiver
        for s_ in range(8):
            assert plan.splits_to_owners(s_)[r] == plan.splits_from_slabs(r)[s_]


@pytest.mark.parametrize("R", [2, 3])
def test_emulated_ranks_match_alg1(R):
    x, q, ref = _reference()
    st = _stages(x)
    plan = sdist.make_plan(_info(st), R)
    phi = sdist.kspace_emulated(torch.from_numpy(x), torch.from_numpy(q), plan, st).numpy()
    assert np.max(np.abs(phi - ref)) <= 1e-12 * np.max(np.abs(ref))


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, q, ref = _reference()
        st = _stages(x)
        plan = sdist.make_plan(_info(st), world)
        phi = sdist.kspace_rank(torch.from_numpy(x), torch.from_numpy(q), plan, st, rank).numpy()
        np.save(f"{result_path}.{rank}.npy", phi)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_spmd_matches_alg1(world, tmp_path):
    x, q, ref = _reference()
    out = str(tmp_path / "phi")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        phi = np.load(f"{out}.{r}.npy")
        assert np.max(np.abs(phi - ref)) <= 1e-12 * np.max(np.abs(ref)), r


# ---------------------------------------------------------------- particle-split baseline
def _parts(N, R):
    b = [N * r // R for r in range(R + 1)]
    return [(b[r], b[r + 1]) for r in range(R)]


@pytest.mark.parametrize("R", [2, 3])
def test_emulated_particle_split_matches_alg1(R):
    """kspace_rank_rs for all ranks in turn: each rank grids and gathers only its particles over
    the whole grid, the planes are summed at their owners (reduce-scatter), transformed, and
    gathered back; the concatenated phi equals the single-process Alg. 1 oracle."""
    x, q, ref = _reference()
    st = _stages(x)
    plan = sdist.make_plan(_info(st), R)
    phi = sdist.kspace_emulated_rs(torch.from_numpy(x), torch.from_numpy(q), plan, st, _parts(len(q), R)).numpy()
    assert np.max(np.abs(phi - ref)) <= 1e-12 * np.max(np.abs(ref))


def _worker_rs(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, q, ref = _reference()
        a, b = _parts(len(q), world)[rank]
        st = _stages(x)
        plan = sdist.make_plan(_info(st), world)
        phi = sdist.kspace_rank_rs(torch.from_numpy(x[a:b]), torch.from_numpy(q[a:b]), plan, st, rank).numpy()
        np.save(f"{result_path}.{rank}.npy", phi)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_particle_split_matches_alg1(world, tmp_path):
    """The particle-split SPMD body over gloo: every rank's phi equals the oracle on its particles."""
    x, q, ref = _reference()
    out = str(tmp_path / "phi")
    mp.spawn(_worker_rs, args=(world, _free_port(), out), nprocs=world, join=True)
    for r, (a, b) in enumerate(_parts(len(q), world)):
        phi = np.load(f"{out}.{r}.npy")
        assert phi.shape == (b - a,)
        assert np.max(np.abs(phi - ref[a:b])) <= 1e-12 * np.max(np.abs(ref)), r
