"""GPU tests of the mode-sharded distributed path's CUDA stages (include/se1p.h distributed
entries, paper_1611_09538_b200/dist.py).  Only one GPU is available, so R ranks are emulated in
one process (kspace_emulated: the stages of every rank run in turn, the transposes are local
copies with the production split sizes -- no kernel waits on another rank), and the real SPMD
body runs over NCCL with world size 1.  The result must equal the single-GPU path."""
import os
import socket

import numpy as np
import pytest

from oracle import se1p_discrete as sd
from se1p_synth import CONFIGS, kspace_kwargs, make_system

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1611_09538_b200 as se1p  # noqa: E402
from paper_1611_09538_b200 import dist as sdist  # noqa: E402


def _run(cfgname, R, N=None):
    c = CONFIGS[cfgname]
    N = N or c.N
    x, q = make_system(N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = kspace_kwargs(c)
    ref = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
    info = se1p.plan_info(c.L, c.xi, c.M, c.P, **kw)
    plan = sdist.make_plan(info, R)
    phi = sdist.kspace_emulated(xd, qd, plan, sdist.CudaBackend(c.L, c.xi, c.M, c.P, **kw))
    torch.cuda.synchronize()
    return ref.cpu().numpy(), phi.cpu().numpy(), x, q


@pytest.mark.parametrize("cfg,R", [("C2", 2), ("C2", 3), ("C3", 4), ("C4", 2), ("C4", 8)])
def test_emulated_ranks_match_single_gpu(cfg, R):
    ref, phi, _, _ = _run(cfg, R)
    assert np.max(np.abs(phi - ref)) <= 1e-13 * np.max(np.abs(ref)), (cfg, R)


def test_emulated_ranks_match_alg1_oracle():
    """Small case against the step-by-step Alg. 1 oracle directly (R = 3, one empty slab)."""
    L, xi, M, P, n_l, S0, SI, SJ = (1.0, 1.0, 1.0), 4.0, 16, 8, 2, 72, 60, 30
    x, q = make_system(60, L, 5)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = dict(n_local=n_l, S0=S0, SI=SI, Ntilde=SJ)
    plan = sdist.make_plan(se1p.plan_info(L, xi, M, P, **kw), 3)
    phi = sdist.kspace_emulated(xd, qd, plan, sdist.CudaBackend(L, xi, M, P, **kw)).cpu().numpy()
    ref = sd.se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    assert np.max(np.abs(phi - ref)) <= 1e-11 * np.max(np.abs(ref))


@pytest.mark.parametrize("cfg,R", [("C2", 2), ("C3", 3), ("C4", 4)])
def test_emulated_particle_split_matches_single_gpu(cfg, R):
    """The particle-split baseline (dist.kspace_rank_rs): every rank grids and
    gathers only its particles over the whole grid; the planes are summed at their owners,
    transformed there and gathered back.  Emulated ranks in turn equal the single-GPU result."""
    c = CONFIGS[cfg]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = kspace_kwargs(c)
    ref = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw).cpu().numpy()
    plan = sdist.make_plan(se1p.plan_info(c.L, c.xi, c.M, c.P, **kw), R)
    b = [c.N * r // R for r in range(R + 1)]
    parts = [(b[r], b[r + 1]) for r in range(R)]
    phi = sdist.kspace_emulated_rs(xd, qd, plan, sdist.CudaBackend(c.L, c.xi, c.M, c.P, **kw), parts)
    got = phi.cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref)), (cfg, R)


def test_backward_requires_matching_forward():
    c = CONFIGS["C2"]
    kw = kspace_kwargs(c)
    buf = torch.zeros((c.M // 2 + 1, 16, 52 + 12, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(se1p.SE1PError):
        se1p.slab_backward(buf, 12345, c.L, c.xi, c.M, c.P, 0, 16, list(range(c.M // 2 + 1)), **kw)


@pytest.mark.parametrize("cfg,R", [("C3", 2), ("C3", 3), ("C4", 8), ("C1", 8)])
def test_real_space_parts_sum_to_the_whole(cfg, R):
    """The real-space sum split over R emulated ranks (se1p.real part=(r, R), as dist.real runs
    it): every part writes only its targets (the rest 0) and the parts sum bitwise to the
    single-GPU call, potential and field (C1: 100 particles, fewer target groups than parts)."""
    c = CONFIGS[cfg]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    ref, eref = se1p.real(xd, qd, c.L, c.xi, c.rc, field=True)
    acc, eacc = torch.zeros_like(ref), torch.zeros_like(eref)
    nonzero = torch.zeros(c.N, dtype=torch.int32, device="cuda")
    for r in range(R):
        p, e = se1p.real(xd, qd, c.L, c.xi, c.rc, field=True, part=(r, R))
        nonzero += (p != 0).int()
        acc += p
        eacc += e
    assert torch.equal(acc, ref) and torch.equal(eacc, eref)
    assert int(nonzero.max()) == 1   # each target written by exactly one part


def test_real_space_parts_fallback_kernel_and_errors():
    """The split on the thread-per-target fallback (xi rc beyond the shared table) and the
    argument checks of opts->reserved[4..5]."""
    L, xi, rc = (1.0, 1.0, 1.0), 160.0, 0.9
    x, q = make_system(300, L, 8)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    ref = se1p.real(xd, qd, L, xi, rc)
    acc = sum(se1p.real(xd, qd, L, xi, rc, part=(r, 3)) for r in range(3))
    assert torch.equal(acc, ref)
    for bad in [(3, 3), (-1, 2), (0, -2)]:
        with pytest.raises(se1p.SE1PError) as e:
            se1p.real(xd, qd, L, 8.0, 0.3, part=bad)
        assert e.value.code == 1


def test_nccl_world_one():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        c = CONFIGS["C3"]
        x, q = make_system(c.N, c.L, c.seed)
        xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
        kw = kspace_kwargs(c)
        phi = sdist.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
        ref = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
        assert torch.equal(phi, ref)
        pr, er = sdist.real(xd, qd, c.L, c.xi, c.rc, field=True)   # the shared real-space sum
        rr, re = se1p.real(xd, qd, c.L, c.xi, c.rc, field=True)
        assert torch.equal(pr, rr) and torch.equal(er, re)
    finally:
        dist.destroy_process_group()


def test_nccl_world_one_particle_split():
    """dist.kspace_rs over NCCL with world size 1 equals the single-GPU result."""
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        c = CONFIGS["C3"]
        x, q = make_system(c.N, c.L, c.seed)
        xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
        kw = kspace_kwargs(c)
        phi = sdist.kspace_rs(xd, qd, c.L, c.xi, c.M, c.P, **kw)
        ref = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
        assert np.max(np.abs((phi - ref).cpu().numpy())) <= 1e-13 * float(ref.abs().max())
    finally:
        dist.destroy_process_group()


def _nccl_worker(rank, world, port, cfgname, out):
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    c = CONFIGS[cfgname]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    phi = sdist.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kspace_kwargs(c))
    pr = sdist.real(xd, qd, c.L, c.xi, c.rc)
    torch.cuda.synchronize()
    if rank == 0:
        np.save(out, phi.cpu().numpy())
        np.save(out + ".real.npy", pr.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="the NCCL path needs two GPUs")
def test_nccl_two_ranks_match_single_gpu(tmp_path):
    """dist.kspace over NCCL with world = 2 (one process per GPU) equals the single-GPU result."""
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "phi.npy")
    mp.spawn(_nccl_worker, args=(2, port, "C3", out), nprocs=2, join=True)
    c = CONFIGS["C3"]
    x, q = make_system(c.N, c.L, c.seed)
    ref = se1p.kspace(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda(), c.L, c.xi, c.M, c.P,
                      **kspace_kwargs(c)).cpu().numpy()
    got = np.load(out)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    rr = se1p.real(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda(), c.L, c.xi, c.rc).cpu().numpy()
    assert np.array_equal(np.load(out + ".real.npy"), rr)   # dist.real: bitwise
