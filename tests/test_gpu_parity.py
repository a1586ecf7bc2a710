"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances:
  * element-wise vs the step-by-step Alg. 1 oracle (same discretisation): |d| <= 1e-11 max|phi|.
    Both evaluate the same discrete sums in fp64; the GPU applies the upsampled planes as an
    exact aperiodic convolution and sums in another order, so they differ by rounding only
    (~ eps * log2(FFT size) * dynamic range of the spectra).
  * full potential vs the exact Ewald1P oracle: relative rms <= 1e-9 (BASELINE north_star).
  * real space vs the oracle's direct sum: |d| <= 1e-12 max|phi|.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import se1p_discrete as sd
from se1p_synth import CONFIGS, kspace_kwargs, make_system

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1611_09538_b200 as se1p  # noqa: E402


def _dev(x, q):
    return (torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())


def _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ, **kw):
    xd, qd = _dev(x, q)
    return se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=S0, SI=SI, Ntilde=SJ, **kw).cpu().numpy()


CASES = [
    # name, N, L, xi, M, P, n_l, S0, SI, SJ, seed
    ("C1", 100, (1, 1, 1), 4.0, 16, 16, 2, 110, 64, 32, 1),
    ("C1-wide", 100, (1, 1, 1), 4.0, 16, 16, 2, 256, 256, 40, 1),
    ("C2", 2000, (1, 1, 1), 8.0, 32, 20, 3, 416, 416, 64, 2),
    ("tiny-odd", 37, (1, 1, 1), 3.0, 8, 6, 1, 40, 36, 15, 5),
    ("ragged-tiles", 333, (1, 1, 1), 5.0, 20, 10, 3, 90, 75, 35, 6),
    ("longz", 150, (1, 1, 2), 4.0, 24, 8, 4, 60, 72, 21, 7),
    ("plain-upsampled", 80, (1, 1, 1), 4.0, 12, 8, 6, 60, 60, 60, 8),
    ("prime-extent", 60, (1, 1, 1), 4.0, 12, 8, 2, 53, 47, 23, 9),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_kspace_matches_alg1_oracle(case):
    name, N, L, xi, M, P, n_l, S0, SI, SJ, seed = case
    x, q = make_system(N, L, seed)
    ref = sd.se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    got = _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    err = np.max(np.abs(got - ref))
    assert err <= 1e-11 * np.max(np.abs(ref)), (name, err, np.max(np.abs(ref)))


def test_kspace_single_particle_and_pair():
    """Degenerate cases: N = 2 coaxial pair (rho = 0 in the zero mode) and a lone particle
    (non-neutral -> refused unless checks are skipped; then it is still well defined)."""
    L = (1.0, 1.0, 1.0)
    x = np.array([[0.45, 0.55, 0.1], [0.45, 0.55, 0.4]])
    q = np.array([1.0, -1.0])
    ref = sd.se1p_kspace(x, q, L, 5.0, 16, 12, 8, 112, 112, 56)
    got = _gpu_kspace(x, q, L, 5.0, 16, 12, 8, 112, 112, 56)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))
    x1, q1 = x[:1], np.array([1.0])
    with pytest.raises(se1p.SE1PError) as ei:
        _gpu_kspace(x1, q1, L, 5.0, 16, 12, 2, 112, 84, 28)
    assert ei.value.code == 3
    ref1 = sd.se1p_kspace(x1, q1, L, 5.0, 16, 12, 2, 112, 84, 28)
    got1 = _gpu_kspace(x1, q1, L, 5.0, 16, 12, 2, 112, 84, 28, skip_checks=True)
    assert abs(got1[0] - ref1[0]) <= 1e-11 * abs(ref1[0])


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_full_potential_vs_exact_oracle(cfg):
    c = CONFIGS[cfg]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = _dev(x, q)
    phi = (se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kspace_kwargs(c))
           + se1p.real(xd, qd, c.L, c.xi, c.rc)).cpu().numpy()
    ref = oracle.phi_exact(x, q, c.L)
    assert oracle.rel_rms(phi, ref) <= 1e-9


@pytest.mark.parametrize("L", [(1.0, 0.625, 1.0), (0.5, 1.0, 1.0)])
def test_rectangular_cross_section(L):
    """L1 != L2 runs on the square embedding [0, max(L1,L2))^2 (reading R-19): element-wise equal
    to Alg. 1 on the square box for the same particles, and the full potential matches the exact
    sum, which does not depend on L1, L2 (Eq. (2))."""
    x, q = make_system(120, L, 21)
    Lsq = (1.0, 1.0, 1.0)
    ref = sd.se1p_kspace(x, q, Lsq, 4.0, 16, 16, 2, 110, 64, 32)
    got = _gpu_kspace(x, q, L, 4.0, 16, 16, 2, 110, 64, 32)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))
    xd, qd = _dev(x, q)
    phi = (se1p.kspace(xd, qd, L, 4.0, 16, 16, n_local=2, S0=110, SI=64, Ntilde=32)
           + se1p.real(xd, qd, L, 4.0, 1.158)).cpu().numpy()
    assert oracle.rel_rms(phi, oracle.phi_exact(x, q, L)) <= 1e-9
    assert np.max(np.abs(oracle.phi_exact(x, q, L) - oracle.phi_exact(x, q, Lsq))) <= 1e-12 * np.max(np.abs(phi))
    # a particle outside the user's box (inside the square) is still refused
    xb = x.copy()
    xb[5, 0 if L[0] < L[1] else 1] = 0.9
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(torch.from_numpy(xb).cuda(), qd, L, 4.0, 16, 16)
    assert e.value.code == 2
    # SE3P keeps the square requirement (its cross-section is periodic)
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace3p(xd, qd, L, 4.0, 16, 8)
    assert e.value.code == 4


def test_real_space_vs_oracle():
    for L, xi, rc, N, seed in [((1, 1, 1), 4.0, 1.158, 100, 1), ((1, 1, 1), 8.0, 0.594, 500, 2),
                               ((1, 1, 2), 12.0, 0.401, 800, 3), ((2, 2, 2), 30.0, 0.1, 3000, 5),
                               ((1, 1, 1), 3.0, 2.7, 40, 4),
                               # xi rc = 9, 13.5: high table degrees; 144: beyond the warp kernel's shared
                               # table (thread-per-target fallback)
                               ((1, 1, 1), 10.0, 0.9, 300, 7), ((1, 1, 1), 15.0, 0.9, 300, 6),
                               ((1, 1, 1), 160.0, 0.9, 300, 8)]:
        x, q = make_system(N, L, seed)
        xd, qd = _dev(x, q)
        got = se1p.real(xd, qd, L, xi, rc).cpu().numpy()
        ref = oracle.phi_real(x, q, L, xi, rc) + oracle.phi_self(q, xi)
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), (L, xi, rc)


def test_real_space_edge_cases():
    """k_real_warp's target groups and candidate ranges on awkward layouts, against the direct sum
    (Eq. (3) + Eq. (6)): one particle, a pair inside / outside rc, every particle in one column,
    a dense cluster (heavy groups next to near-empty columns), rc below the cell size with most
    particles alone, a rectangular box with z images, and particles on the box faces."""
    rng = np.random.default_rng(11)
    cases = []
    cases.append(((1, 1, 1), 6.0, 0.3, np.array([[0.5, 0.5, 0.5]]), np.array([0.7])))
    cases.append(((1, 1, 1), 6.0, 0.3, np.array([[0.1, 0.1, 0.1], [0.2, 0.15, 0.95]]), np.array([1.0, -1.0])))
    cases.append(((1, 1, 1), 6.0, 0.3, np.array([[0.1, 0.1, 0.1], [0.9, 0.9, 0.5]]), np.array([1.0, -1.0])))
    n = 600   # one column
    x = np.column_stack([0.5 + 1e-3 * rng.random(n), 0.5 + 1e-3 * rng.random(n), rng.random(n)])
    cases.append(((1, 1, 1), 10.0, 0.25, x, rng.uniform(-1, 1, n)))
    n = 3000   # a dense cluster plus a uniform background
    x = np.concatenate([0.3 + 0.02 * rng.random((n // 2, 3)), rng.random((n - n // 2, 3))])
    cases.append(((1, 1, 1), 12.0, 0.2, x, rng.uniform(-1, 1, n)))
    n = 2000   # rc far below the cell size
    cases.append(((1, 1, 1), 300.0, 0.01, rng.random((n, 3)), rng.uniform(-1, 1, n)))
    n = 1500   # rectangular, z images (rc > L3 / 2)
    L = (1.0, 2.0, 0.5)
    cases.append((L, 8.0, 0.3, rng.random((n, 3)) * np.array(L), rng.uniform(-1, 1, n)))
    n = 800   # on the faces: x = 0, y = 0, z = 0 and z just below L3
    x = rng.random((n, 3))
    x[: n // 4, 0] = 0.0
    x[n // 4: n // 2, 1] = 0.0
    x[n // 2: 3 * n // 4, 2] = 0.0
    x[3 * n // 4:, 2] = np.nextafter(1.0, 0.0)
    cases.append(((1, 1, 1), 8.0, 0.4, x, rng.uniform(-1, 1, n)))
    for L, xi, rc, x, q in cases:
        q = q - (q.mean() if q.size > 1 else 0.0)
        x = np.ascontiguousarray(x, dtype=np.float64)
        xd, qd = _dev(x, q)
        got = se1p.real(xd, qd, L, xi, rc, skip_checks=True).cpu().numpy()
        ref = oracle.phi_real(x, q, L, xi, rc) + oracle.phi_self(q, xi)
        assert np.max(np.abs(got - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300), (L, xi, rc, x.shape)
        _, fg = se1p.real(xd, qd, L, xi, rc, skip_checks=True, field=True)
        fr = oracle.field_real(x, q, L, xi, rc)
        assert np.max(np.abs(fg.cpu().numpy() - fr)) <= 1e-12 * max(np.max(np.abs(fr)), 1e-300), (L, xi, rc)


def test_real_space_random_configurations():
    """Seeded random real-space configurations -- box shape (rectangular, long or short periodic
    axis), density, xi rc from 1 to 12 (table degrees 7 .. 15), rc from a fraction of a cell to
    beyond L3 (several z images), uniform or half-clustered positions -- potential and field
    against the direct sum (Eq. (3) + Eq. (6)) at 1e-12 of the largest value."""
    rng = np.random.default_rng(2024)
    for case in range(30):
        L = tuple(float(v) for v in rng.choice([0.5, 1.0, 1.5, 2.0], size=3))
        N = int(rng.integers(2, 2500))
        rc = float(rng.uniform(0.05, 1.2) * min(L))
        xi = float(rng.uniform(1.0, 12.0) / rc)
        x = rng.random((N, 3)) * np.array(L)
        if case % 3 == 0:   # half of the particles in a small cluster
            k = N // 2
            x[:k] = np.array(L) * (0.2 + 0.1 * rng.random((k, 3)))
        q = rng.uniform(-1, 1, N)
        q -= q.mean()
        xd, qd = _dev(x, q)
        got, fg = se1p.real(xd, qd, L, xi, rc, skip_checks=True, field=True)
        ref = oracle.phi_real(x, q, L, xi, rc) + oracle.phi_self(q, xi)
        fr = oracle.field_real(x, q, L, xi, rc)
        assert np.max(np.abs(got.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref)), (case, L, N, xi, rc)
        assert np.max(np.abs(fg.cpu().numpy() - fr)) <= 1e-12 * max(np.max(np.abs(fr)), 1e-300), (case, L, N, xi, rc)


def test_bitwise_determinism_and_host_io():
    c = CONFIGS["C2"]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = _dev(x, q)
    kw = dict(n_local=3, S0=416, SI=416, Ntilde=64)
    a = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw).cpu().numpy()
    b = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw).cpu().numpy()
    h = se1p.kspace(x, q, c.L, c.xi, c.M, c.P, **kw)          # numpy in -> host I/O path
    assert np.array_equal(a, b)
    assert np.array_equal(a, h)
    r1 = se1p.real(xd, qd, c.L, c.xi, c.rc).cpu().numpy()
    r2 = se1p.real(x, q, c.L, c.xi, c.rc)
    assert np.array_equal(r1, r2)


def test_invariances():
    """z-translation by one grid step is exact on the grid; permuting particles permutes phi;
    phi is linear in q."""
    L, xi, M, P = (1.0, 1.0, 1.0), 6.0, 24, 14
    x, q = make_system(300, L, 11)
    kw = dict(n_local=3, S0=300, SI=300, Ntilde=48)
    base = _gpu_kspace(x, q, L, xi, M, P, **{"n_l": 3, "S0": 300, "SI": 300, "SJ": 48})
    xs = x.copy()
    xs[:, 2] = (xs[:, 2] + 1.0 / M) % 1.0
    shifted = _gpu_kspace(xs, q, L, xi, M, P, 3, 300, 300, 48)
    assert np.max(np.abs(shifted - base)) <= 1e-12 * np.max(np.abs(base))
    p = np.random.default_rng(0).permutation(300)
    perm = _gpu_kspace(x[p], q[p], L, xi, M, P, 3, 300, 300, 48)
    assert np.max(np.abs(perm - base[p])) <= 1e-12 * np.max(np.abs(base))
    neg = _gpu_kspace(x, -2.5 * q, L, xi, M, P, 3, 300, 300, 48)
    assert np.max(np.abs(neg + 2.5 * base)) <= 1e-12 * np.max(np.abs(base))
    del kw


def test_errors():
    L = (1.0, 1.0, 1.0)
    x, q = make_system(50, L, 12)
    xd, qd = _dev(x, q)
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(xd, qd + 0.1, L, 4.0, 16, 8)
    assert e.value.code == 3
    xb = x.copy()
    xb[3, 0] = 1.2
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(torch.from_numpy(xb).cuda(), qd, L, 4.0, 16, 8)
    assert e.value.code == 2
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(xd, qd, (1.0, 1.0, 1.0), 4.0, 15, 8)      # odd M
    assert e.value.code == 4
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(xd, qd, (1.0, 1.3, 1.0), 4.0, 16, 8)      # L2/h not an integer
    assert e.value.code == 4
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(xd, qd, L, 4.0, 16, 8, n_local=20)
    assert e.value.code == 4
    # z outside [0, L3) is folded, not an error
    xz = x.copy()
    xz[:, 2] += 3.0
    a = se1p.kspace(torch.from_numpy(xz).cuda(), qd, L, 4.0, 16, 8, n_local=2, S0=96, SI=72, Ntilde=24).cpu().numpy()
    b = se1p.kspace(xd, qd, L, 4.0, 16, 8, n_local=2, S0=96, SI=72, Ntilde=24).cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_plan_info_defaults():
    info = se1p.plan_info((1.0, 1.0, 1.0), 4.0, 16, 16, s0=2 + math.sqrt(2), sf=2.0, n_local=2)
    assert info["Mt"] == 32 and info["S0"] == 110 and info["SI"] == 64
    assert info["LK"] >= 2 * 32 - 1 and info["n_kernel_planes"] == 3 and info["n_planes"] == 9
    assert abs(info["eta"] - 16 * 16.0 / 256 / (0.95 ** 2 * math.pi)) < 1e-15


EDGE = [
    # name, N, L, xi, M, P, n_l, S0, SI, SJ, seed
    ("odd-P7", 90, (1, 1, 1), 4.0, 16, 7, 2, 64, 48, 24, 21),
    ("odd-P9-M18", 70, (1, 1, 1), 4.0, 18, 9, 3, 70, 56, 28, 22),
    ("P32-M48", 120, (1, 1, 1), 6.0, 48, 32, 4, 200, 160, 80, 23),
    ("P40-M64", 60, (1, 1, 1), 7.0, 64, 40, 3, 260, 208, 104, 24),
    ("P64-max", 40, (1, 1, 1), 9.0, 64, 64, 2, 260, 260, 128, 25),
    ("M4-P2", 30, (1, 1, 1), 1.5, 4, 2, 1, 12, 12, 6, 26),
    ("P-equals-M", 50, (1, 1, 1), 3.0, 8, 8, 2, 40, 32, 16, 27),
    ("flat-box-L3-0.5", 80, (1, 1, 0.5), 8.0, 16, 10, 2, 200, 160, 52, 28),
]


@pytest.mark.parametrize("case", EDGE, ids=[c[0] for c in EDGE])
def test_kspace_odd_and_large_stencils(case):
    """Odd P (reading R-3 covers both parities) and stencils wider than a 32-node z tile and
    than the 16-column tiles (several tiles per axis, periodic wrap of the stencil)."""
    name, N, L, xi, M, P, n_l, S0, SI, SJ, seed = case
    x, q = make_system(N, L, seed)
    ref = sd.se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    got = _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref)), (name, np.max(np.abs(got - ref)))


def test_kspace_degenerate_positions():
    """Particles exactly on grid nodes, on the faces x = 0, y = 0, z = 0, just below L3, and
    coincident pairs (same (x, y): rho = 0 in the zero mode; same point up to z images)."""
    L, xi, M, P, n_l, S0, SI, SJ = (1.0, 1.0, 1.0), 4.0, 16, 10, 3, 80, 64, 26
    h = 1.0 / M
    x = np.array([[0.0, 0.0, 0.0], [5 * h, 7 * h, 3 * h], [0.5, 0.5, np.nextafter(1.0, 0.0)],
                  [0.25, 0.75, 0.5], [0.25, 0.75, 0.9], [np.nextafter(1.0, 0.0), 0.3, 0.2],
                  [0.6, np.nextafter(1.0, 0.0), 0.0], [0.6, 0.1, 0.45]])
    q = np.array([1.0, -0.5, 0.25, -1.0, 0.75, 0.5, -0.25, -0.75])
    q -= q.mean()
    ref = sd.se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    got = _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_empty_and_tiny_inputs_rejected_or_exact():
    L = (1.0, 1.0, 1.0)
    xd = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    qd = torch.zeros(0, dtype=torch.float64, device="cuda")
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace(xd, qd, L, 4.0, 16, 8)
    assert e.value.code == 1
    with pytest.raises(se1p.SE1PError) as e:
        se1p.real(xd, qd, L, 4.0, 0.5)
    assert e.value.code == 1


def test_ragged_tiles_all_configs_of_tz():
    """Grids whose extents are not multiples of the tile sizes: M~ = M_free + P not a multiple of
    16 and M not a multiple of the 32-node z tile (M >= 64 uses TZ = 32)."""
    for (N, M, P, SJ, seed) in [(200, 72, 13, 90, 31), (150, 66, 10, 80, 32)]:
        L = (1.0, 1.0, 1.0)
        x, q = make_system(N, L, seed)
        xi = 0.25 * M / 1.0 * 0.5
        ref = sd.se1p_kspace(x, q, L, xi, M, P, 3, 2 * (M + P), 2 * (M + P), SJ)
        got = _gpu_kspace(x, q, L, xi, M, P, 3, 2 * (M + P), 2 * (M + P), SJ)
        assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref)), (M, P)


def test_graph_mode_replays_bitwise():
    """CUDA-graph mode (captured on the first call, replayed after): same bits as the eager path,
    including after the inputs change in place (the graph reads the same buffers)."""
    c = CONFIGS["C2"]
    kw = kspace_kwargs(c)
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = _dev(x, q)
    out = torch.empty(c.N, dtype=torch.float64, device="cuda")
    eager = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
    g1 = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, graph=True, out=out, **kw).clone()
    assert torch.equal(g1, eager)
    x2, q2 = make_system(c.N, c.L, c.seed + 100)
    xd.copy_(torch.from_numpy(x2))
    qd.copy_(torch.from_numpy(q2))
    g2 = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, graph=True, out=out, **kw).clone()
    assert se1p.launch_count() > 5      # the captured kernels (replayed as one graph)
    assert torch.equal(g2, se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw))
    fo = torch.empty(c.N, 3, dtype=torch.float64, device="cuda")
    _, e1 = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, graph=True, out=out, field=True, field_out=fo, **kw)
    _, e2 = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, field=True, **kw)
    assert torch.equal(e1, e2)
    with pytest.raises(se1p.SE1PError):
        se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, graph=True, profile=True, **kw)
    # release frees workspace, plans and graphs; the next graph call re-captures
    se1p.release()
    g3 = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, graph=True, out=out, **kw).clone()
    assert torch.equal(g3, se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw))


def test_multi_tier_matches_oracle():
    """Per-mode extents (se1p_kspace_tiers_ex) element-wise against the Alg. 1 oracle's tiers."""
    L, xi, M, P, n_l = (1.0, 1.0, 1.0), 6.0, 24, 16, 4
    Mt = M + P
    x, q = make_system(300, L, 42)
    tiers = [170, 120, 97, 53]
    ref = sd.se1p_kspace(x, q, L, xi, M, P, n_l, 4 * Mt, tiers, 2 * Mt)
    xd, qd = _dev(x, q)
    got = se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=4 * Mt, Ntilde=2 * Mt, S_modes=tiers).cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))
    flat = se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=4 * Mt, SI=97, Ntilde=2 * Mt).cpu().numpy()
    same = se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=4 * Mt, Ntilde=2 * Mt, S_modes=[97] * n_l).cpu().numpy()
    assert np.array_equal(flat, same)
    with pytest.raises(se1p.SE1PError):
        se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=4 * Mt, Ntilde=2 * Mt, S_modes=[Mt - 1] * n_l)


def _random_config(rng):
    """A seeded random valid configuration (tools/fuzz_parity.py's generator), or None."""
    M = int(rng.choice([8, 10, 12, 14, 16, 20, 24, 30, 32, 36, 40, 48]))
    P = int(rng.integers(2, min(M, 28) + 1))
    L3 = float(rng.choice([0.5, 1.0, 1.5, 2.0]))
    m1 = int(rng.choice([M // 2, M, (3 * M) // 2])) if M % 2 == 0 else M
    h = L3 / M
    m2 = int(rng.integers(max(1, m1 // 2), m1 + 1)) if rng.random() < 0.3 else m1   # rectangular (R-19)
    Lsq = (m1 * h, m1 * h, L3)
    L = (m1 * h, m2 * h, L3) if rng.random() < 0.5 else (m2 * h, m1 * h, L3)
    xi = float(rng.uniform(2.0, 9.0)) / max(L)
    eta = P * xi ** 2 * h ** 2 / (0.95 ** 2 * math.pi)
    if not (0.05 < eta < 0.95):
        return None
    Mt = m1 + P
    n_l = int(rng.integers(0, M // 2 + 1))
    S0 = int(Mt * rng.uniform(2.5, 4.0))
    SI = int(Mt * rng.uniform(1.0, 3.0)) if n_l else Mt
    SJ = int(rng.integers(Mt, 2 * Mt))
    while not all(f in (2, 3, 5, 7) for f in _factors(SJ)):
        SJ += 1
    if not all(f in (2, 3, 5, 7) for f in _factors(M)):
        return None
    N = int(rng.integers(2, 400))
    return M, P, L, Lsq, xi, n_l, S0, SI, SJ, N, int(rng.integers(1, 10 ** 6))


def test_random_configurations_match_oracle():
    """40 seeded random valid configurations (M, P, box aspect incl. rectangular cross-sections
    against the square-embedding oracle, reading R-19, xi, n_l, extents, N): element-wise parity
    with the Alg. 1 oracle; every 4th also the field, and the SE3P path where it applies."""
    rng = np.random.default_rng(2024)
    checked = 0
    while checked < 40:
        c = _random_config(rng)
        if c is None:
            continue
        M, P, L, Lsq, xi, n_l, S0, SI, SJ, N, seed = c
        x, q = make_system(N, L, seed)
        ref = sd.se1p_kspace(x, q, Lsq, xi, M, P, n_l, S0, SI, SJ)
        got = _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
        err = np.max(np.abs(got - ref))
        assert err <= 1e-11 * np.max(np.abs(ref)), (M, P, L, xi, n_l, S0, SI, SJ, N, err)
        if checked % 4 == 0:
            _, Eref = sd.se1p_kspace(x, q, Lsq, xi, M, P, n_l, S0, SI, SJ, return_field=True)
            xd, qd = _dev(x, q)
            _, E = se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=S0, SI=SI, Ntilde=SJ, field=True)
            assert np.max(np.abs(E.cpu().numpy() - Eref)) <= 1e-11 * np.max(np.abs(Eref)), ("field", c)
            if P % 2 == 0 and L[0] == L[1] == L[2]:
                from oracle import se3p_discrete as s3
                r3 = s3.se3p_kspace(x, q, L, xi, M, P)
                g3 = se1p.kspace3p(xd, qd, L, xi, M, P).cpu().numpy()
                assert np.max(np.abs(g3 - r3)) <= 1e-11 * np.max(np.abs(r3)), ("3p", c)
        checked += 1


@pytest.mark.parametrize("M,P,N,L3", [(64, 24, 20000, 1.0), (96, 23, 30000, 2.0)])
def test_large_sweeps_match_oracle(M, P, N, L3):
    """Sizes where the sweep kernels run many batches per group (BM-sized pieces, carried k-step
    entries), several periodic-axis chunks per column tile (overhang added to the next chunk) and
    many work items per CTA: element-wise parity with the Alg. 1 oracle."""
    L = (L3 * 64 / M, L3 * 64 / M, L3) if M != 64 else (1.0, 1.0, 1.0)
    h = L[2] / M
    Mt = int(round(L[0] / h)) + P
    xi = 12.0 / L[0]
    x, q = make_system(N, L, 77 + M)
    n_l, S0, SI, SJ = 4, 4 * Mt, 3 * Mt, Mt + (Mt % 2)
    while not all(f in (2, 3, 5, 7) for f in _factors(SJ)):
        SJ += 1
    ref = sd.se1p_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    got = _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))


def _factors(n):
    f, d = [], 2
    while d * d <= n:
        while n % d == 0:
            f.append(d)
            n //= d
        d += 1
    return f + ([n] if n > 1 else [])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_plans_and_workspaces_are_per_device():
    """The same parameters on cuda:0 and cuda:1 (plans keyed on the device): each
    device's result equals the other's bitwise, and releasing one device leaves the other's plan
    usable."""
    c = CONFIGS["C2"]
    x, q = make_system(c.N, c.L, c.seed)
    kw = kspace_kwargs(c)
    outs = []
    for d in (0, 1):
        with torch.cuda.device(d):
            xd = torch.from_numpy(x).to(f"cuda:{d}")
            qd = torch.from_numpy(q).to(f"cuda:{d}")
            outs.append(se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw).cpu())
    assert torch.equal(outs[0], outs[1])
    with torch.cuda.device(0):
        se1p.release()
    with torch.cuda.device(1):
        xd, qd = torch.from_numpy(x).to("cuda:1"), torch.from_numpy(q).to("cuda:1")
        assert torch.equal(se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw).cpu(), outs[1])


def test_stream_ordered_calls_on_two_streams():
    """Asynchronous calls on two streams share the device's workspace: each call's stream waits
    for the previous call's work, so interleaved k-space and real-space calls on
    different streams return the results of the same calls made synchronously."""
    c = CONFIGS["C3"]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = kspace_kwargs(c)
    ref_k = se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, **kw)
    ref_r = se1p.real(xd, qd, c.L, c.xi, c.rc)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for i in range(3):
        st = s1 if i % 2 == 0 else s2
        outs.append(("k", se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, stream=st, sync=False, skip_checks=True, **kw)))
        st2 = s2 if i % 2 == 0 else s1
        outs.append(("r", se1p.real(xd, qd, c.L, c.xi, c.rc, stream=st2, sync=False, skip_checks=True)))
    torch.cuda.synchronize()
    for kind, o in outs:
        assert torch.equal(o, ref_k if kind == "k" else ref_r), kind
