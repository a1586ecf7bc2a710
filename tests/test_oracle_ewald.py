"""Pins for the exact Ewald1P oracle (Eqs. (1)-(6)) against the definition
(brute-force image sums), a textbook closed form, the xi-independence of the total,
symmetries, and the Kolafa-Perram real-space estimate."""
import math

import numpy as np
import pytest
from scipy import special

import oracle
from se1p_synth import make_system


def coaxial_pair_closed_form(dz, L3):
    """q1=+1 and q2=-1 on the same (x,y) line, separated by dz along the periodic axis.
    From Eq. (1) with P_1 and the series of the digamma function:
      phi(x1) = -1/|dz| + (psi(1+t) + psi(1-t) + 2 gamma)/L3,  t = |dz|/L3."""
    t = abs(dz) / L3
    return -1.0 / abs(dz) + (special.digamma(1 + t) + special.digamma(1 - t) + 2 * np.euler_gamma) / L3


@pytest.mark.parametrize("dz,L3", [(0.3, 1.0), (0.05, 1.0), (0.91, 1.0), (0.7, 2.0), (1.9, 2.0)])
def test_coaxial_pair_closed_form(dz, L3):
    L = np.array([1.0, 1.0, L3])
    x = np.array([[0.4, 0.6, 0.02], [0.4, 0.6, 0.02 + dz]])
    q = np.array([1.0, -1.0])
    ref = coaxial_pair_closed_form(dz, L3)
    got = oracle.phi_exact(x, q, L, [0])[0]
    assert abs(got - ref) <= 1e-13 * abs(ref)
    # the other particle sees the mirror value with the opposite sign
    assert abs(oracle.phi_exact(x, q, L, [1])[0] + ref) <= 1e-13 * abs(ref)


@pytest.mark.parametrize("N,L,seed", [(2, (1, 1, 1), 3), (6, (1, 1, 1), 4), (10, (1.0, 1.0, 2.0), 5),
                                      (8, (2.0, 2.0, 2.0), 6)])
def test_brute_force_images(N, L, seed):
    """The definition: symmetric image sum |alpha| <= A with Richardson extrapolation in A."""
    x, q = make_system(N, L, seed)
    ex = oracle.phi_exact(x, q, L)
    br = oracle.phi_brute_extrapolated(x, q, L, A=4000)
    assert np.max(np.abs(ex - br)) <= 2e-11 * np.max(np.abs(ex))


def test_xi_invariance():
    """xi 'does not alter the total result'.  Every term changes with xi; the sum not."""
    x, q = make_system(40, (1.0, 1.0, 1.0), 8)
    L = (1.0, 1.0, 1.0)
    base, comps = oracle.phi_exact(x, q, L, components=True)
    for xi in [0.3, 1.3, 2.9, 5.0]:
        other, c2 = oracle.phi_exact(x, q, L, xi_o=xi, components=True)
        assert np.max(np.abs(other - base)) <= 1e-13 * np.max(np.abs(base))
        assert np.max(np.abs(c2 - comps)) > 1e-3          # the split itself did move


def test_components_sum_and_self():
    x, q = make_system(12, (1.0, 1.0, 1.0), 9)
    L = (1.0, 1.0, 1.0)
    xi = 2.0
    tot, comps = oracle.phi_exact(x, q, L, xi_o=xi, components=True)
    assert np.allclose(comps.sum(axis=1), tot, rtol=1e-15, atol=1e-14)
    assert np.allclose(comps[:, 3], -2 * xi * q / math.sqrt(math.pi), rtol=1e-15)   # Eq. (6)
    assert np.allclose(comps[:, 1], oracle.phi_k3nz(x, q, L, xi), rtol=1e-14)
    assert np.allclose(comps[:, 2], oracle.phi_k30(x, q, L, xi), rtol=1e-14)


def test_symmetries():
    L = (1.0, 1.0, 1.0)
    x, q = make_system(16, L, 10)
    base = oracle.phi_exact(x, q, L)
    # rigid shift along the periodic axis (folded back into the box)
    xs = x.copy()
    xs[:, 2] = (xs[:, 2] + 0.37) % 1.0
    assert np.max(np.abs(oracle.phi_exact(xs, q, L) - base)) <= 1e-13 * np.max(np.abs(base))
    # rigid shift in the free plane (no images there, only relative positions matter)
    xs = x.copy()
    xs[:, :2] *= 0.5
    xs2 = xs.copy()
    xs2[:, :2] += 0.25
    assert np.max(np.abs(oracle.phi_exact(xs2, q, L) - oracle.phi_exact(xs, q, L))) <= 1e-13 * np.max(np.abs(base))
    # linearity in q
    assert np.allclose(oracle.phi_exact(x, -2.0 * q, L), -2.0 * base, rtol=1e-14, atol=1e-13)
    # permutation
    p = np.random.default_rng(0).permutation(16)
    assert np.allclose(oracle.phi_exact(x[p], q[p], L), base[p], rtol=1e-14, atol=1e-13)


def test_kolafa_perram_real_space():
    """fig:kolafa_perram: N=100 random particles, L=2, xi=7; measured rms error of the
    truncated real-space sum tracks Eq. (trunc_error_estimate_real) within a factor 5."""
    L = (2.0, 2.0, 2.0)
    x, q = make_system(100, L, 21)
    Q = float(np.sum(q * q))
    xi = 7.0
    conv = oracle.phi_real(x, q, L, xi, None)
    for rc in [0.3, 0.4, 0.5, 0.6]:
        trunc = oracle.phi_real(x, q, L, xi, rc)
        meas = math.sqrt(np.mean((trunc - conv) ** 2))
        est = math.sqrt(Q * rc / (2 * 2.0 ** 3)) * (xi * rc) ** -2 * math.exp(-(xi * rc) ** 2)
        assert est / 5 <= meas <= est * 5, (rc, meas, est)
