"""Pins for the oracle's electric field E = -grad phi (force on particle m: q_m E(x_m); the
paper's force formulas P:535-551 written as gradients of Eqs. (3)-(5)).  NEXT-1 of SURVEY 8(f).

Pinned against things other than the oracle's own formulas: mpmath quadrature of the derivative
of the incomplete Bessel function's definition, finite differences of the (separately
pinned) potential, the brute-force image sum of Coulomb fields, a coaxial-pair closed form from
the digamma series, and xi-invariance."""
import math

import mpmath as mp
import numpy as np
import pytest
from scipy import special

import oracle
from se1p_synth import make_system


@pytest.mark.parametrize("a,b", [(0.05, 0.01), (0.3, 2.0), (1.0, 1.0), (2.5, 0.2), (0.01, 5.0), (10.0, 30.0),
                                 (40.0, 0.5)])
def test_dK0db_definition(a, b):
    """dK0(a,b)/db = -int_1^inf e^{-at - b/t} dt/t^2, by mpmath quadrature of P:95 differentiated."""
    mp.mp.dps = 30
    ref = -mp.quad(lambda t: mp.exp(-a * t - b / t) / t ** 2, [1, 2, 10, mp.inf])
    got = oracle.dK0db(a, b)
    assert abs(got - float(ref)) <= 1e-13 * abs(float(ref)) + 1e-300


def test_dK0db_is_derivative_of_K0():
    """Central difference (Richardson) of the pinned K0(a,b) in b."""
    for a, b in [(0.2, 0.7), (1.5, 0.3), (0.05, 3.0)]:
        def fd(h):
            return (oracle.K0inc(a, b + h) - oracle.K0inc(a, b - h)) / (2 * h)
        est = (4 * fd(1e-4) - fd(2e-4)) / 3
        assert abs(est - oracle.dK0db(a, b)) <= 1e-9 * abs(est)


def coaxial_field(dz, L3):
    """E_z at particle 1 (+1) from particle 2 (-1) at dz above on the same axis, all z images:
    from phi_1 = -1/dz + (psi(1+t) + psi(1-t) + 2 gamma)/L3, t = dz/L3 (Eq. (1) with P_1),
    E_z = -d phi_1/d z_1 = (1/t^2 + psi'(1+t) - psi'(1-t)) / L3^2."""
    t = dz / L3
    return (1.0 / t ** 2 + special.polygamma(1, 1 + t) - special.polygamma(1, 1 - t)) / L3 ** 2


@pytest.mark.parametrize("dz,L3", [(0.3, 1.0), (0.05, 1.0), (0.91, 1.0), (0.7, 2.0)])
def test_coaxial_pair_field(dz, L3):
    L = np.array([1.0, 1.0, L3])
    x = np.array([[0.4, 0.6, 0.02], [0.4, 0.6, 0.02 + dz]])
    q = np.array([1.0, -1.0])
    e = oracle.field_exact(x, q, L, [0])[0]
    ref = coaxial_field(dz, L3)
    assert abs(e[2] - ref) <= 1e-12 * abs(ref)
    assert abs(e[0]) <= 1e-14 * abs(ref) and abs(e[1]) <= 1e-14 * abs(ref)


@pytest.mark.parametrize("N,L,seed", [(2, (1, 1, 1), 3), (6, (1, 1, 1), 4), (10, (1.0, 1.0, 2.0), 5)])
def test_field_brute_force_images(N, L, seed):
    x, q = make_system(N, L, seed)
    ex = oracle.field_exact(x, q, L)
    br = oracle.field_brute_extrapolated(x, q, L, A=4000)
    assert np.max(np.abs(ex - br)) <= 1e-10 * np.max(np.abs(ex))


def test_field_is_minus_gradient_of_potential():
    """4th-order central differences of phi_m under displacement of particle m (its own images
    move with it and contribute no force)."""
    L = (1.0, 1.0, 1.0)
    x, q = make_system(8, L, 6)
    m = 3
    e = oracle.field_exact(x, q, L, [m])[0]
    for c in range(3):
        def phi_at(d):
            xs = x.copy()
            xs[m, c] += d
            return oracle.phi_exact(xs, q, L, [m])[0]
        h = 1e-3
        d1 = (phi_at(h) - phi_at(-h)) / (2 * h)
        d2 = (phi_at(2 * h) - phi_at(-2 * h)) / (4 * h)
        grad = (4 * d1 - d2) / 3
        assert abs(-grad - e[c]) <= 1e-8 * np.max(np.abs(e)), (c, -grad, e[c])


def test_field_xi_invariance_and_components():
    L = (1.0, 1.0, 1.0)
    x, q = make_system(30, L, 7)
    base = oracle.field_exact(x, q, L)
    for xi in [0.4, 1.7, 3.0]:
        other = oracle.field_exact(x, q, L, xi_o=xi)
        assert np.max(np.abs(other - base)) <= 1e-11 * np.max(np.abs(base))
    # the zero mode has no z component; the k-space part equals total minus real space
    xi = 2.0
    k30 = oracle.field_k30(x, q, L, xi)
    assert np.all(k30[:, 2] == 0.0)
    tot = oracle.field_real(x, q, L, xi, None) + oracle.field_k3nz(x, q, L, xi) + k30
    assert np.max(np.abs(tot - base)) <= 1e-11 * np.max(np.abs(base))
