"""Parameters from a tolerance: se1p_plan_from_tol, host-only, no GPU.

Pinned against the paper's estimates written out here from the paper (Eqs. (trunc_error_estimate_
real/fourier); Eq. (approximation_error_oneterm)), scipy's Lambert W, and --
what a planner is for -- the measured error: the planned parameters run through the Alg. 1
oracle and the real-space oracle meet the tolerance against the exact Ewald1P sum."""
import math

import numpy as np
import pytest
from scipy.special import lambertw

import oracle
from oracle import se1p_discrete as sd
from se1p_synth import make_system

import paper_1611_09538_b200 as se1p

C = 0.95


def est_real(rc, xi, Q, V):
    return math.sqrt(Q * rc / (2 * V)) * (xi * rc) ** -2 * math.exp(-(xi * rc) ** 2)


def est_fourier(kinf, xi, Q, L):
    return xi / math.pi ** 2 * kinf ** -1.5 * math.sqrt(Q) * math.exp(-(math.pi * kinf / (xi * L)) ** 2)


PLANS = [((10.0, 10.0, 10.0), 1.0, 1.5, 1e-6), ((10.0, 10.0, 10.0), 1.0, 3.0, 1e-12),
         ((1.0, 1.0, 1.0), 100.0, 6.0, 1e-8), ((1.0, 1.0, 2.0), 100.0, 5.0, 1e-10), ((2.0, 2.0, 2.0), 7e5, 30.0, 1e-9)]


@pytest.mark.parametrize("L,Q,xi,tol", PLANS)
def test_plan_inverts_the_estimates(L, Q, xi, tol):
    p = se1p.plan_from_tol(L, Q, xi, tol)
    V, L3 = L[0] * L[1] * L[2], L[2]
    # Eq. (rc) and Eq. (kinf) are the inverses of the two truncation estimates (budget R-18)
    assert est_real(p["rc"], xi, Q, V) == pytest.approx(0.5 * tol, rel=1e-9)
    assert est_fourier(p["kinf"], xi, Q, L3) == pytest.approx(0.1 * tol, rel=1e-9)
    # and they match the closed forms with scipy's Lambert W
    Cr = Q / (2 * V * xi * (0.5 * tol) ** 2)
    assert p["rc"] == pytest.approx(math.sqrt(3 * lambertw(4 / 3 * Cr ** (2 / 3)).real) / (2 * xi), rel=1e-12)
    # P: the smallest even support meeting the window budget
    A = math.sqrt(Q * xi * L3) / L3
    assert p["P"] % 2 == 0 and A * math.exp(-C * C * math.pi * p["P"] / 2) <= 0.01 * tol
    assert A * math.exp(-C * C * math.pi * (p["P"] - 2) / 2) > 0.01 * tol or p["P"] == 2
    # M: even, resolves kinf, integer free-axis counts, eta <= 0.8 (Eq. (comp_eta))
    M, h = p["M"], L3 / p["M"]
    assert M % 2 == 0 and M >= 2 * p["kinf"]
    assert p["Mfree"] == round(L[0] / h) and abs(L[0] / h - p["Mfree"]) < 1e-9 * p["Mfree"]
    assert p["eta"] == pytest.approx(p["P"] * xi ** 2 * h ** 2 / (C * C * math.pi), rel=1e-14)
    assert p["eta"] <= 0.8
    # upsampling: e^{-2 pi s_l} < tol/10, n_l ~ M/10, s0 >= 1 + sqrt(2)
    assert math.exp(-2 * math.pi * p["s_l"]) <= 0.1 * tol * (1 + 1e-12)
    assert p["n_local"] == max(1, math.ceil(M / 10))
    assert p["SI"] >= p["s_l"] * p["Mt"] - 1e-9 and p["S0"] >= (1 + math.sqrt(2)) * p["Mt"] - 1e-9
    assert p["Ntilde"] >= p["Mt"] and p["Mt"] == p["Mfree"] + p["P"]
    # image distance of the padded transforms (reading R-18): sqrt(Q) e^{-k3 (S h - L_free)} <= tol/10
    # at the slowest mode of each set (k3 = 2 pi/L3 for I, 2 pi (n_l+1)/L3 for J)
    for S, k3 in [(p["SI"], 2 * math.pi / L3), (p["Ntilde"], 2 * math.pi * (p["n_local"] + 1) / L3)]:
        assert math.sqrt(Q) * math.exp(-k3 * (S * h - L[0])) <= 0.1 * tol * (1 + 1e-9)


def test_lambert_region_and_errors():
    p = se1p.plan_from_tol((1, 1, 1), 1.0, 4.0, 0.5)      # loose tolerance: small arguments of W
    assert p["P"] >= 2 and p["M"] >= 2
    for args in [((1, 1, 1), 0.0, 4.0, 1e-6), ((1, 1, 1), 1.0, -1.0, 1e-6), ((1, 1, 1), 1.0, 4.0, 0.0),
                 ((1, 1, 1), 1.0, 4.0, 1.5), ((0, 1, 1), 1.0, 4.0, 1e-6)]:
        with pytest.raises(se1p.SE1PError) as e:
            se1p.plan_from_tol(*args)
        assert e.value.code == 1
    # rectangular cross-section: planned on the square [0, max(L1, L2))^2 (reading R-19)
    r = se1p.plan_from_tol((1.0, 2.0, 1.0), 1.0, 4.0, 1e-6)
    s = se1p.plan_from_tol((2.0, 2.0, 1.0), 1.0, 4.0, 1e-6)
    assert r["Mfree"] == round(2.0 / r["h"]) and r["Mt"] == r["Mfree"] + r["P"]
    assert (r["M"], r["P"], r["Mfree"], r["Ntilde"]) == (s["M"], s["P"], s["Mfree"], s["Ntilde"])


# (L, N, normalise Q to 1, xi, tol): the paper's Table 1 systems and unit boxes
ACHIEVE = [((10.0, 10.0, 10.0), 120, True, 1.5, 1e-6), ((10.0, 10.0, 10.0), 120, True, 3.0, 1e-6),
           ((10.0, 10.0, 10.0), 120, True, 1.5, 1e-12), ((10.0, 10.0, 10.0), 120, True, 3.0, 1e-12),
           ((1.0, 1.0, 1.0), 300, False, 6.0, 1e-8), ((1.0, 1.0, 2.0), 300, False, 5.0, 1e-10),
           ((1.0, 1.0, 1.0), 300, False, 8.0, 1e-4), ((1.0, 1.0, 1.0), 300, False, 12.0, 1e-10),
           ((1.0, 1.0, 2.0), 500, False, 6.0, 1e-6)]


@pytest.mark.parametrize("L,N,norm,xi,tol", ACHIEVE)
def test_planned_parameters_meet_the_tolerance(L, N, norm, xi, tol):
    """The point of the planner: absolute rms error of the k-space part (Alg. 1
    oracle, the same discrete sums as the CUDA path) and of the truncated real space, each
    against the exact sums, below tol."""
    x, q = make_system(N, L, 7)
    if norm:
        q = q / math.sqrt(np.sum(q * q))
    p = se1p.plan_from_tol(L, float(np.sum(q * q)), xi, tol)
    phi = sd.se1p_kspace(x, q, L, xi, p["M"], p["P"], p["n_local"], p["S0"], p["SI"], p["Ntilde"], eta=p["eta"])
    ref = oracle.phi_kspace_reference(x, q, L, xi)
    err_k = math.sqrt(np.mean((phi - ref) ** 2))
    err_r = math.sqrt(np.mean((oracle.phi_real(x, q, L, xi, p["rc"]) - oracle.phi_real(x, q, L, xi, None)) ** 2))
    assert err_k <= tol, (err_k, p)
    assert err_r <= tol, (err_r, p)
