"""Pins for the triply periodic oracle (the SE3P baseline of the paper's
Ex. 5): the Ewald 3P sum (oracle/ewald3p.c) against textbook Madelung constants and
xi-invariance; the step-by-step SE3P oracle (oracle/se3p_discrete.py) against the exact 3P
k-space sum, converging like Theorem 1's window error."""
import math

import numpy as np
import pytest

import oracle
from oracle import se3p_discrete as s3
from se1p_synth import make_system

# Madelung constants referred to the nearest-neighbour distance (textbook values)
NACL = 1.747564594633182190636212
CSCL = 1.762674773070988023555


@pytest.mark.parametrize("shift", [0.0, 0.1, 0.37])
def test_nacl_madelung(shift):
    """Rock salt in a unit conventional cell (r0 = 1/2): phi = -+ M/r0 at the ions."""
    na = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]])
    cl = np.array([[.5, 0, 0], [0, .5, 0], [0, 0, .5], [.5, .5, .5]])
    x = (np.vstack([na, cl]) + shift) % 1.0
    q = np.array([1.0] * 4 + [-1.0] * 4)
    phi = oracle.phi3_exact(x, q, (1.0, 1.0, 1.0))
    assert np.max(np.abs(phi - (-q) * NACL / 0.5)) <= 1e-13


def test_cscl_madelung_and_box_scaling():
    """CsCl (r0 = sqrt(3)/2 a), in a cube of side 2: phi scales as 1/a."""
    x = np.array([[0.3, 0.1, 0.2], [1.3, 1.1, 1.2]])
    q = np.array([1.0, -1.0])
    phi = oracle.phi3_exact(x, q, (2.0, 2.0, 2.0))
    assert phi == pytest.approx([-CSCL / math.sqrt(3.0), CSCL / math.sqrt(3.0)], rel=1e-13)


def test_xi_invariance_and_split():
    L = (1.0, 1.0, 1.5)
    x, q = make_system(40, L, 9)
    base = oracle.phi3_exact(x, q, L)
    for xi in [2.0, 4.5, 7.0]:
        assert np.max(np.abs(oracle.phi3_exact(x, q, L, xi_o=xi) - base)) <= 1e-12 * np.max(np.abs(base))
    xi = 5.0
    parts = oracle.phi3_real(x, q, L, xi) + oracle.phi3_kspace(x, q, L, xi) - 2 * xi * q / math.sqrt(math.pi)
    assert np.max(np.abs(parts - base)) <= 1e-12 * np.max(np.abs(base))


def test_se3p_discrete_converges_to_the_exact_kspace_sum():
    """Window/trapezoid error decays like e^{-c^2 pi P/2} (Thm 1) to rounding."""
    L = (1.0, 1.0, 1.0)
    x, q = make_system(60, L, 3)
    xi = 6.0
    ref = oracle.phi3_kspace(x, q, L, xi)
    errs = []
    for M, P in [(24, 8), (24, 12), (24, 16), (32, 24)]:
        phi = s3.se3p_kspace(x, q, L, xi, M, P)
        errs.append(math.sqrt(np.mean((phi - ref) ** 2) / np.mean(ref ** 2)))
    assert all(b < a / 100 for a, b in zip(errs[:3], errs[1:3]))
    assert errs[-1] < 1e-13
    # non-cubic box with integer L_d/h
    L2 = (1.0, 1.0, 2.0)
    x2, q2 = make_system(40, L2, 4)
    ref2 = oracle.phi3_kspace(x2, q2, L2, 5.0)
    phi2 = s3.se3p_kspace(x2, q2, L2, 5.0, 48, 24)
    assert math.sqrt(np.mean((phi2 - ref2) ** 2) / np.mean(ref2 ** 2)) < 1e-12
