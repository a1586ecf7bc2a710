"""Pins for the oracle's special functions (App. A) against values and
routines independent of this repo: mpmath (arbitrary precision), scipy.special, closed forms."""
import csv
import itertools
import math
import os

import mpmath as mp
import numpy as np
import pytest
from scipy import special

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "special_values.csv")


def _golden():
    with open(GOLD) as f:
        rows = [r for r in csv.reader(line for line in f if not line.startswith("#"))]
    return [(n, float(a), (float(b) if b else None), float(v)) for n, a, b, v in rows]


@pytest.mark.parametrize("row", _golden())
def test_golden_values(row):
    name, a, b, v = row
    got = {"E1": lambda: oracle.e1(a), "erfc": lambda: math.erfc(a), "k0": lambda: oracle.k0(a),
           "K0inc": lambda: oracle.K0inc(a, b)}[name]()
    # App. A reports ~1e-15 absolute for K0; relative 5e-15 elsewhere
    assert abs(got - v) <= max(5e-15 * abs(v), 2e-18 if name == "K0inc" else 0.0)


def test_e1_against_scipy_range():
    """E1: series below the switch, continued fraction above."""
    for x in np.concatenate([np.logspace(-8, 2.7, 200), [0.9, 1.0, 1.1, 1.49, 1.5, 1.51, 2.0]]):
        ref = special.exp1(x)
        assert abs(oracle.e1(x) - ref) <= 2e-15 * ref, x


def test_g_limit_and_series():
    """gamma + log x + E1(x) -> 0 as x -> 0 (Eq. (limit)) and its series."""
    assert oracle.g(0.0) == 0.0
    mp.mp.dps = 50
    for u in np.concatenate([np.logspace(-12, 1.5, 80), [1.0, 1.5, 2.0]]):
        ref = float(mp.euler + mp.log(u) + mp.e1(u))
        assert abs(oracle.g(u) - ref) <= 2e-15 * abs(ref), u
    # leading term of the series: g(u) = u - u^2/4 + ...
    assert abs(oracle.g(1e-10) - (1e-10 - 0.25e-20)) < 1e-25


def test_k0_against_scipy():
    for v in np.logspace(-6, 2.5, 120):
        ref = special.k0(v)
        assert abs(oracle.k0(v) - ref) <= 3e-15 * ref, v


def test_incomplete_k0_definition_grid():
    """K0(a,b) = int_0^1 e^{-a/t-bt} dt/t against mpmath quadrature over a log grid."""
    mp.mp.dps = 30
    for a, b in itertools.product(np.logspace(-3, 2, 7), np.logspace(-4, 2, 7)):
        ref = float(mp.quad(lambda t: mp.exp(-a / t - b * t) / t,
                            [0, 1e-5, 1e-4, 1e-3, 0.01, 0.05, 0.1, 0.25, 0.5, 1]))
        got = oracle.K0inc(a, b)
        assert abs(got - ref) <= max(1e-14 * ref, 2e-15), (a, b, got, ref)


def test_incomplete_k0_identities():
    """K0(a,0) = E1(a) and K0(a,b) = 2 k0(2 sqrt(ab)) - K0(b,a)."""
    for a in [1e-3, 0.1, 1.0, 9.87, 40.0]:
        assert abs(oracle.K0inc(a, 0.0) - special.exp1(a)) <= 4e-15 * special.exp1(a)
    for a, b in itertools.product([0.5, 1.0, 5.0, 0.03], [0.5, 1.0, 5.0, 7.0]):
        lhs = oracle.K0inc(a, b)
        rhs = 2.0 * special.k0(2.0 * math.sqrt(a * b)) - oracle.K0inc(b, a)
        assert abs(lhs - rhs) <= 1e-14 * max(1.0, abs(lhs)), (a, b)


def test_gauss_legendre_exactness():
    xs, ws = oracle.gauss_legendre()
    n = xs.size
    assert abs(ws.sum() - 2.0) < 1e-14
    for deg in range(0, 2 * n, 7):
        exact = 0.0 if deg % 2 else 2.0 / (deg + 1)
        assert abs(np.dot(ws, xs ** deg) - exact) < 1e-13, deg
