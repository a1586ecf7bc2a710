"""The real-space kernel's erfc table (se1p_real_table, host only -- runs without a GPU): its
polynomials reproduce erfc(xi r) (scipy) within the stated 2e-16 absolute bound on a fine grid of
every interval, at the configs' xi rc and across the supported range, and the degrees DESIGN.md
quotes.  The table is product code (the CUDA path), checked here against an independent erfc."""
import numpy as np
import pytest
from scipy.special import erfc

import paper_1611_09538_b200 as se1p


def _max_err(xi, rc):
    deg, K, c = se1p.real_table(xi, rc)
    assert deg > 0 and c.shape == (deg + 1, K)
    w = rc / K
    worst = 0.0
    for i in range(K):
        r = np.linspace(i * w, (i + 1) * w, 257)
        u = r - (i + 0.5) * w
        p = np.zeros_like(u)
        for n in range(deg, -1, -1):
            p = p * u + c[n, i]
        worst = max(worst, float(np.max(np.abs(p - erfc(xi * r)))))
    return deg, worst


@pytest.mark.parametrize("xi,rc,deg", [(30.0, 0.1, 8), (30.0, 0.164, 9), (20.0, 0.247, 9), (4.0, 1.158, 9),
                                       (8.0, 0.594, 9), (12.0, 0.401, 9)])
def test_table_at_the_configs(xi, rc, deg):
    d, err = _max_err(xi, rc)
    assert d == deg
    assert err <= 4e-16   # 2e-16 by construction (long double) + double evaluation and scipy's rounding


@pytest.mark.parametrize("X", [0.5, 1.0, 2.0, 6.0, 13.5, 45.0, 100.0])
def test_table_across_xi_rc(X):
    _, err = _max_err(X / 0.3, 0.3)
    assert err <= 4e-16


def test_fallback_and_errors():
    deg, K, c = se1p.real_table(160.0, 0.9)   # xi rc = 144: beyond degree 31
    assert deg == 0 and c.size == 0
    with pytest.raises(se1p.SE1PError) as e:
        se1p.real_table(-1.0, 0.1)
    assert e.value.code == 1
