"""GPU parity of the SE3P baseline through the C ABI: element-wise against
the step-by-step SE3P oracle (same discrete sums, tolerance 1e-11 max|phi| as for SE1P) and
against the exact triply periodic k-space sum."""
import math

import numpy as np
import pytest

import oracle
from oracle import se3p_discrete as s3
from se1p_synth import make_system

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1611_09538_b200 as se1p  # noqa: E402

CASES = [
    # name, N, L, xi, M, P, seed
    ("cube", 500, (1.0, 1.0, 1.0), 6.0, 24, 16, 1),
    ("ragged", 333, (1.0, 1.0, 1.0), 5.0, 20, 10, 2),
    ("longz", 400, (1.0, 1.0, 2.0), 5.0, 40, 12, 3),
    ("tiny", 37, (1.0, 1.0, 1.0), 3.0, 8, 6, 4),
    ("tiles", 3000, (1.0, 1.0, 1.0), 10.0, 48, 20, 5),
]


def _dev(x, q):
    return torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_se3p_matches_oracle(case):
    name, N, L, xi, M, P, seed = case
    x, q = make_system(N, L, seed)
    ref = s3.se3p_kspace(x, q, L, xi, M, P)
    got = se1p.kspace3p(*_dev(x, q), L, xi, M, P).cpu().numpy()
    err = np.max(np.abs(got - ref))
    assert err <= 1e-11 * np.max(np.abs(ref)), (name, err)


def test_se3p_vs_exact_and_host_io():
    L, xi = (1.0, 1.0, 1.0), 8.0
    x, q = make_system(2000, L, 6)
    xd, qd = _dev(x, q)
    got = se1p.kspace3p(xd, qd, L, xi, 40, 24).cpu().numpy()
    t = np.arange(0, 2000, 7)
    ref = oracle.phi3_kspace(x, q, L, xi, targets=t)
    assert oracle.rel_rms(got[t], ref) <= 1e-12
    assert np.array_equal(got, se1p.kspace3p(x, q, L, xi, 40, 24))     # numpy -> host I/O, bitwise
    # total 3P potential with the oracle's real space: Madelung-pinned exact sum
    tot = got[t] + oracle.phi3_real(x, q, L, xi, targets=t) - 2 * xi * q[t] / math.sqrt(math.pi)
    assert oracle.rel_rms(tot, oracle.phi3_exact(x, q, L, targets=t)) <= 1e-12


def test_se3p_errors():
    L = (1.0, 1.0, 1.0)
    x, q = make_system(50, L, 7)
    xd, qd = _dev(x, q)
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace3p(xd, qd, L, 4.0, 16, 7)
    assert e.value.code == 4
    with pytest.raises(se1p.SE1PError) as e:
        se1p.kspace3p(xd, qd + 0.1, L, 4.0, 16, 8)
    assert e.value.code == 3
