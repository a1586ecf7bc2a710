"""The tolerance planner (NEXT-2) driving the CUDA path: planned parameters meet the tolerance
(absolute rms) against the exact Ewald1P potential on seeded targets."""
import math

import numpy as np
import pytest

import oracle
from se1p_synth import make_system, sample_targets

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1611_09538_b200 as se1p  # noqa: E402


@pytest.mark.parametrize("L,N,xi,tol", [((1.0, 1.0, 1.0), 20000, 10.0, 1e-9), ((1.0, 1.0, 2.0), 5000, 6.0, 1e-6),
                                        ((2.0, 2.0, 2.0), 50000, 12.0, 1e-11)])
def test_planned_gpu_potential_meets_tol(L, N, xi, tol):
    x, q = make_system(N, L, 17)
    p = se1p.plan_from_tol(L, float(np.sum(q * q)), xi, tol)
    M, P, kw = se1p.kspace_args(p)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    phi = (se1p.kspace(xd, qd, L, xi, M, P, **kw) + se1p.real(xd, qd, L, xi, p["rc"])).cpu().numpy()
    t = sample_targets(N, 256, 17)
    ref = oracle.phi_exact(x, q, L, t)
    err = math.sqrt(np.mean((phi[t] - ref) ** 2))
    print(f"planned M={M} P={P} rc={p['rc']:.3f}: abs rms {err:.2e} (tol {tol:.0e})")
    assert err <= tol
