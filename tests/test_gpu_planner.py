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


def test_potential_and_forces_from_tol():
    """potential(..., tol=) and energy_forces(..., tol=) pick the planner's parameters."""
    L, xi, tol = (1.0, 1.0, 1.0), 8.0, 1e-8
    x, q = make_system(3000, L, 18)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    phi = se1p.potential(xd, qd, L, xi, tol=tol).cpu().numpy()
    t = sample_targets(3000, 128, 18)
    ref = oracle.phi_exact(x, q, L, t)
    assert math.sqrt(np.mean((phi[t] - ref) ** 2)) <= tol
    U, phi2, F = se1p.energy_forces(xd, qd, L, xi, tol=tol)
    assert torch.max(torch.abs(phi2.cpu() - torch.from_numpy(phi))) <= 1e-12 * np.max(np.abs(phi))
    Eref = oracle.field_exact(x, q, L, t)
    err = math.sqrt(np.mean(((F.cpu().numpy()[t] / q[t, None]) - Eref) ** 2))
    assert err <= 100 * tol      # the field's error constant is larger
