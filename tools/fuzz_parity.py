"""Seeded random-configuration parity fuzz (80 cases, 30 % rectangular cross-sections against the
square-embedding oracle, reading R-19): python tools/fuzz_parity.py SEED [all]"""
import sys, math
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from oracle import se1p_discrete as sd
from se1p_synth import make_system
import paper_1611_09538_b200 as se1p
from test_gpu_parity import _gpu_kspace, _factors
def test_random_configurations_match_oracle():
    """Seeded random valid configurations (M, P, box aspect, xi, n_l, extents, N): element-wise
    parity with the Alg. 1 oracle -- catches index/tiling assumptions the named cases miss."""
    import sys
    rng = np.random.default_rng(int(sys.argv[1]))
    checked = 0
    while checked < 80:
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
            continue
        Mt = m1 + P
        n_l = int(rng.integers(0, M // 2 + 1))
        S0 = int(Mt * rng.uniform(2.5, 4.0))
        SI = int(Mt * rng.uniform(1.0, 3.0)) if n_l else Mt
        SJ = int(rng.integers(Mt, 2 * Mt))
        while not all(f in (2, 3, 5, 7) for f in _factors(SJ)):
            SJ += 1
        if not all(f in (2, 3, 5, 7) for f in _factors(M)):
            continue
        N = int(rng.integers(2, 400))
        x, q = make_system(N, L, int(rng.integers(1, 10 ** 6)))
        ref = sd.se1p_kspace(x, q, Lsq, xi, M, P, n_l, S0, SI, SJ)   # the square embedding
        got = _gpu_kspace(x, q, L, xi, M, P, n_l, S0, SI, SJ)
        err = np.max(np.abs(got - ref))
        assert err <= 1e-11 * np.max(np.abs(ref)), (M, P, L, xi, n_l, S0, SI, SJ, N, err)
        if len(sys.argv) > 2 and sys.argv[2] == "all":
            _, Eref = sd.se1p_kspace(x, q, Lsq, xi, M, P, n_l, S0, SI, SJ, return_field=True)
            xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
            _, E = se1p.kspace(xd, qd, L, xi, M, P, n_local=n_l, S0=S0, SI=SI, Ntilde=SJ, field=True)
            errE = np.max(np.abs(E.cpu().numpy() - Eref))
            assert errE <= 1e-11 * np.max(np.abs(Eref)), ("field", M, P, L, errE)
            if P % 2 == 0 and L[0] == L[2] and L[1] == L[0]:
                from oracle import se3p_discrete as s3
                r3 = s3.se3p_kspace(x, q, L, xi, M, P)
                g3 = se1p.kspace3p(xd, qd, L, xi, M, P).cpu().numpy()
                assert np.max(np.abs(g3 - r3)) <= 1e-11 * np.max(np.abs(r3)), ("3p", M, P, L)
        checked += 1



test_random_configurations_match_oracle()
print("fuzz ok")
