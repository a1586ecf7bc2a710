"""GPU parity at BASELINE.json's full sizes (C3, C4, C5), in the launch configuration bench.py
times (same kwargs, same stream path), against the exact Ewald1P potential (oracle/, Eqs. (2)-(6),
P:80-92) on the oracle evaluation sets of SURVEY.md 8(c) step 7: C3 1024 seeded targets + 128
within 2w of a free face (computed here), C4 2048 + 256 and C5 512 + 256 (precomputed by
tests/golden/make_fullsize_oracle.py, which calls only oracle/; each target against all N
sources).

Gate (BASELINE north_star): relative rms of phi = phi^F + phi^R + phi^self against the exact
potential <= 1e-9.  C5 fixes rc = 0.1, whose real-space truncation error (Kolafa-Perram) is
far above 1e-10; it is reported twice (reading R-13): (i) at rc = 0.1 against the oracle
whose real-space term is truncated at the same rc (every other term exact), which isolates the
implementation error, plus the k-space part alone against the exact k-space potential; (ii) at
rc = 0.164, the cutoff of Eq. (rc) for a 1e-10 estimate, against the exact potential.
"""
import os

import numpy as np
import pytest

import oracle
from se1p_synth import CONFIGS, edge_targets, kspace_kwargs, make_system, sample_targets

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1611_09538_b200 as se1p  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RC_1E10_C5 = 0.164   # Eq. (rc), at E = 1e-10 for C5


def _golden(name, x):
    """Stored oracle set; the targets are re-derived from the seeded generator and must match."""
    d = np.load(os.path.join(GOLDEN, f"fullsize_{name}.npz"))
    cfg = CONFIGS[name]
    h = cfg.L[2] / cfg.M
    m, me = {"C4": (2048, 256), "C5": (512, 256)}[name]
    tg = np.unique(np.concatenate([sample_targets(cfg.N, m, cfg.seed + 31),
                                   edge_targets(x, cfg.L, cfg.P * h, me, cfg.seed + 31)]))
    assert np.array_equal(tg, d["targets"]), "golden targets do not match the seeded generator"
    return d


def _kspace_bench_path(cfg, xd, qd):
    """The call bench.py times (stream-ordered, checks skipped), after a validated call."""
    kw = kspace_kwargs(cfg)
    phik = torch.empty(cfg.N, dtype=torch.float64, device="cuda")
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, out=phik, **kw)
    se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, out=phik, stream=torch.cuda.current_stream(), sync=False,
                skip_checks=True, **kw)
    torch.cuda.synchronize()
    return phik.cpu().numpy()


def test_full_potential_c3():
    cfg = CONFIGS["C3"]
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    h = cfg.L[2] / cfg.M
    tg = np.unique(np.concatenate([sample_targets(cfg.N, 1024, cfg.seed), edge_targets(x, cfg.L, cfg.P * h, 128,
                                                                                        cfg.seed)]))
    got = _kspace_bench_path(cfg, xd, qd) + se1p.real(xd, qd, cfg.L, cfg.xi, cfg.rc).cpu().numpy()
    err = oracle.rel_rms(got[tg], oracle.phi_exact(x, q, cfg.L, tg))
    print(f"C3 rel rms {err:.3e} on {tg.size} targets")
    assert err <= 1e-9


def test_full_potential_c4():
    cfg = CONFIGS["C4"]
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    d = _golden("C4", x)
    tg = d["targets"]
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    got = _kspace_bench_path(cfg, xd, qd) + se1p.real(xd, qd, cfg.L, cfg.xi, cfg.rc).cpu().numpy()
    err = oracle.rel_rms(got[tg], d["exact"])
    print(f"C4 rel rms {err:.3e} on {tg.size} targets")
    assert err <= 1e-9


def test_full_potential_c5_both_cutoffs():
    cfg = CONFIGS["C5"]
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    d = _golden("C5", x)
    tg, exact = d["targets"], d["exact"]
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    phik = _kspace_bench_path(cfg, xd, qd)[tg]
    self_t = oracle.phi_self(q, cfg.xi, tg)
    # (i) rc = 0.1: same truncated real-space rule on both sides (R-13)
    got = phik + se1p.real(xd, qd, cfg.L, cfg.xi, cfg.rc).cpu().numpy()[tg]
    ref = exact - d["real_conv"] + d["real_trunc"]
    err_i = oracle.rel_rms(got, ref)
    kref = exact - d["real_conv"] - self_t
    err_k = oracle.rel_rms(phik, kref)
    # (ii) rc = 0.164 (Eq. (rc) at 1e-10) against the exact potential
    got2 = phik + se1p.real(xd, qd, cfg.L, cfg.xi, RC_1E10_C5).cpu().numpy()[tg]
    err_ii = oracle.rel_rms(got2, exact)
    print(f"C5 rel rms: rc=0.1 vs truncated oracle {err_i:.3e}; k-space {err_k:.3e}; rc=0.164 vs exact {err_ii:.3e}")
    assert err_i <= 1e-9
    assert err_k <= 1e-9 * np.sqrt(np.mean(exact ** 2) / np.mean(kref ** 2))
    assert err_ii <= 1e-9


def test_kspace_repeat_bitwise_c4():
    """Stream-ordered repeated calls (the bench loop) give bitwise identical results."""
    cfg = CONFIGS["C4"]
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = kspace_kwargs(cfg)
    a = se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, **kw)
    outs = []
    for _ in range(3):
        outs.append(se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, sync=False, skip_checks=True, **kw))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, a)


def test_c3_at_the_papers_rule_values():
    """C3 at the paper's literal upsampling rule: s_l from e^{-2 pi s_l} < 1e-10
    (P:695), n_l = M/10, s0 = 2.4, J modes at M~ (no widening).  The result equals
    the Alg. 1 oracle at those parameters (so any error is the method's), and its error against
    the exact potential exceeds 1e-9: the rule, written for cubic boxes, under-pads the L3 = 2 box
    (reading R-8); the same n_l and M~ with S0 = SI = 8 M~ meet the gate."""
    from oracle import se1p_discrete as sd
    cfg = CONFIGS["C3"]
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    h = cfg.L[2] / cfg.M
    Mt = int(round(cfg.L[0] / h)) + cfg.P
    s_l = np.log(1e10) / (2 * np.pi)
    rule = dict(n_local=round(cfg.M / 10), sf=s_l, s0=2.4, Ntilde=Mt)
    info = se1p.plan_info(cfg.L, cfg.xi, cfg.M, cfg.P, **rule)
    phik = se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, **rule).cpu().numpy()
    ref_alg1 = sd.se1p_kspace(x, q, cfg.L, cfg.xi, cfg.M, cfg.P, info["n_local"], info["S0"], info["SI"],
                              info["Ntilde"])
    assert np.max(np.abs(phik - ref_alg1)) <= 1e-11 * np.max(np.abs(ref_alg1))
    phir = se1p.real(xd, qd, cfg.L, cfg.xi, cfg.rc).cpu().numpy()
    tg = np.unique(np.concatenate([sample_targets(cfg.N, 1024, cfg.seed), edge_targets(x, cfg.L, cfg.P * h, 128,
                                                                                        cfg.seed)]))
    exact = oracle.phi_exact(x, q, cfg.L, tg)
    err_rule = oracle.rel_rms(phik[tg] + phir[tg], exact)
    wide = dict(n_local=round(cfg.M / 10), S0=8 * Mt, SI=8 * Mt, Ntilde=Mt)
    phiw = se1p.kspace(xd, qd, cfg.L, cfg.xi, cfg.M, cfg.P, **wide).cpu().numpy()
    err_wide = oracle.rel_rms(phiw[tg] + phir[tg], exact)
    print(f"C3 paper rule (S0={info['S0']}, SI={info['SI']}): rel rms {err_rule:.3e}; S0=SI=8M~: {err_wide:.3e}")
    assert err_rule > 1e-9 and err_wide <= 1e-9
