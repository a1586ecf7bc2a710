"""GPU analogue of the paper's Ex. 5 (figs. 1p3p_tole5/tole10): k-space run time of
SE1P vs the SE3P baseline on the systems of tab:params: N/L^3 = 125, xi = 4,
tol 1e-5 (P = 12, s_l = 2) and 1e-9 (P = 24, s_l = 3), s0 ~ 2.4, J modes not upsampled.
    python tools/se1p_vs_se3p.py   ->  JSON lines + a table of SE1P/SE3P ratios"""
import json
import math
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import make_system  # noqa: E402

XI = 4.0
# (N, L, M and n_l at 1e-5, M and n_l at 1e-9) -- tab:params
ROWS = [(20000, 5.43, 52, 7, 68, 10), (40000, 6.84, 64, 9, 82, 11), (60000, 7.83, 76, 10, 94, 13),
        (80000, 8.62, 88, 10, 104, 14), (100000, 9.29, 96, 12, 114, 15),
        # B200-scale rows at the same density, h and M/n_l as the table (extrapolated, not the paper's)
        (500000, 15.874, 152, 20, 200, 29), (2000000, 25.198, 240, 32, 320, 47)]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    best.sort()
    return best[len(best) // 2]


def _factors(n):
    f, d = [], 2
    while d * d <= n:
        while n % d == 0:
            f.append(d)
            n //= d
        d += 1
    return f + ([n] if n > 1 else [])


def fft_part(st):
    return st["zfft"] + st["modes"] + st["izfft"]


out = []
for tol, P, sl in [(1e-5, 12, 2.0), (1e-9, 24, 3.0)]:
    for N, Lb, M5, nl5, M9, nl9 in ROWS:
        M, nl = (M5, nl5) if tol == 1e-5 else (M9, nl9)
        L = (Lb, Lb, Lb)
        x, q = make_system(N, L, 11)
        xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
        Mt = M + P
        # J modes unpadded (the paper's AFT): the FFT-friendly extent >= M~
        Nt = next((n for n in range(Mt, 2 * Mt) if all(p in (2, 3, 5) for p in _factors(n))), Mt)
        kw = dict(n_local=nl, S0=int(math.ceil(2.4 * Mt)), SI=int(math.ceil(sl * Mt)), Ntilde=Nt)
        t1 = timed(lambda: se1p.kspace(xd, qd, L, XI, M, P, skip_checks=True, **kw))
        se1p.kspace(xd, qd, L, XI, M, P, skip_checks=True, profile=True, **kw)
        s1 = se1p.stage_times()
        t3 = timed(lambda: se1p.kspace3p(xd, qd, L, XI, M, P, skip_checks=True))
        se1p.kspace3p(xd, qd, L, XI, M, P, skip_checks=True, profile=True)
        s3 = se1p.stage_times()
        r = dict(tol=tol, N=N, L=Lb, M=M, P=P, n_l=nl, se1p_ms=t1, se3p_ms=t3, ratio=t1 / t3,
                 se1p_fft_ms=fft_part(s1), se3p_fft_ms=fft_part(s3), fft_ratio=fft_part(s1) / fft_part(s3))
        out.append(r)
        print(json.dumps(r), flush=True)
print("tol    N       SE1P ms  SE3P ms  ratio  FFT+scale ratio")
for r in out:
    print(f"{r['tol']:.0e} {r['N']:7d} {r['se1p_ms']:8.3f} {r['se3p_ms']:8.3f} {r['ratio']:6.2f} {r['fft_ratio']:6.2f}")
