"""GPU analogue of the paper's Table 2 (tab:mfft_mifft): run-time ratio of the FFT/IFFT
work (z-FFT + mode stage + inverse z-FFT) between the "plain upsampled FFT" (s_l = s0 = s on every
mode, n_l = M/2) and the adaptive transform (n_l = 8, s_l = s0 = s), for M = 16..128, s in {2, 4}.
    python tools/table2.py  ->  one JSON line per (M, s) and a summary table"""
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import make_system  # noqa: E402

P, xi, L = 12, 1.0, (1.0, 1.0, 1.0)


def _factors(n):
    f, d = [], 2
    while d * d <= n:
        while n % d == 0:
            f.append(d)
            n //= d
        d += 1
    return f + ([n] if n > 1 else [])


def fft_ms(x, q, M, n_l, S, Nt):
    kw = dict(n_local=n_l, S0=S, SI=S, Ntilde=Nt, skip_checks=True, profile=True)
    acc = 0.0
    for r in range(7):
        se1p.kspace(x, q, L, xi * M / 16, M, P, **kw)
        st = se1p.stage_times()
        if r >= 2:
            acc += (st["zfft"] + st["modes"] + st["izfft"]) / 5
    return acc


x, q = make_system(20000, L, 3)
x, q = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
rows = {}
for s in (2, 4):
    for M in (16, 32, 48, 64, 80, 96, 112, 128, 192, 256):
        Mt = M + P
        S = -(-s * Mt // 1)
        # J modes of the AFT unpadded (s = 1, as in the paper): the FFT-friendly extent >= M~
        Nt = next(n for n in range(Mt, 2 * Mt) if all(f in (2, 3, 5) for f in _factors(n)))
        info = se1p.plan_info(L, xi * M / 16, M, P, n_local=8 if M > 16 else M // 2, S0=S, SI=S, Ntilde=Nt)
        t_aft = fft_ms(x, q, M, min(8, M // 2), S, Nt)
        t_plain = fft_ms(x, q, M, M // 2, S, Nt)
        rows[(s, M)] = t_plain / t_aft
        print(json.dumps({"s": s, "M": M, "Mt": Mt, "S": S, "Ntilde": Nt, "LK": info["LK"], "aft_ms": t_aft,
                          "plain_ms": t_plain, "ratio": t_plain / t_aft}), flush=True)
MS = (16, 32, 48, 64, 80, 96, 112, 128, 192, 256)
print("M    " + " ".join(f"{M:6d}" for M in MS))
for s in (2, 4):
    print(f"s={s}  " + " ".join(f"{rows[(s, M)]:6.2f}" for M in MS))
