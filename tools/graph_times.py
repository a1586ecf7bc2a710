"""Eager vs CUDA-graph k-space calls (opts graph mode) on the configs and a paper-size system:
median device time per call with the inputs resident.   python tools/graph_times.py"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1611_09538_b200 as se1p  # noqa: E402
from se1p_synth import CONFIGS, kspace_kwargs, make_system  # noqa: E402


def med(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for name in ["C1", "C2", "C3", "C4", "C5"]:
    c = CONFIGS[name]
    x, q = make_system(c.N, c.L, c.seed)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    out = torch.empty(c.N, dtype=torch.float64, device="cuda")
    kw = kspace_kwargs(c)
    te = med(lambda: se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, skip_checks=True, out=out, sync=False, **kw))
    tg = med(lambda: se1p.kspace(xd, qd, c.L, c.xi, c.M, c.P, skip_checks=True, out=out, sync=False, graph=True, **kw))
    print(f"{name}: N={c.N:8d} eager {te:8.3f} ms  graph {tg:8.3f} ms  ({te / tg:.2f}x)", flush=True)
