"""bench.py -- SE1P k-space throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

A step is one pass of the whole k-space hot path (bin/sort, gridding, z-FFT,
mode stage, inverse z-FFT, gather) over the config's synthetic system with the inputs resident
in HBM.  value = particles of the system / time.  Multi-GPU (torchrun): ONE system sharded over
the ranks (paper_1611_09538_b200/dist.py: x slabs, k3 modes owned by ranks, two all-to-all
transposes and an all-reduce over NCCL) -> "scaling": "strong"; time = max over ranks.
The CPU oracle (oracle/) is timed beside it on a bounded sample (cpu_baseline), and
--impl reference times the oracle as the reference arm.  Run with --gpus N > 1 outside torchrun,
bench.py launches itself under torch.distributed.run with N ranks (127.0.0.1).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from se1p_synth import CONFIGS, kspace_kwargs, make_system, sample_targets  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "SE1P k-space particles/sec (fp64) and achieved HBM GB/s fraction at 1/2/4/8 B200"   # BASELINE.json
# FP64 CUDA-core peak derived from unit counts and clock:
#   148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dist", default="slab", choices=["slab", "rs"],
                    help="N > 1: slab (x slabs + k3 modes, every rank holds all particles) or rs (the "
                         "particle-split baseline: each rank holds N/R particles, planes reduce-scattered)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def kspace_flops_spread(cfg):
    return 2.0 * cfg.N * cfg.P ** 3       # one FMA per stencil point (Eq. (spread_1p))


def cpu_oracle_rate(cfg, seconds):
    """Oracle (plain CPU Ewald1P, oracle/ewald1p.c) on seeded targets vs all N sources; its
    source sums are split over fixed source blocks, so all cores work for any number of targets."""
    import oracle
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    # calibrate on a few targets, then run a sample sized for ~`seconds`
    t0 = time.perf_counter()
    oracle.phi_exact(x, q, cfg.L, sample_targets(cfg.N, 4, cfg.seed))
    per_target = max((time.perf_counter() - t0) / 4, 1e-6)
    m = int(max(4, min(cfg.N, seconds / per_target)))
    tg = sample_targets(cfg.N, m, cfg.seed + 1)
    t0 = time.perf_counter()
    oracle.phi_exact(x, q, cfg.L, tg)
    dt = time.perf_counter() - t0
    cores = oracle.threads_used(cfg.N, m)
    return {"value": m / dt, "unit": "particles/s", "cores": cores, "kind": "oracle",
            "sample": f"{m} seeded targets of {cfg.name} (exact Ewald1P potential, all {cfg.N} sources each), {dt:.1f} s"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(self.idx), "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def bench_ours(args, cfg, rank, world, local):
    import torch
    import paper_1611_09538_b200 as se1p
    from paper_1611_09538_b200 import dist as sdist

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    x_np, q_np = make_system(cfg.N, cfg.L, cfg.seed)        # the same system on every rank
    rs = world > 1 and args.dist == "rs"
    if rs:   # the particle-split baseline: this rank holds (and uploads) only its share
        a, b = cfg.N * rank // world, cfg.N * (rank + 1) // world
        x_np, q_np = np.ascontiguousarray(x_np[a:b]), np.ascontiguousarray(q_np[a:b])
    n_loc = q_np.shape[0]
    x = torch.from_numpy(x_np).to(dev)
    q = torch.from_numpy(q_np).to(dev)
    phi = torch.empty(n_loc, dtype=torch.float64, device=dev)
    # single GPU: a side stream so the step can run as a captured CUDA graph (the legacy default
    # stream cannot be captured); multi-GPU keeps torch's current stream for NCCL
    stream = torch.cuda.Stream(device=dev) if world == 1 else torch.cuda.current_stream(dev)
    torch.cuda.set_stream(stream)
    kw = kspace_kwargs(cfg)
    info = se1p.plan_info(cfg.L, cfg.xi, cfg.M, cfg.P, **kw)

    def step(xs=x, qs=q, out=phi):
        if rs:
            return sdist.kspace_rs(xs, qs, cfg.L, cfg.xi, cfg.M, cfg.P, stream=stream, **kw)
        if world > 1:
            return sdist.kspace(xs, qs, cfg.L, cfg.xi, cfg.M, cfg.P, stream=stream, **kw)
        se1p.kspace(xs, qs, cfg.L, cfg.xi, cfg.M, cfg.P, out=out, stream=stream, sync=False, skip_checks=True,
                    graph=True, **kw)
        return out

    se1p.kspace(x, q, cfg.L, cfg.xi, cfg.M, cfg.P, out=phi, **kw)   # plan + workspace, validated inputs
    for _ in range(args.warmup):
        step()
    launches_per_step = se1p.launch_count() if world == 1 else None
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([v], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    clk = ClockSampler(local)
    barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # end-to-end through the C ABI with HOST buffers (se1p_kspace_ex, opts->host_io): every call
    # copies x, q from pinned host memory into the library's device buffers, runs the step and
    # copies phi back to pinned host memory before it returns (synchronous), K calls timed on the
    # device between events on the call's stream.  Multi-GPU: the torch-staged copies below.
    xh = torch.from_numpy(x_np).pin_memory()
    qh = torch.from_numpy(q_np).pin_memory()
    ph = torch.empty(n_loc, dtype=torch.float64).pin_memory()
    ke = max(3, args.steps // 2)
    e2e_pipelined = None
    if world == 1:
        xhn, qhn, phn = xh.numpy(), qh.numpy(), ph.numpy()
        legacy = torch.cuda.default_stream(dev)
        se1p.kspace(xhn, qhn, cfg.L, cfg.xi, cfg.M, cfg.P, out=phn, skip_checks=True, **kw)   # host staging buffers
        torch.cuda.synchronize(dev)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(legacy)
        for _ in range(ke):
            se1p.kspace(xhn, qhn, cfg.L, cfg.xi, cfg.M, cfg.P, out=phn, skip_checks=True, **kw)
        f1.record(legacy)
        torch.cuda.synchronize(dev)
        e2e_s = f0.elapsed_time(f1) / ke * 1e-3
        assert np.array_equal(phn, phi.cpu().numpy()), "host-buffer result differs from the device step"

    # end-to-end as a streaming user pipelines it (torch-staged copies): two buffer slots and copy
    # streams, so step i+1's H2D and step i-1's D2H overlap step i; multi-GPU: one slot, serial.
    nslot = 2 if world == 1 else 1
    slots = [dict(x=torch.empty_like(x), q=torch.empty_like(q), phi=torch.empty_like(phi),
                  ph=torch.empty(n_loc, dtype=torch.float64).pin_memory(),
                  loaded=torch.cuda.Event(), computed=torch.cuda.Event(), read=torch.cuda.Event())
             for _ in range(nslot)]
    h2d = torch.cuda.Stream(device=dev) if world == 1 else stream
    d2h = torch.cuda.Stream(device=dev) if world == 1 else stream

    def e2e_run(n):
        for i in range(n):
            s = slots[i % nslot]
            h2d.wait_event(s["computed"])        # the slot's previous step has consumed its inputs
            with torch.cuda.stream(h2d):
                s["x"].copy_(xh, non_blocking=True)
                s["q"].copy_(qh, non_blocking=True)
            s["loaded"].record(h2d)
            stream.wait_event(s["loaded"])
            stream.wait_event(s["read"])          # the slot's previous phi has reached the host
            out = step(s["x"], s["q"], s["phi"])
            s["computed"].record(stream)
            d2h.wait_event(s["computed"])
            with torch.cuda.stream(d2h):
                s["ph"].copy_(out, non_blocking=True)
            s["read"].record(d2h)
        stream.wait_stream(d2h)

    e2e_run(nslot)                                # capture each slot's graph
    torch.cuda.synchronize(dev)
    barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_run(ke)
    f1.record(stream)
    torch.cuda.synchronize(dev)
    pipe_s = max_over_ranks(f0.elapsed_time(f1) / ke) * 1e-3
    if world == 1:
        assert np.array_equal(slots[0]["ph"].numpy(), phi.cpu().numpy()), "e2e result differs from the device step"
        e2e_pipelined = cfg.N / pipe_s
    else:
        e2e_s = pipe_s

    # full SE1P at this config (BASELINE C5: real-space erfc sum with cell lists at rc plus k-space):
    # the real-space call timed alone on the step's stream (N > 1: dist.real, each rank its part of
    # the targets and one all-reduce, max over ranks), reported beside the k-space metric
    full = None
    if not rs and getattr(cfg, "rc", None):
        rbuf = torch.empty(n_loc, dtype=torch.float64, device=dev)

        def real_step():
            if world > 1:
                return sdist.real(x, q, cfg.L, cfg.xi, cfg.rc, stream=stream)
            return se1p.real(x, q, cfg.L, cfg.xi, cfg.rc, out=rbuf, stream=stream, sync=False, skip_checks=True)

        se1p.real(x, q, cfg.L, cfg.xi, cfg.rc, out=rbuf, stream=stream)   # erfc table, workspace, checked
        real_step()
        torch.cuda.synchronize(dev)
        barrier()
        nreal = 3
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(nreal):
            real_step()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        real_ms = max_over_ranks(g0.elapsed_time(g1) / nreal)
        full = {"value": cfg.N / ((ms + real_ms) * 1e-3), "unit": "particles/s", "rc": cfg.rc,
                "real_ms": real_ms, "kspace_ms": ms,
                "how": ("se1p_real_ex (k_real_warp) timed alone with CUDA events on the step's stream, "
                        "added to the k-space step time" if world == 1 else
                        "dist.real (each rank its part of the targets + one NCCL all-reduce), max over ranks, "
                        "added to the k-space step time")}

    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if rank != 0:
        return None

    # per-stage device times (separate profiled single-GPU passes; events on the launching stream)
    stage_sum = {}
    nprof = max(3, min(args.steps, 10))
    if rs:   # the stage split of the whole system on this GPU
        xf, qf = make_system(cfg.N, cfg.L, cfg.seed)
        xp, qp = torch.from_numpy(xf).to(dev), torch.from_numpy(qf).to(dev)
        pp = torch.empty(cfg.N, dtype=torch.float64, device=dev)
    else:
        xp, qp, pp = x, q, phi
    for _ in range(nprof):
        se1p.kspace(xp, qp, cfg.L, cfg.xi, cfg.M, cfg.P, out=pp, stream=stream, skip_checks=True, profile=True, **kw)
        for k, v in se1p.stage_times().items():
            stage_sum[k] = stage_sum.get(k, 0.0) + v / nprof
    if launches_per_step is None:
        launches_per_step = se1p.launch_count()

    spread_ms = stage_sum.get("spread", float("nan"))
    gather_ms = stage_sum.get("gather", float("nan"))
    dom_name, dom_ms = ("gather", gather_ms) if gather_ms >= spread_ms else ("spread", spread_ms)
    flops = kspace_flops_spread(cfg)          # gather: the same N P^3 FMAs
    achieved = flops / (dom_ms * 1e-3) / 1e12
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    traffic = kernel_traffic(dom_name)
    value = cfg.N / (ms * 1e-3)
    b_alg = 64.0 * cfg.N + 32.0 * cfg.M * info["Mt"] * info["Mt"]   # one system (strong scaling)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "particles/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded uniform neutral charges, se1p_synth.py)",
        "config": {"workload": f"{cfg.name}: N={cfg.N} L={list(cfg.L)} xi={cfg.xi} M={cfg.M} P={cfg.P} "
                               f"n_l={info['n_local']} S0={info['S0']} SI={info['SI']} Ntilde={info['Ntilde']} "
                               f"LK={info['LK']}",
                   "N": cfg.N,
                   "parallelism": ("particle-split x%d (N/R particles per rank, planes summed at their owners "
                                   "and gathered back: 2 all-to-all)" % world if rs else
                                   f"mode-sharded x{world} (x slabs + k3 planes, 2 all-to-all + all-reduce)")
                                  if world > 1 else "single GPU",
                   "l2": "per-step working set %.0f MB (particle records, grid, planes) > 126 MB L2; no flush"
                         % (info["workspace_bytes"] / 1e6 + 700 * cfg.N / 1e6)},
        "stages_ms": stage_sum,
        "roofline": {"bound": "alu", "kernel": f"k_sweep ({dom_name})", "achieved": achieved,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": traffic,
                     "note": "FP64 pipe (DMMA): 2 N P^3 algorithmic flops per launch / CUDA-event launch time on "
                             "the launching stream; peak = 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md; "
                             "measured DMMA 37.1, DFMA 34.2 TFLOP/s). traffic = ncu dram read+write bytes per "
                             "launch from profiles/ (null if not captured for this kernel)"},
        "hbm_gbs_peak": peaks.get("hbm_gbs"),
        # the metric's second part: whole-path algorithmic HBM bytes (64 N for the
        # particles + 32 G for the grid, G = M M~^2) per step time, as a fraction of the measured copy
        "hbm": {"bytes_per_step": b_alg, "achieved_gbs": b_alg / (ms * 1e-3) / 1e9,
                "peak_gbs": peaks.get("hbm_gbs"),
                "frac": (b_alg / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]) if peaks.get("hbm_gbs") else None,
                "note": "the path is FP64-bound (see roofline); DESIGN.md section 5"},
        "e2e": {"value": cfg.N / e2e_s, "unit": "particles/s",
                "h2d_bytes_per_step": 32 * cfg.N * (1 if rs else world), "d2h_bytes_per_step": 8 * cfg.N * (1 if rs else world),
                "how": "C ABI se1p_kspace_ex with host buffers (pinned), synchronous per call" if world == 1
                       else "torch-staged pinned copies around the distributed step"},
        "e2e_pipelined": ({"value": e2e_pipelined, "unit": "particles/s",
                           "how": "torch-staged pinned copies on two copy streams overlapping the graph step"}
                          if e2e_pipelined else None),
        "plan_ms": info.get("plan_ms"),
        "full_se1p": full,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    return line


def kernel_traffic(which):
    """dram bytes per launch of the dominant tile kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(path)).get(which)
    except (OSError, ValueError):
        return None


def bench_reference(args, cfg, rank, world=1):
    if rank != 0:
        return None
    import oracle
    x, q = make_system(cfg.N, cfg.L, cfg.seed)
    t0 = time.perf_counter()
    oracle.phi_exact(x, q, cfg.L, sample_targets(cfg.N, 2, cfg.seed))
    per_target = max((time.perf_counter() - t0) / 2, 1e-6)
    budget = 150.0 / max(1, args.steps + args.warmup)    # whole run within a few minutes
    # at least one target per core, so the reference arm and cpu_baseline time the same thing
    budget = max(budget, per_target * min(16, len(os.sched_getaffinity(0))) * 1.01)
    m = int(max(2, min(cfg.N, budget / per_target)))
    for i in range(args.warmup):
        oracle.phi_exact(x, q, cfg.L, sample_targets(cfg.N, m, cfg.seed + 10 + i))
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.phi_exact(x, q, cfg.L, sample_targets(cfg.N, m, cfg.seed + 100 + i))
    dt = (time.perf_counter() - t0) / args.steps
    value = m / dt
    cores = oracle.threads_used(cfg.N, m)
    sample = f"{m} seeded targets per step of {cfg.name} (exact Ewald1P, all {cfg.N} sources)"
    return {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "particles/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded uniform neutral charges, se1p_synth.py)",
            "config": {"workload": f"{cfg.name}: N={cfg.N} L={list(cfg.L)} xi={cfg.xi} M={cfg.M} P={cfg.P} "
                                   f"(the exact Ewald1P potential of the same system, on {cores} host cores)",
                       "N": cfg.N, "parallelism": "CPU oracle (rank 0 only)"},
            "cpu_baseline": {"value": value, "unit": "particles/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run with N ranks on
    127.0.0.1 (NCCL init lines on, for the rank check) and return its exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank, world, local = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        line = bench_reference(args, cfg, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    line = bench_ours(args, cfg, rank, world, local)
    if line is None:
        return
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_rate(cfg, args.cpu_seconds)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
