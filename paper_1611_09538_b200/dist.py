"""Mode-sharded SE1P k-space over R ranks.

One process per GPU, torch.distributed (NCCL) for the two all-to-all transposes and the final
all-reduce; every step of the method runs in libse1p's kernels (include/se1p.h, distributed
entries).  Per rank r:

  1. se1p_kspace_slab_forward: grid the x slab [xlo_r, xlo_{r+1}) of the extended grid
     (output-stationary tiles: no reduction between ranks) and z-transform it (AFT step 1,
     P:749) into the slab buffer [M/2+1 slots][W_r][M~], slots ordered by plane owner;
  2. all-to-all #1: the chunk of owner r' goes to rank r'; rank r receives its owned planes
     from every slab (the split buffer);
  3. se1p_kspace_modes on the owned planes (Alg. 2 steps 2-4, scaling, Alg. 3 steps 1-3,
     P:750-768) -- the k3 modes are independent, which is what shards;
  4. all-to-all #2 (the reverse) returns every rank its slab buffer;
  5. se1p_kspace_slab_backward: inverse z-transform and the gather
     over the slab's tiles -> phi_partial; all-reduce(sum) gives phi^F on every rank.

Plane ownership: greedy longest-processing-time on cost ~ W^2 log2 W per plane (W = the
plane's transform extent: LK for k3 = 0 and the upsampled I modes, Ntilde otherwise), so the
expensive upsampled planes spread over ranks.  The index bookkeeping
(slab bounds, owners, split sizes) is plain Python and is unit-tested on CPU with gloo.

kspace_rs / kspace_rank_rs: the particle-split baseline of SURVEY 8(e) (north_star literal:
particles split, the grid reduce-scattered, the k3 modes distributed, the inverse gathered back),
built from the same three entries over the whole grid.
"""
from __future__ import annotations

import dataclasses
import math

TILE = 16   # x extent of the gridding/gather tiles: slab bounds are multiples of it


def tile_weights(Mt: int, P: int) -> list:
    """Gridding/gather work of each 16-row x tile of the extended grid: the number of
    (particle column, stencil row) incidences, particles uniform over the M_free = Mt - P columns
    with stencil rows j0 .. j0+P-1, j0 = 1 .. M_free (reading R-3).  Boundary tiles are light."""
    Mf = Mt - P
    nt = (Mt + TILE - 1) // TILE
    w = []
    for t in range(nt):
        s = 0
        for r in range(t * TILE, min(Mt, (t + 1) * TILE)):
            s += max(0, min(Mf, r) - max(1, r - P + 1) + 1)
        w.append(float(s))
    return w


def slab_bounds(Mt: int, R: int, P=None) -> list:
    """R+1 x-row bounds 0 = b_0 <= ... <= b_R = Mt, multiples of TILE (b_R = Mt).  Without P the
    ceil(Mt/TILE) tiles are split as evenly as possible (lower ranks take the extra ones); with P
    the contiguous split minimises the largest slab's tile work (tile_weights; ties: the earliest
    bounds), since the boundary tiles carry little work."""
    if R < 1:
        raise ValueError("R >= 1")
    nt = (Mt + TILE - 1) // TILE
    if P is None:
        bounds = [0]
        for r in range(R):
            cnt = nt // R + (1 if r < nt % R else 0)
            bounds.append(min(Mt, bounds[-1] + TILE * cnt))
        bounds[-1] = Mt
        return bounds
    w = tile_weights(Mt, P)
    pre = [0.0]
    for v in w:
        pre.append(pre[-1] + v)
    INF = float("inf")
    # best[k][t]: minimal max load splitting tiles [0, t) into k slabs; cut[k][t]: last cut
    best = [[INF] * (nt + 1) for _ in range(R + 1)]
    cut = [[0] * (nt + 1) for _ in range(R + 1)]
    best[0][0] = 0.0
    for k in range(1, R + 1):
        for t in range(nt + 1):
            for s in range(t + 1):
                v = max(best[k - 1][s], pre[t] - pre[s])
                if v < best[k][t] - 1e-9 * max(1.0, v):
                    best[k][t], cut[k][t] = v, s
    ends = [nt]
    for k in range(R, 0, -1):
        ends.append(cut[k][ends[-1]])
    tiles = ends[::-1]                       # R+1 tile indices, 0 .. nt
    return [min(Mt, TILE * t) for t in tiles[:-1]] + [Mt]


def plane_costs(info: dict) -> list:
    """Relative cost of each of the M/2+1 planes in the mode stage: W^2 log2 W."""
    n_planes, n_kernel = info["n_planes"], info["n_kernel_planes"]
    out = []
    for n in range(n_planes):
        W = info["LK"] if n < n_kernel else info["Ntilde"]
        out.append(W * W * math.log2(W))
    return out


def assign_planes(costs: list, R: int) -> list:
    """LPT: planes in decreasing cost (ties: lower index first) to the least loaded rank (ties:
    lower rank).  Returns owned[r] = sorted plane indices of rank r."""
    load = [0.0] * R
    owned = [[] for _ in range(R)]
    for n in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(R), key=lambda k: (load[k], k))
        owned[r].append(n)
        load[r] += costs[n]
    return [sorted(o) for o in owned]


@dataclasses.dataclass
class DistPlan:
    Mt: int
    n_planes: int
    R: int
    bounds: list          # slab bounds (R+1)
    owned: list           # owned[r]: plane indices
    order: list           # plane_order: planes grouped by owner, rank 0 first

    def width(self, r):
        return self.bounds[r + 1] - self.bounds[r]

    def count(self, r):
        return len(self.owned[r])

    # split sizes in float64 elements (a complex entry is 2 doubles)
    def splits_to_owners(self, r):
        """all-to-all #1, rank r: input chunks (to owner r') of its slab buffer."""
        return [2 * self.count(q) * self.width(r) * self.Mt for q in range(self.R)]

    def splits_from_slabs(self, r):
        """all-to-all #1, rank r: output chunks (from slab r') of its split buffer."""
        return [2 * self.count(r) * self.width(q) * self.Mt for q in range(self.R)]


def make_plan(info: dict, R: int) -> DistPlan:
    Mt, n_planes = info["Mt"], info["n_planes"]
    owned = assign_planes(plane_costs(info), R)
    order = [n for r in range(R) for n in owned[r]]
    return DistPlan(Mt, n_planes, R, slab_bounds(Mt, R, info.get("P")), owned, order)


class CudaBackend:
    """The product stages: libse1p's distributed entries on this rank's GPU."""

    def __init__(self, L, xi, M, P, stream=None, **kw):
        self.args = (L, xi, M, P)
        self.kw = kw
        self.stream = stream

    def forward(self, x, q, x_lo, x_hi, order):
        import paper_1611_09538_b200 as se1p
        return se1p.slab_forward(x, q, *self.args, x_lo, x_hi, order, stream=self.stream, skip_checks=True,
                                 **self.kw)

    def modes(self, buf, plane_ids, bounds):
        import paper_1611_09538_b200 as se1p
        if plane_ids:
            se1p.modes(buf, *self.args, plane_ids, bounds, stream=self.stream, **self.kw)
        return buf

    def backward(self, buf, N, x_lo, x_hi, order):
        import paper_1611_09538_b200 as se1p
        return se1p.slab_backward(buf, N, *self.args, x_lo, x_hi, order, stream=self.stream, **self.kw)


def kspace_rank(x, q, plan: DistPlan, backend, rank: int, group=None):
    """SPMD body of rank `rank` (torch.distributed initialised; works with nccl and gloo).
    Returns phi^F (all N particles) on every rank."""
    import torch
    import torch.distributed as dist
    r = rank
    x_lo, x_hi = plan.bounds[r], plan.bounds[r + 1]
    N = q.shape[0]
    slab = backend.forward(x, q, x_lo, x_hi, plan.order)
    split = torch.empty(2 * plan.count(r) * plan.Mt * plan.Mt, dtype=torch.float64, device=slab.device)
    dist.all_to_all_single(split, slab.reshape(-1), plan.splits_from_slabs(r), plan.splits_to_owners(r), group=group)
    backend.modes(split, plan.owned[r], plan.bounds)
    back = torch.empty_like(slab).reshape(-1)
    dist.all_to_all_single(back, split, plan.splits_to_owners(r), plan.splits_from_slabs(r), group=group)
    phi = backend.backward(back.reshape(slab.shape), N, x_lo, x_hi, plan.order)
    dist.all_reduce(phi, group=group)
    return phi


def kspace_emulated(x, q, plan: DistPlan, backend):
    """All R ranks of kspace_rank run in turn in one process (the transposes become local copies
    with the same split sizes).  Used to test the decomposition on one GPU; no kernel waits on
    another rank."""
    import torch
    R, N = plan.R, q.shape[0]
    slabs = [backend.forward(x, q, plan.bounds[r], plan.bounds[r + 1], plan.order).reshape(-1) for r in range(R)]
    chunks = [list(torch.split(slabs[r], plan.splits_to_owners(r))) for r in range(R)]
    splits = [torch.cat([chunks[src][r] for src in range(R)]) for r in range(R)]   # all-to-all #1
    for r in range(R):
        backend.modes(splits[r], plan.owned[r], plan.bounds)
    back = [list(torch.split(splits[r], plan.splits_from_slabs(r))) for r in range(R)]
    phi = None
    for r in range(R):
        buf = torch.cat([back[owner][r] for owner in range(R)])                       # all-to-all #2
        # the device workspace holds the particle state of the LAST forward, and each rank's
        # forward keeps only its slab's particles: redo rank r's forward (its planes are discarded)
        if R > 1:
            backend.forward(x, q, plan.bounds[r], plan.bounds[r + 1], plan.order)
        part = backend.backward(buf.reshape(plan.n_planes, plan.width(r), plan.Mt, 2), N, plan.bounds[r],
                                plan.bounds[r + 1], plan.order)
        phi = part.clone() if phi is None else phi + part
    return phi


# ------------------------------------------------------------------ particle-split baseline
def rs_chunks(plan: DistPlan) -> list:
    """Full-grid plane buffer [M/2+1 slots in owner order][Mt][Mt] complex: the float64 sizes of
    the owners' chunks (owner q's planes, all rows)."""
    return [2 * plan.count(q) * plan.Mt * plan.Mt for q in range(plan.R)]


def kspace_rank_rs(x, q, plan: DistPlan, backend, rank: int, group=None):
    """SPMD body of the north_star-literal baseline: rank r holds only ITS particles
    (x [N_r, 3], q [N_r]) and returns phi^F of them.

      1. forward over the whole grid (x rows [0, Mt)): its particles' gridding and z-transform,
         i.e. their partial spectrum of every plane (the transforms are linear);
      2. reduce-scatter: owner q receives the sum over ranks of its planes (all-to-all of the plane
         chunks, then a local sum in rank order -- deterministic, and gloo has no reduce-scatter);
      3. the mode stage on the owned planes (one slab: bounds [0, Mt]);
      4. all-gather: every rank receives every processed plane (all-to-all of its chunk);
      5. backward over the whole grid: inverse z-transform and the gather of its own particles
         (no all-reduce: each rank owns its particles' phi).
    Against the slab path it trades the full-N gridding/gather on every rank for full-grid
    transforms on every rank and full-grid collectives (2 x (M/2+1) Mt^2 complex per rank)."""
    import torch
    import torch.distributed as dist
    R, r, Mt = plan.R, rank, plan.Mt
    N = q.shape[0]
    full = backend.forward(x, q, 0, Mt, plan.order)
    shape = full.shape
    sizes = rs_chunks(plan)
    flat = full.reshape(-1)
    recv = torch.empty(R * sizes[r], dtype=flat.dtype, device=flat.device)
    dist.all_to_all_single(recv, flat, [sizes[r]] * R, sizes, group=group)
    mine = recv[:sizes[r]].clone()
    for src in range(1, R):
        mine += recv[src * sizes[r]:(src + 1) * sizes[r]]
    backend.modes(mine, plan.owned[r], [0, Mt])
    out = torch.empty_like(flat)
    dist.all_to_all_single(out, mine.repeat(R), sizes, [sizes[r]] * R, group=group)
    return backend.backward(out.reshape(shape), N, 0, Mt, plan.order)


def kspace_emulated_rs(x, q, plan: DistPlan, backend, parts):
    """kspace_rank_rs for all ranks in turn in one process; parts[r] = (lo, hi) particle range of
    rank r.  Returns phi^F of all particles (rank ranges concatenated)."""
    import torch
    R, Mt = plan.R, plan.Mt
    sizes = rs_chunks(plan)
    fulls = [backend.forward(x[a:b], q[a:b], 0, Mt, plan.order).reshape(-1).clone() for a, b in parts]
    shape = None
    owned = []
    for r in range(R):
        chunk = None
        for src in range(R):
            c = torch.split(fulls[src], sizes)[r]
            chunk = c.clone() if chunk is None else chunk + c
        backend.modes(chunk, plan.owned[r], [0, Mt])
        owned.append(chunk)
    allp = torch.cat(owned)
    out = []
    for r, (a, b) in enumerate(parts):
        full = backend.forward(x[a:b], q[a:b], 0, Mt, plan.order)   # this rank's particle state
        shape = full.shape
        out.append(backend.backward(allp.reshape(shape).clone(), b - a, 0, Mt, plan.order).clone())
    return torch.cat(out)


_PLANS = {}


def cached_plan(L, xi, M, P, R, **kw):
    """DistPlan of the parameters for R ranks, built once (plan_info and the slab-bound DP are
    host work that does not change between calls)."""
    import paper_1611_09538_b200 as se1p
    pk = {k: kw.get(k) for k in ("eta", "s0", "sf", "n_local", "Ntilde", "S0", "SI")}
    key = (tuple(float(v) for v in L), float(xi), int(M), int(P), int(R), tuple(sorted(pk.items())))
    if key not in _PLANS:
        _PLANS[key] = make_plan(se1p.plan_info(L, xi, M, P, **pk), R)
    return _PLANS[key]


def kspace_rs(x, q, L, xi, M, P, group=None, stream=None, **kw):
    """phi^F of this rank's particles (x [N_r, 3], q [N_r]; CUDA float64) of one system whose
    particles are split over the ranks of `group` (the particle-split baseline, kspace_rank_rs)."""
    import torch
    import torch.distributed as dist
    R = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = cached_plan(L, xi, M, P, R, **kw)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.stream(st):
        return kspace_rank_rs(x, q, plan, CudaBackend(L, xi, M, P, stream=st, **kw), rank, group)


def kspace(x, q, L, xi, M, P, group=None, stream=None, **kw):
    """phi^F of one system sharded over the ranks of `group` (default: the world), every rank
    passing the same x [N,3], q [N] (CUDA, float64) and parameters.  The library stages and the
    collectives run on one stream (`stream`, default torch's current one), so each collective is
    ordered after the stage that produced its input."""
    import torch
    import torch.distributed as dist
    R = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = cached_plan(L, xi, M, P, R, **kw)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.stream(st):
        return kspace_rank(x, q, plan, CudaBackend(L, xi, M, P, stream=st, **kw), rank, group)


def real(x, q, L, xi, rc, group=None, stream=None, field=False, skip_checks=True):
    """phi^R + phi^self (se1p.real) of one system shared by the ranks of `group`: every rank passes
    the same x, q, computes its part of the targets (include/se1p.h: the target groups split in
    R near-equal parts, the other entries 0) and one all-reduce (sum) on the stream gives every
    rank the whole result -- bitwise equal to the single-GPU call (each entry has one nonzero
    contributor).  field=True also returns E^R."""
    import torch
    import torch.distributed as dist
    import paper_1611_09538_b200 as se1p
    R = dist.get_world_size(group)
    rank = dist.get_rank(group)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.stream(st):
        res = se1p.real(x, q, L, xi, rc, stream=st, sync=False, skip_checks=skip_checks, field=field,
                        part=(rank, R) if R > 1 else None)
        for t in (res if field else (res,)):
            if R > 1:
                dist.all_reduce(t, group=group)
    return res
