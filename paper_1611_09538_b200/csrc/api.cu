// api.cu -- the C ABI of libse1p (include/se1p.h): argument validation, the parameter
// planner (Alg. 1 step 1 and DESIGN.md "Parameter choices"), workspaces, stage sequencing.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/se1p.h"
#include <nvtx3/nvToolsExt.h>

#include "kspace.cuh"
#include "real.cuh"
#include "sort.cuh"
#include "tiles.cuh"

namespace se1p {

static thread_local std::string g_err;
static thread_local int g_launches = 0;
static thread_local double g_stage_ms[10];
static thread_local int g_nstages = 0;
static std::mutex g_mu;

void count_launch() { ++g_launches; }

struct DevState {
  KWork w;
  KParams fwd_prm{};           // last se1p_kspace_slab_forward (state the backward relies on)
  int64_t fwd_N = -1;
  int* dmap = nullptr;          // device copies of plane maps (distributed path)
  int64_t dmap_cap = 0;
  int64_t fwd_nrel = -1;        // particles of the slab (compacted set) of the last forward
  int* sel = nullptr;           // [2N+1+scan scratch] flags, positions
  int64_t sel_cap = 0;
  int* idmap = nullptr;         // compacted index -> user index
  int64_t idmap_cap = 0;
  double* xsel = nullptr;       // compacted x (3n), q (n), phi partial (n)
  int64_t xsel_cap = 0;
  double* ef = nullptr;         // se1p_energy_forces: x, q staging, field parts, outputs
  int64_t ef_cap = 0;
  double* dx = nullptr;   // host_io staging (device side)
  double* dq = nullptr;
  double* dphi = nullptr;
  int64_t io_cap = 0;
  cudaEvent_t ws_done = nullptr;   // recorded after every call's work on its stream (WsOrder)
  cudaStream_t ws_stream = nullptr;
};
static DevState g_dev[64];
static uint64_t g_dev_used = 0;   // devices with state (se1p_set_allocator releases them all)

static DevState& dev_state() {
  int d = 0;
  SE1P_CUDA_TRY(cudaGetDevice(&d));
  g_dev_used |= 1ull << (d & 63);
  return g_dev[d & 63];
}

// Calls may come on different streams (graph mode's side stream, the caller's streams) and all
// share the device's workspace: each call's stream first waits for the work of the last call.
struct WsOrder {
  DevState& ds;
  cudaStream_t st;
  WsOrder(DevState& d, cudaStream_t s) : ds(d), st(s) {
    if (!ds.ws_done) SE1P_CUDA_TRY(cudaEventCreateWithFlags(&ds.ws_done, cudaEventDisableTiming));
    else if (ds.ws_stream != st) SE1P_CUDA_TRY(cudaStreamWaitEvent(st, ds.ws_done, 0));
  }
  ~WsOrder() {
    if (cudaEventRecord(ds.ws_done, st) == cudaSuccess) ds.ws_stream = st;
    else cudaGetLastError();
  }
};

static uint64_t g_ws_generation = 1;   // bumped on every workspace reallocation (graphs bake pointers)

// se1p_set_allocator hook (null: cudaMalloc / cudaFree)
static void* (*g_alloc_fn)(size_t, void*) = nullptr;
static void (*g_release_fn)(void*, void*) = nullptr;
static void* g_alloc_ctx = nullptr;

void* dev_alloc(size_t bytes) {
  bytes = std::max<size_t>(bytes, 8);
  void* p = nullptr;
  if (g_alloc_fn) {
    p = g_alloc_fn(bytes, g_alloc_ctx);
    if (!p) throw Error{5, "allocator hook returned null (" + std::to_string(bytes) + " bytes)"};
    return p;
  }
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    throw Error{5, "cudaMalloc failed (" + std::to_string(bytes) + " bytes)"};
  }
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  if (g_release_fn) {
    // the hook's memory may be handed out again at once: no library kernel may still use it
    // (cudaFree synchronises implicitly; frees are rare -- growth, eviction, release)
    cudaDeviceSynchronize();
    g_release_fn(p, g_alloc_ctx);
    return;
  }
  cudaFree(p);
}

template <typename T>
static void grow(T*& p, int64_t& cap, int64_t need) {
  if (need <= cap) return;
  ++g_ws_generation;
  dev_free(p);
  p = nullptr;
  cap = 0;
  dev_alloc(p, (size_t)std::max<int64_t>(need, 1));
  cap = need;
}

static void ensure_particles(KWork& w, int64_t N, int nbins) {
  grow(w.xs, w.cap_xs, 4 * N);
  grow(w.s4, w.cap_s4, 4 * N);
  grow(w.perm, w.cap_perm, N);
  grow(w.keys, w.cap_keys, N);
  grow(w.bin_start, w.cap_bs, (int64_t)nbins + 1);
  grow(w.scratch, w.scratch_cap, sort_scratch_ints(N, nbins));
  if (!w.red) {
    int64_t c1 = 0, c2 = 0;
    grow(w.red, c1, 4);
    grow(w.flag, c2, 4);
  }
}

// gather partial slots, records and the sweep kernels' overhang buffer and item table
static void ensure_sweep(KWork& w, const KDev& dv, int64_t N, int nvals) {
  grow(w.gpart, w.gpart_cap, N * gather_slots(dv) * nvals);
  grow(w.rec, w.cap_rec, N * (int64_t)rec_doubles(dv.P));
  grow(w.over, w.over_cap, sweep_overhang_doubles(dv));
  grow(w.items, w.items_cap, sweep_items_max(dv));
}

// ------------------------------------------------------------------ input checks
__global__ void k_check(const double* __restrict__ x, const double* __restrict__ q, int64_t N, double L0, double L1,
                        double* __restrict__ red, int* __restrict__ flag) {
  // single block, fixed-order reduction: sum q, sum |q|; flag bit 0 = domain, bit 1 = non-finite
  __shared__ double s1[1024], s2[1024];
  __shared__ int sf[1024];
  double a = 0.0, b = 0.0;
  int f = 0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
    const double px = x[3 * i], py = x[3 * i + 1], pz = x[3 * i + 2], qi = q[i];
    if (!isfinite(px) || !isfinite(py) || !isfinite(pz) || !isfinite(qi)) f |= 2;
    if (!(px >= 0.0 && px < L0 && py >= 0.0 && py < L1)) f |= 1;
    a += qi;
    b += fabs(qi);
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  sf[threadIdx.x] = f;
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      s1[threadIdx.x] += s1[threadIdx.x + off];
      s2[threadIdx.x] += s2[threadIdx.x + off];
      sf[threadIdx.x] |= sf[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    red[0] = s1[0];
    red[1] = s2[0];
    flag[0] = sf[0];
  }
}

static void check_inputs(KWork& w, const double* x, const double* q, int64_t N, const double L[3], bool neutral,
                         cudaStream_t st) {
  k_check<<<1, 1024, 0, st>>>(x, q, N, L[0], L[1], w.red, w.flag);
  SE1P_LAUNCH_CHECK();
  double red[2];
  int flag = 0;
  SE1P_CUDA_TRY(cudaMemcpyAsync(red, w.red, sizeof red, cudaMemcpyDeviceToHost, st));
  SE1P_CUDA_TRY(cudaMemcpyAsync(&flag, w.flag, sizeof flag, cudaMemcpyDeviceToHost, st));
  SE1P_CUDA_TRY(cudaStreamSynchronize(st));
  if (flag & 2) throw Error{1, "non-finite coordinate or charge"};
  if (flag & 1) throw Error{2, "an x or y coordinate lies outside [0,L1) x [0,L2) (free axes)"};
  if (neutral && std::fabs(red[0]) > 1e-12 * red[1])
    throw Error{3, "system is not charge neutral: |sum q| = " + std::to_string(std::fabs(red[0])) +
                       " > 1e-12 sum|q| (Eq. (5) needs neutrality, P:106-110)"};
}

// ------------------------------------------------------------------ planner
static int extent_from_factor(double s, int Mt) { return (int)std::ceil(s * Mt - 1e-9); }

// Resolve defaults.  Reading of the paper's recipe for B200:
//   eta    Eq. (comp_eta) with c = 0.95
//   n_l    given, else ~M/16 (>= 1)
//   S0,SI  given (opts or ceil(s M~)), else 8 M~: on this path an upsampled plane costs the
//          same for any S, so the planner takes a generous S
//   SJ     given, else the smallest FFT-friendly extent with Ntilde h - L >= 23 L3/(2 pi (n_l+1))
//          (aliasing distance of the first J mode for a 1e-10 estimate, SURVEY c-6)
//
// A rectangular free cross-section (L1 != L2, embed = true) is solved on the square domain
// [0, max(L1,L2))^2: phi^F is the free-space solution in x, y, so it does not depend
// on L1, L2 once every particle lies inside the grid's domain, and the truncated kernel's R
// (reading R-6) covers the larger square.  The particle checks still use the user's box.
static KParams resolve(const se1p_opts* o, const double Lu[3], double xi, int M, int P, double eta, double s0,
                       double sf, int n_local, bool embed = true) {
  if (!Lu || !(Lu[0] > 0) || !(Lu[1] > 0) || !(Lu[2] > 0)) throw Error{1, "box lengths must be positive"};
  const double Lsq = std::max(Lu[0], Lu[1]);
  const double L[3] = {embed ? Lsq : Lu[0], embed ? Lsq : Lu[1], Lu[2]};
  if (!(xi > 0)) throw Error{1, "xi must be positive"};
  if (M < 2) throw Error{1, "M must be >= 2"};
  KParams p{};
  p.L[0] = L[0];
  p.L[1] = L[1];
  p.L[2] = L[2];
  p.xi = xi;
  p.M = M;
  p.P = P;
  const double h = L[2] / M;
  const double m1 = L[0] / h, m2 = L[1] / h;
  const long M1 = std::lround(m1), M2 = std::lround(m2);
  if (std::fabs(m1 - M1) > 1e-9 * m1 || std::fabs(m2 - M2) > 1e-9 * m2)
    throw Error{4, "L1/h and L2/h must be integers (h = L3/M)"};
  if (M % 2) throw Error{4, "M must be even (Hermitian half along z)"};
  if (P < 2 || P > M || P > (int)M1 + P || P > 64) throw Error{4, "P must satisfy 2 <= P <= min(M, 64)"};
  const int Mt = (int)M1 + P;
  p.eta = (eta > 0) ? eta : P * xi * xi * h * h / (0.95 * 0.95 * kPi);
  if (!(p.eta > 0 && p.eta < 1)) throw Error{4, "eta must lie in (0,1) so the scaling damps (P:250)"};
  p.n_l = (n_local >= 0) ? n_local : std::max(1, (int)std::lround(M / 16.0));
  if (p.n_l > M / 2) throw Error{4, "n_local must be <= M/2"};
  const int S0o = o ? o->S0 : 0, SIo = o ? o->SI : 0, SJo = o ? o->Ntilde : 0;
  auto even = [](int v) { return v + (v & 1); };
  p.S0 = S0o > 0 ? S0o : (s0 > 0 ? extent_from_factor(s0, Mt) : even(8 * Mt));
  p.SI = SIo > 0 ? SIo : (sf > 0 ? extent_from_factor(sf, Mt) : even(8 * Mt));
  if (SJo > 0) {
    p.SJ = SJo;
  } else {
    const double gap = 23.0 * L[2] / (2.0 * kPi * (p.n_l + 1));
    p.SJ = next_friendly(std::max(Mt, (int)std::ceil((L[0] + gap) / h)));
  }
  if (p.S0 < Mt || p.SI < Mt || p.SJ < Mt) throw Error{4, "padded FFT extents must be >= M~ = M_free + P"};
  std::vector<int> r;
  if (!fft_factor(p.SJ, r) || !fft_factor(M, r)) throw Error{4, "FFT extent with a prime factor > 61"};
  return p;
}

static void fill_info(const KPlan& pl, se1p_plan_info* info) {
  if (!info) return;
  info->h = pl.dv.h;
  info->eta = pl.prm.eta;
  info->M = pl.prm.M;
  info->Mfree = pl.dv.Mfree;
  info->Mt = pl.dv.Mt;
  info->P = pl.prm.P;
  info->n_local = pl.prm.n_l;
  info->Ntilde = pl.prm.SJ;
  info->S0 = pl.prm.S0;
  info->SI = pl.prm.SI;
  info->LK = pl.LK;
  info->n_kernel_planes = pl.n_kernel;
  info->n_planes = pl.n_planes;
  info->grid_points = (int64_t)pl.dv.Mt * pl.dv.Mt * pl.prm.M;
  info->workspace_bytes = info->grid_points * 8 + (int64_t)pl.n_planes * pl.dv.Mt * pl.dv.Mt * 16 + pl.t_off_total * 16;
  info->plan_ms = pl.plan_ms;
}

// Stage boundaries of a k-space call: CUDA events on the call's stream (profiling mode) and NVTX
// ranges named after the stages (SURVEY 5 "Tracing"; no-ops without a tool attached).
struct StageTimer {
  static constexpr const char* kNames[8] = {"se1p bin", "se1p records", "se1p spread", "se1p zfft",
                                            "se1p modes", "se1p izfft",  "se1p gather", "se1p finish"};
  bool on;
  cudaStream_t st;
  cudaEvent_t ev[10];
  int n = 0, nm = 0;
  StageTimer(bool on_, cudaStream_t s) : on(on_), st(s) {
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark() {
    if (nm > 0 && nm <= 8) nvtxRangePop();
    if (nm < 8) nvtxRangePushA(kNames[nm]);
    ++nm;
    if (on && n < 10) cudaEventRecord(ev[n++], st);
  }
  void finish() {
    if (!on) return;
    cudaEventSynchronize(ev[n - 1]);
    g_nstages = n - 1;
    for (int i = 0; i + 1 < n; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      g_stage_ms[i] = ms;
    }
  }
  ~StageTimer() {
    if (nm > 0 && nm <= 8) nvtxRangePop();
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
};

// CUDA graphs of the k-space call (opts->reserved[3] == 1): the stage sequence is captured once per
// (plan, N, pointers, stream, workspace generation) and replayed -- one launch instead of ~30.
struct GraphEntry {
  KParams prm;
  int64_t N;
  const void *x, *q, *phi, *field;
  cudaStream_t st;
  uint64_t gen;
  int launches;
  cudaGraphExec_t exec;
};
static std::vector<GraphEntry> g_graphs;

template <class F>
static void run_graphed(const KParams& prm, int64_t N, const void* x, const void* q, const void* phi,
                        const void* field, cudaStream_t st, F&& stages) {
  for (auto& g : g_graphs)
    if (g.prm == prm && g.N == N && g.x == x && g.q == q && g.phi == phi && g.field == field && g.st == st &&
        g.gen == g_ws_generation + kplan_generation()) {
      SE1P_CUDA_TRY(cudaGraphLaunch(g.exec, st));
      g_launches = g.launches;
      return;
    }
  if (st == 0) throw Error{1, "graph mode needs a non-default stream"};
  cudaGraph_t graph = nullptr;
  SE1P_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int l0 = g_launches;
  try {
    stages();
  } catch (...) {
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    throw;
  }
  SE1P_CUDA_TRY(cudaStreamEndCapture(st, &graph));
  cudaGraphExec_t exec = nullptr;
  SE1P_CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  if (g_graphs.size() >= 8) {
    cudaGraphExecDestroy(g_graphs.front().exec);
    g_graphs.erase(g_graphs.begin());
  }
  g_graphs.push_back(GraphEntry{prm, N, x, q, phi, field, st, g_ws_generation + kplan_generation(), g_launches - l0,
                                exec});
  SE1P_CUDA_TRY(cudaGraphLaunch(exec, st));
}

static void sync_and_check(cudaStream_t st) {
  SE1P_CUDA_TRY(cudaStreamSynchronize(st));
  SE1P_CUDA_TRY(cudaGetLastError());
}

static void kspace_impl(const se1p_opts* o, cudaStream_t st, const double* x, const double* q, int64_t N,
                        const double L[3], double xi, int M, int P, double eta, double s0, double sf, int n_local,
                        double* phi_out, double* field_out = nullptr, const int* S_modes = nullptr) {
  if (!x || !q || (!phi_out && !field_out)) throw Error{1, "null pointer"};
  if (N < 1) throw Error{1, "N must be >= 1"};
  if (N > (int64_t)2000000000) throw Error{1, "N too large for int32 indices"};
  KParams prm = resolve(o, L, xi, M, P, eta, s0, sf, n_local);
  if (S_modes) {   // multi-tier upsampling
    const int Mt = (int)std::lround(prm.L[0] / (L[2] / M)) + P;
    prm.SIn.assign(S_modes, S_modes + prm.n_l);
    for (int S : prm.SIn)
      if (S < Mt) throw Error{4, "every per-mode extent must be >= M~ = M_free + P"};
  }
  KPlan* pl = kplan_get(prm, st);
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  KWork& w = ds.w;
  const KDev& dv = pl->dv;
  ensure_particles(w, N, dv.nbx * dv.M * dv.Mfree);
  grow(w.grid, w.grid_cap, (int64_t)dv.Mt * dv.Mt * dv.M);
  grow(w.planes, w.planes_cap, (int64_t)pl->n_planes * dv.Mt * dv.Mt);
  grow(w.T, w.T_cap, pl->t_off_total);
  const bool host_io = o && o->host_io;
  const bool field = field_out != nullptr;
  const double *dx = x, *dq = q;
  double* dphi = phi_out;
  double* dfield = field_out;
  if (host_io) {
    grow(ds.dx, ds.io_cap, 8 * N);
    dx = ds.dx;
    dq = ds.dx + 3 * N;
    dphi = phi_out ? ds.dx + 4 * N : nullptr;
    dfield = field ? ds.dx + 5 * N : nullptr;
    SE1P_CUDA_TRY(cudaMemcpyAsync((void*)dx, x, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    SE1P_CUDA_TRY(cudaMemcpyAsync((void*)dq, q, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  }
  if (!(o && o->skip_checks)) check_inputs(w, dx, dq, N, L, true, st);
  StageTimer tm(o && o->reserved[0] == 1, st);
  SE1P_CUDA_TRY(cudaMemsetAsync(w.flag + 1, 0, sizeof(int), st));
  const int stop = o ? o->reserved[1] : 0;
  if (o && o->reserved[2]) throw Error{1, "opts->reserved[2] is unused and must be 0"};
  ensure_sweep(w, dv, N, field ? 4 : 1);
  const bool graph = o && o->reserved[3] == 1;
  if (graph && (host_io || stop || tm.on))
    throw Error{1, "graph mode takes device pointers and no profiling / early stop"};
  if (graph) {
    run_graphed(prm, N, dx, dq, dphi, dfield, st, [&] {
      k_bin_particles(*pl, w, dx, dq, N, st);
      k_records_stage(*pl, w, N, st);
      k_spread_tiles(*pl, w, N, st);
      const SlabLayout Lg = single_layout(dv.Mt, pl->n_planes);
      k_zfft_forward(*pl, w, w.planes, Lg, nullptr, st);
      k_mode_stage(*pl, w, w.planes, Lg, nullptr, nullptr, 0, nullptr, nullptr, 0, st);
      k_zfft_inverse(*pl, w, w.planes, Lg, nullptr, st);
      k_gather_tiles(*pl, w, N, st, 0, -1, field);
      k_gather_finish_stage(*pl, w, N, dphi, st, 0, -1, dfield);
    });
  }
  // stages (se1p_last_stage_times): bin, records, spread, zfft, modes, izfft, gather, finish
  if (!graph) {
  tm.mark();
  k_bin_particles(*pl, w, dx, dq, N, st);
  tm.mark();
  k_records_stage(*pl, w, N, st);
  tm.mark();
  k_spread_tiles(*pl, w, N, st);
  tm.mark();
  if (stop == 1) return sync_and_check(st);
  const SlabLayout L1 = single_layout(dv.Mt, pl->n_planes);
  k_zfft_forward(*pl, w, w.planes, L1, nullptr, st);
  tm.mark();
  if (stop == 2) return sync_and_check(st);
  k_mode_stage(*pl, w, w.planes, L1, nullptr, nullptr, 0, nullptr, nullptr, 0, st);
  tm.mark();
  if (stop == 3) return sync_and_check(st);
  k_zfft_inverse(*pl, w, w.planes, L1, nullptr, st);
  tm.mark();
  if (stop == 4) return sync_and_check(st);
  k_gather_tiles(*pl, w, N, st, 0, -1, field);
  tm.mark();
  k_gather_finish_stage(*pl, w, N, dphi, st, 0, -1, dfield);
  tm.mark();
  }
  if (host_io && phi_out) SE1P_CUDA_TRY(cudaMemcpyAsync(phi_out, dphi, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
  if (host_io && field)
    SE1P_CUDA_TRY(cudaMemcpyAsync(field_out, dfield, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, st));
  tm.finish();
  if (!o || o->sync || host_io) {
    SE1P_CUDA_TRY(cudaStreamSynchronize(st));
    int kerr = 0;
    SE1P_CUDA_TRY(cudaMemcpy(&kerr, w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost));
    if (kerr) throw Error{6, "sweep kernel internal bounds check failed (code " + std::to_string(kerr) + ")"};
  }
  SE1P_CUDA_TRY(cudaGetLastError());
}

// SE3P baseline (the paper's Ex. 5): the 1P tile plan grids and
// gathers on the extended grid; a periodic transform plan (every plane a J plane of extent
// M_free, k = 0 dropped) does the 3D transform and the 3P scaling on the folded grid.
static void kspace3p_impl(const se1p_opts* o, cudaStream_t st, const double* x, const double* q, int64_t N,
                          const double L[3], double xi, int M, int P, double eta, double* phi_out) {
  if (!x || !q || !phi_out) throw Error{1, "null pointer"};
  if (N < 1) throw Error{1, "N must be >= 1"};
  if (N > (int64_t)2000000000) throw Error{1, "N too large for int32 indices"};
  if (P % 2) throw Error{4, "SE3P needs an even P (the folded stencil nodes are then lattice nodes)"};
  se1p_opts none{};
  if (L && L[0] != L[1]) throw Error{4, "SE3P in this build requires a square periodic cross-section (L1 == L2)"};
  KParams pa = resolve(&none, L, xi, M, P, eta, -1.0, -1.0, 0, false);
  const int Mf = (int)std::lround(L[0] / (L[2] / M));
  pa.n_l = -1;   // tile plan only: no kernel planes, no upsampling
  pa.S0 = pa.SI = Mf + P;
  std::vector<int> r;
  if (!fft_factor(Mf, r)) throw Error{4, "L1/h has a prime factor > 61"};
  KParams pb = pa;
  pb.periodic = 1;
  pb.SJ = Mf;
  KPlan* pl = kplan_get(pa, st);
  KPlan* p3 = kplan_get(pb, st);
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  KWork& w = ds.w;
  const KDev& dv = pl->dv;
  ensure_particles(w, N, dv.nbx * dv.M * dv.Mfree);
  grow(w.grid, w.grid_cap, (int64_t)dv.Mt * dv.Mt * dv.M);
  grow(w.grid3, w.grid3_cap, (int64_t)Mf * Mf * dv.M);
  grow(w.planes, w.planes_cap, (int64_t)p3->n_planes * Mf * Mf);
  grow(w.T, w.T_cap, p3->t_off_total);
  ensure_sweep(w, dv, N, 1);
  const bool host_io = o && o->host_io;
  const double *dx = x, *dq = q;
  double* dphi = phi_out;
  if (host_io) {
    grow(ds.dx, ds.io_cap, 5 * N);
    dx = ds.dx;
    dq = ds.dx + 3 * N;
    dphi = ds.dx + 4 * N;
    SE1P_CUDA_TRY(cudaMemcpyAsync((void*)dx, x, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    SE1P_CUDA_TRY(cudaMemcpyAsync((void*)dq, q, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  }
  if (!(o && o->skip_checks)) check_inputs(w, dx, dq, N, L, true, st);
  StageTimer tm(o && o->reserved[0] == 1, st);
  SE1P_CUDA_TRY(cudaMemsetAsync(w.flag + 1, 0, sizeof(int), st));
  // stages: bin, records, spread, fold + z-FFT, modes, inverse z-FFT + unfold, gather, finish
  tm.mark();
  k_bin_particles(*pl, w, dx, dq, N, st);
  tm.mark();
  k_records_stage(*pl, w, N, st);
  tm.mark();
  k_spread_tiles(*pl, w, N, st);
  tm.mark();
  k_fold_3p(*pl, w.grid, w.grid3, st);
  KWork w3 = w;          // the transform stages read and write the periodic grid
  w3.grid = w.grid3;
  const SlabLayout L3 = single_layout(Mf, p3->n_planes);
  k_zfft_forward(*p3, w3, w.planes, L3, nullptr, st);
  tm.mark();
  k_mode_stage(*p3, w3, w.planes, L3, nullptr, nullptr, 0, nullptr, nullptr, 0, st);
  tm.mark();
  k_zfft_inverse(*p3, w3, w.planes, L3, nullptr, st);
  k_unfold_3p(*pl, w.grid3, w.grid, st);
  tm.mark();
  k_gather_tiles(*pl, w, N, st);
  tm.mark();
  k_gather_finish_stage(*pl, w, N, dphi, st);
  tm.mark();
  if (host_io) SE1P_CUDA_TRY(cudaMemcpyAsync(phi_out, dphi, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
  tm.finish();
  if (!o || o->sync || host_io) {
    SE1P_CUDA_TRY(cudaStreamSynchronize(st));
    int kerr = 0;
    SE1P_CUDA_TRY(cudaMemcpy(&kerr, w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost));
    if (kerr) throw Error{6, "sweep kernel internal bounds check failed (code " + std::to_string(kerr) + ")"};
  }
  SE1P_CUDA_TRY(cudaGetLastError());
}

static void real_impl(const se1p_opts* o, cudaStream_t st, const double* x, const double* q, int64_t N,
                      const double L[3], double xi, double rc, double* phi_out, double* field_out = nullptr) {
  if (!x || !q || (!phi_out && !field_out) || !L) throw Error{1, "null pointer"};
  if (N < 1) throw Error{1, "N must be >= 1"};
  if (!(xi > 0) || !(rc > 0) || !(L[0] > 0) || !(L[1] > 0) || !(L[2] > 0)) throw Error{1, "xi, rc, L must be > 0"};
  const int nparts = o ? std::max(1, o->reserved[4]) : 1, part = o ? o->reserved[5] : 0;
  if (o && (o->reserved[4] < 0 || part < 0 || part >= nparts))
    throw Error{1, "opts->reserved[4] (parts) >= 0 and 0 <= opts->reserved[5] (part) < max(parts, 1) required"};
  const RDev d = real_geometry(L, xi, rc, N);
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  KWork& w = ds.w;
  ensure_particles(w, N, real_nbins(d));
  grow(w.scratch, w.scratch_cap, real_scratch_ints(d, N));
  const bool host_io = o && o->host_io;
  const double *dx = x, *dq = q;
  double* dphi = phi_out;
  double* dfield = field_out;
  if (host_io) {
    grow(ds.dx, ds.io_cap, 8 * N);
    dx = ds.dx;
    dq = ds.dx + 3 * N;
    dphi = phi_out ? ds.dx + 4 * N : nullptr;
    dfield = field_out ? ds.dx + 5 * N : nullptr;
    SE1P_CUDA_TRY(cudaMemcpyAsync((void*)dx, x, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    SE1P_CUDA_TRY(cudaMemcpyAsync((void*)dq, q, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  }
  if (!(o && o->skip_checks)) check_inputs(w, dx, dq, N, L, false, st);
  if (nparts > 1) {   // the other parts' entries are 0, so the parts of all ranks sum exactly
    if (dphi) SE1P_CUDA_TRY(cudaMemsetAsync(dphi, 0, sizeof(double) * N, st));
    if (dfield) SE1P_CUDA_TRY(cudaMemsetAsync(dfield, 0, sizeof(double) * 3 * N, st));
  }
  real_space(d, w, dx, dq, N, dphi, st, dfield, part, nparts);
  if (host_io && phi_out)
    SE1P_CUDA_TRY(cudaMemcpyAsync(phi_out, dphi, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
  if (host_io && field_out)
    SE1P_CUDA_TRY(cudaMemcpyAsync(field_out, dfield, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, st));
  if (!o || o->sync || host_io) SE1P_CUDA_TRY(cudaStreamSynchronize(st));
  SE1P_CUDA_TRY(cudaGetLastError());
}


// ------------------------------------------------------------------ distributed path
static void check_slab(const KPlan& pl, int x_lo, int x_hi) {
  const int Mt = pl.dv.Mt;
  if (x_lo < 0 || x_hi > Mt || x_lo > x_hi || (x_lo % 16 && x_lo != Mt) || (x_hi % 16 && x_hi != Mt))
    throw Error{1, "slab bounds must satisfy 0 <= x_lo <= x_hi <= M~, multiples of 16 or M~"};
}

static std::vector<int> check_order(const KPlan& pl, const int* plane_order) {
  if (!plane_order) throw Error{1, "null plane_order"};
  std::vector<int> slot(pl.n_planes, -1);
  for (int i = 0; i < pl.n_planes; ++i) {
    const int n = plane_order[i];
    if (n < 0 || n >= pl.n_planes || slot[n] >= 0) throw Error{1, "plane_order must be a permutation of 0..M/2"};
    slot[n] = i;
  }
  return slot;
}

static int* upload_ints(DevState& ds, const std::vector<int>& v, cudaStream_t st) {
  grow(ds.dmap, ds.dmap_cap, (int64_t)v.size());
  SE1P_CUDA_TRY(cudaMemcpyAsync(ds.dmap, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice, st));
  return ds.dmap;
}

static void finish_call(const se1p_opts* o, KWork& w, cudaStream_t st) {
  if (!o || o->sync) {
    SE1P_CUDA_TRY(cudaStreamSynchronize(st));
    int kerr = 0;
    SE1P_CUDA_TRY(cudaMemcpy(&kerr, w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost));
    if (kerr) throw Error{6, "sweep kernel internal bounds check failed (code " + std::to_string(kerr) + ")"};
  }
  SE1P_CUDA_TRY(cudaGetLastError());
}

static void slab_forward_impl(const se1p_opts* o, cudaStream_t st, const double* x, const double* q, int64_t N,
                              const double L[3], double xi, int M, int P, double eta, double s0, double sf,
                              int n_local, int x_lo, int x_hi, const int* plane_order, void* planes_out) {
  if (!x || !q || (!planes_out && x_hi > x_lo)) throw Error{1, "null pointer"};
  if (o && o->host_io) throw Error{1, "the distributed entries take device pointers only"};
  if (N < 1 || N > (int64_t)2000000000) throw Error{1, "N out of range"};
  const KParams prm = resolve(o, L, xi, M, P, eta, s0, sf, n_local);
  KPlan* pl = kplan_get(prm, st);
  check_slab(*pl, x_lo, x_hi);
  const std::vector<int> slot = check_order(*pl, plane_order);
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  KWork& w = ds.w;
  const KDev& dv = pl->dv;
  ensure_particles(w, N, dv.nbx * dv.M * dv.Mfree);
  grow(w.grid, w.grid_cap, (int64_t)dv.Mt * dv.Mt * dv.M);
  ensure_sweep(w, dv, N, 1);
  if (!(o && o->skip_checks)) check_inputs(w, x, q, N, L, true, st);
  SE1P_CUDA_TRY(cudaMemsetAsync(w.flag + 1, 0, sizeof(int), st));
  // only the particles whose stencils meet the slab's tiles are binned and gridded (the rest
  // cannot touch them): rows [16 ceil(x_lo/16), 16 ceil(x_hi/16))
  const int tlo = (int)ceil_div(x_lo, 16), thi = (int)ceil_div(x_hi, 16);
  grow(ds.sel, ds.sel_cap, 2 * N + 2 + scan_scratch_ints(N));
  grow(ds.idmap, ds.idmap_cap, N);
  grow(ds.xsel, ds.xsel_cap, 5 * N);
  int* flags = ds.sel;
  int* pos = ds.sel + N;
  double* xc = ds.xsel;
  double* qc = ds.xsel + 3 * N;
  k_slab_select(*pl, x, q, N, 16 * tlo, 16 * thi, flags, pos, pos + N + 1, xc, qc, ds.idmap, st);
  int nrel = 0;
  SE1P_CUDA_TRY(cudaMemcpyAsync(&nrel, pos + N, sizeof(int), cudaMemcpyDeviceToHost, st));
  SE1P_CUDA_TRY(cudaStreamSynchronize(st));
  if (nrel > 0) {
    k_bin_particles(*pl, w, xc, qc, nrel, st);
    k_records_stage(*pl, w, nrel, st);
    k_spread_tiles(*pl, w, nrel, st, tlo, thi);
  } else if (thi > tlo) {   // no particle meets the slab: its rows are zero
    const int64_t r0 = 16 * (int64_t)tlo, r1 = std::min<int64_t>(16 * (int64_t)thi, dv.Mt);
    SE1P_CUDA_TRY(cudaMemsetAsync(w.grid + r0 * dv.Mt * dv.M, 0, sizeof(double) * (r1 - r0) * dv.Mt * dv.M, st));
  }
  ds.fwd_nrel = nrel;
  SlabLayout Ls{};
  Ls.nslab = 1;
  Ls.nloc = pl->n_planes;
  Ls.xlo[0] = x_lo;
  Ls.xlo[1] = x_hi;
  k_zfft_forward(*pl, w, (double2*)planes_out, Ls, upload_ints(ds, slot, st), st);
  ds.fwd_prm = prm;
  ds.fwd_N = N;
  finish_call(o, w, st);
}

static void modes_impl(const se1p_opts* o, cudaStream_t st, const double L[3], double xi, int M, int P, double eta,
                       double s0, double sf, int n_local, int n_own, const int* plane_ids, int nslab,
                       const int* slab_lo, void* planes) {
  const KParams prm = resolve(o, L, xi, M, P, eta, s0, sf, n_local);
  KPlan* pl = kplan_get(prm, st);
  const int Mt = pl->dv.Mt;
  if (n_own < 0 || n_own > pl->n_planes || (n_own > 0 && (!plane_ids || !planes)))
    throw Error{1, "bad plane list"};
  if (nslab < 1 || nslab > kMaxSlabs || !slab_lo || slab_lo[0] != 0 || slab_lo[nslab] != Mt)
    throw Error{1, "slab_lo must hold nslab+1 increasing bounds from 0 to M~ (nslab <= 16)"};
  SlabLayout Ls{};
  Ls.nslab = nslab;
  Ls.nloc = n_own;
  for (int r = 0; r <= nslab; ++r) {
    if (r && slab_lo[r] < slab_lo[r - 1]) throw Error{1, "slab bounds must be non-decreasing"};
    Ls.xlo[r] = slab_lo[r];
  }
  std::vector<int> seen(pl->n_planes, 0), maps;   // glK liK glJ liJ
  std::vector<int> glK, liK, glJ, liJ;
  for (int i = 0; i < n_own; ++i) {
    const int n = plane_ids[i];
    if (n < 0 || n >= pl->n_planes || seen[n]++) throw Error{1, "plane_ids must be distinct planes in 0..M/2"};
    if (n < pl->n_kernel) {
      glK.push_back(n);
      liK.push_back(i);
    } else {
      glJ.push_back(n);
      liJ.push_back(i);
    }
  }
  if (n_own == 0) return;
  maps.insert(maps.end(), glK.begin(), glK.end());
  maps.insert(maps.end(), liK.begin(), liK.end());
  maps.insert(maps.end(), glJ.begin(), glJ.end());
  maps.insert(maps.end(), liJ.begin(), liJ.end());
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  KWork& w = ds.w;
  grow(w.T, w.T_cap, pl->t_off_total);
  if (!w.flag) ensure_particles(w, 1, 1);
  int* d = upload_ints(ds, maps, st);
  const int nK = (int)glK.size(), nJ = (int)glJ.size();
  k_mode_stage(*pl, w, (double2*)planes, Ls, d, d + nK, nK, d + 2 * nK, d + 2 * nK + nJ, nJ, st);
  finish_call(o, w, st);
}

static void slab_backward_impl(const se1p_opts* o, cudaStream_t st, int64_t N, const double L[3], double xi, int M,
                               int P, double eta, double s0, double sf, int n_local, int x_lo, int x_hi,
                               const int* plane_order, const void* planes_in, double* phi_partial) {
  if (!phi_partial || (!planes_in && x_hi > x_lo)) throw Error{1, "null pointer"};
  const KParams prm = resolve(o, L, xi, M, P, eta, s0, sf, n_local);
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  if (!(ds.fwd_N == N && ds.fwd_prm == prm))
    throw Error{1, "se1p_kspace_slab_backward needs the particle state of a matching se1p_kspace_slab_forward "
                   "on this device (same N and parameters)"};
  KPlan* pl = kplan_get(prm, st);
  check_slab(*pl, x_lo, x_hi);
  const std::vector<int> slot = check_order(*pl, plane_order);
  KWork& w = ds.w;
  SlabLayout Ls{};
  Ls.nslab = 1;
  Ls.nloc = pl->n_planes;
  Ls.xlo[0] = x_lo;
  Ls.xlo[1] = x_hi;
  k_zfft_inverse(*pl, w, (const double2*)planes_in, Ls, upload_ints(ds, slot, st), st);
  // the slab's particles (compacted by the forward): partials into their slots, then scattered
  // to user order; every other particle's partial is zero
  const int64_t nrel = ds.fwd_nrel;
  const int tlo = (int)ceil_div(x_lo, 16), thi = (int)ceil_div(x_hi, 16);
  SE1P_CUDA_TRY(cudaMemsetAsync(phi_partial, 0, sizeof(double) * N, st));
  if (nrel > 0) {
    double* phic = ds.xsel + 4 * N;
    k_gather_tiles(*pl, w, nrel, st, tlo, thi);
    k_gather_finish_stage(*pl, w, nrel, phic, st, tlo, thi);
    k_scatter_partial_stage(phic, ds.idmap, nrel, phi_partial, st);
  }
  finish_call(o, w, st);
}

// phi = phi^F + phi^R, F = q (E^F + E^R) per particle
__global__ void k_combine_forces(const double* __restrict__ q, const double* __restrict__ pk,
                                 const double* __restrict__ ek, const double* __restrict__ pr,
                                 const double* __restrict__ er, int64_t N, double* __restrict__ phi,
                                 double* __restrict__ F) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (phi) phi[i] = pk[i] + pr[i];
#pragma unroll
  for (int c = 0; c < 3; ++c) F[3 * i + c] = q[i] * (ek[3 * i + c] + er[3 * i + c]);
}

// U = 1/2 sum q (phi^F + phi^R): one block, fixed per-thread strides and a fixed tree
__global__ void k_energy(const double* __restrict__ q, const double* __restrict__ pk, const double* __restrict__ pr,
                         int64_t N, double* __restrict__ U) {
  __shared__ double s[1024];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) a += q[i] * (pk[i] + pr[i]);
  s[threadIdx.x] = a;
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (threadIdx.x < off) s[threadIdx.x] += s[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *U = 0.5 * s[0];
}

static void energy_forces_impl(const se1p_opts* o, cudaStream_t st, const double* x, const double* q, int64_t N,
                               const double L[3], double xi, double rc, int M, int P, double eta, double s0,
                               double sf, int n_local, double* U_out, double* phi_out, double* F_out) {
  if (!x || !q || !U_out || !F_out || !L) throw Error{1, "null pointer"};
  if (N < 1 || N > (int64_t)2000000000) throw Error{1, "N out of range"};
  DevState& ds = dev_state();
  WsOrder ws_order(ds, st);
  const bool host_io = o && o->host_io;
  grow(ds.ef, ds.ef_cap, 17 * N + 1);
  double *dx = ds.ef, *dq = dx + 3 * N, *pk = dq + N, *ek = pk + N, *pr = ek + 3 * N, *er = pr + N;
  double *dphi = er + 3 * N, *dF = dphi + N, *dU = dF + 3 * N;
  if (host_io) {
    SE1P_CUDA_TRY(cudaMemcpyAsync(dx, x, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    SE1P_CUDA_TRY(cudaMemcpyAsync(dq, q, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  } else {
    dx = const_cast<double*>(x);
    dq = const_cast<double*>(q);
    dphi = phi_out;
    dF = F_out;
    dU = U_out;
  }
  se1p_opts od{};
  if (o) od = *o;
  od.host_io = 0;
  od.sync = 0;
  kspace_impl(&od, st, dx, dq, N, L, xi, M, P, eta, s0, sf, n_local, pk, ek);
  od.skip_checks = 1;
  od.reserved[4] = od.reserved[5] = 0;   // the whole real-space sum
  real_impl(&od, st, dx, dq, N, L, xi, rc, pr, er);
  k_combine_forces<<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(dq, pk, ek, pr, er, N, dphi, dF);
  SE1P_LAUNCH_CHECK();
  k_energy<<<1, 1024, 0, st>>>(dq, pk, pr, N, dU);
  SE1P_LAUNCH_CHECK();
  if (host_io) {
    SE1P_CUDA_TRY(cudaMemcpyAsync(U_out, dU, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (phi_out) SE1P_CUDA_TRY(cudaMemcpyAsync(phi_out, dphi, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    SE1P_CUDA_TRY(cudaMemcpyAsync(F_out, dF, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, st));
  }
  if (!o || o->sync || host_io) {
    SE1P_CUDA_TRY(cudaStreamSynchronize(st));
    int kerr = 0;
    SE1P_CUDA_TRY(cudaMemcpy(&kerr, ds.w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost));
    if (kerr) throw Error{6, "sweep kernel internal bounds check failed (code " + std::to_string(kerr) + ")"};
  }
  SE1P_CUDA_TRY(cudaGetLastError());
}

template <typename F>
static int guarded(F&& f) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  try {
    f();
    return SE1P_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SE1P_ECUDA;
  }
}

}  // namespace se1p

using namespace se1p;

extern "C" {

int se1p_kspace(const double* x, const double* q, int64_t N, const double L[3], double xi, int M, int P, double eta,
                double s0, double sf, int n_local, double* phi_out) {
  return guarded([&] {
    se1p_opts o{};
    o.sync = 1;
    kspace_impl(&o, 0, x, q, N, L, xi, M, P, eta, s0, sf, n_local, phi_out);
  });
}

int se1p_kspace_ex(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                   const double L[3], double xi, int M, int P, double eta, double s0, double sf, int n_local,
                   double* phi_out) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    kspace_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, M, P, eta, s0, sf, n_local, phi_out);
  });
}

int se1p_real(const double* x, const double* q, int64_t N, const double L[3], double xi, double rc, double* phi_out) {
  return guarded([&] {
    se1p_opts o{};
    o.sync = 1;
    real_impl(&o, 0, x, q, N, L, xi, rc, phi_out);
  });
}

int se1p_real_ex(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N, const double L[3],
                 double xi, double rc, double* phi_out) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    real_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, rc, phi_out);
  });
}

int se1p_kspace3p_ex(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                     const double L[3], double xi, int M, int P, double eta, double* phi_out) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    kspace3p_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, M, P, eta, phi_out);
  });
}

int se1p_kspace_tiers_ex(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                         const double L[3], double xi, int M, int P, double eta, double s0, int n_local,
                         const int* S_modes, double* phi_out) {
  return guarded([&] {
    if (!S_modes) throw Error{1, "null pointer"};
    if (n_local < 0) throw Error{1, "the tiers entry needs an explicit n_local (the length of S_modes)"};
    se1p_opts o{};
    if (opts) o = *opts;
    kspace_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, M, P, eta, s0, -1.0, n_local, phi_out, nullptr, S_modes);
  });
}

int se1p_kspace_field_ex(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                         const double L[3], double xi, int M, int P, double eta, double s0, double sf, int n_local,
                         double* phi_out, double* field_out) {
  return guarded([&] {
    if (!field_out) throw Error{1, "null pointer"};
    se1p_opts o{};
    if (opts) o = *opts;
    kspace_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, M, P, eta, s0, sf, n_local, phi_out, field_out);
  });
}

int se1p_real_field_ex(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                       const double L[3], double xi, double rc, double* phi_out, double* field_out) {
  return guarded([&] {
    if (!field_out) throw Error{1, "null pointer"};
    se1p_opts o{};
    if (opts) o = *opts;
    real_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, rc, phi_out, field_out);
  });
}

int se1p_energy_forces(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                       const double L[3], double xi, double rc, int M, int P, double eta, double s0, double sf,
                       int n_local, double* U_out, double* phi_out, double* F_out) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    energy_forces_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, rc, M, P, eta, s0, sf, n_local, U_out, phi_out,
                       F_out);
  });
}

int se1p_kspace_slab_forward(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                             const double L[3], double xi, int M, int P, double eta, double s0, double sf,
                             int n_local, int x_lo, int x_hi, const int* plane_order, void* planes_out) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    slab_forward_impl(&o, (cudaStream_t)stream, x, q, N, L, xi, M, P, eta, s0, sf, n_local, x_lo, x_hi, plane_order,
                      planes_out);
  });
}

int se1p_kspace_modes(const se1p_opts* opts, void* stream, const double L[3], double xi, int M, int P, double eta,
                      double s0, double sf, int n_local, int n_own, const int* plane_ids, int nslab,
                      const int* slab_lo, void* planes) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    modes_impl(&o, (cudaStream_t)stream, L, xi, M, P, eta, s0, sf, n_local, n_own, plane_ids, nslab, slab_lo, planes);
  });
}

int se1p_kspace_slab_backward(const se1p_opts* opts, void* stream, int64_t N, const double L[3], double xi, int M,
                              int P, double eta, double s0, double sf, int n_local, int x_lo, int x_hi,
                              const int* plane_order, const void* planes_in, double* phi_partial) {
  return guarded([&] {
    se1p_opts o{};
    if (opts) o = *opts;
    slab_backward_impl(&o, (cudaStream_t)stream, N, L, xi, M, P, eta, s0, sf, n_local, x_lo, x_hi, plane_order,
                       planes_in, phi_partial);
  });
}

int se1p_plan_query(const se1p_opts* opts, const double L[3], double xi, int M, int P, double eta, double s0,
                    double sf, int n_local, se1p_plan_info* info) {
  return guarded([&] {
    const KParams prm = resolve(opts, L, xi, M, P, eta, s0, sf, n_local);
    KPlan* pl = kplan_get(prm, 0);
    fill_info(*pl, info);
  });
}

int se1p_plan_from_tol(const double L[3], double Q, double xi, double tol, se1p_tol_plan* out) {
  return guarded([&] { plan_from_tol(L, Q, xi, tol, out); });
}

int se1p_real_table(double xi, double rc, int* degree, int* intervals, double* coeffs, int capacity) {
  return guarded([&] {
    if (!degree || !intervals) throw Error{1, "null pointer"};
    if (!(xi > 0) || !(rc > 0)) throw Error{1, "xi, rc must be > 0"};
    const std::vector<double> t = real_table_host(xi, rc, *degree, *intervals);
    if (coeffs && capacity >= (int)t.size()) std::copy(t.begin(), t.end(), coeffs);
  });
}

int se1p_last_stage_times(double* ms, int max_stages) {
  int n = std::min(max_stages, g_nstages);
  for (int i = 0; i < n; ++i) ms[i] = g_stage_ms[i];
  return n;
}

int se1p_last_launch_count(void) { return g_launches; }

int se1p_debug_copy(int which, double* host_dst, int64_t count) {
  return guarded([&] {
    KWork& w = dev_state().w;
    if (!host_dst || count < 0) throw Error{1, "bad arguments"};
    if (which == 0) {
      if (count > w.grid_cap) throw Error{1, "grid buffer smaller than requested"};
      SE1P_CUDA_TRY(cudaMemcpy(host_dst, w.grid, sizeof(double) * count, cudaMemcpyDeviceToHost));
    } else if (which == 1) {
      if (count > 2 * w.planes_cap) throw Error{1, "plane buffer smaller than requested"};
      SE1P_CUDA_TRY(cudaMemcpy(host_dst, w.planes, sizeof(double) * count, cudaMemcpyDeviceToHost));
    } else {
      throw Error{1, "unknown buffer"};
    }
  });
}

}  // extern "C"

namespace se1p {
// Frees everything the library holds on the CURRENT device d: its plans, workspace, tables,
// streams and the CUDA graphs (which bake the freed pointers).  Caller holds g_mu.
static void release_device(int d) {
  kplan_release_all(d);
  DevState& ds = g_dev[d & 63];
  KWork& w = ds.w;
  for (void* p : {(void*)w.xs, (void*)w.perm, (void*)w.keys, (void*)w.bin_start, (void*)w.scratch,
                  (void*)w.grid, (void*)w.planes, (void*)w.T, (void*)w.red, (void*)w.flag, (void*)ds.dx,
                  (void*)w.gpart, (void*)w.rec, (void*)w.s4, (void*)ds.dmap, (void*)w.grid3, (void*)ds.sel,
                  (void*)ds.idmap, (void*)ds.xsel, (void*)w.over, (void*)w.items, (void*)ds.ef})
    dev_free(p);
  real_release_tables(d);
  if (w.side) cudaStreamDestroy(w.side);
  if (w.ev_fork) cudaEventDestroy(w.ev_fork);
  if (w.ev_join) cudaEventDestroy(w.ev_join);
  if (w.side2) cudaStreamDestroy(w.side2);
  if (w.ev_join2) cudaEventDestroy(w.ev_join2);
  if (ds.ws_done) cudaEventDestroy(ds.ws_done);
  ds = DevState{};
  g_dev_used &= ~(1ull << (d & 63));
  for (auto& g : g_graphs) cudaGraphExecDestroy(g.exec);
  g_graphs.clear();
  ++g_ws_generation;
}
}  // namespace se1p

extern "C" {

void se1p_release(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  int d = 0;
  cudaGetDevice(&d);
  release_device(d);
}

int se1p_set_allocator(void* (*alloc)(size_t, void*), void (*release)(void*, void*), void* ctx) {
  if ((alloc == nullptr) != (release == nullptr)) {
    g_err = "se1p_set_allocator: alloc and release must both be set or both be null";
    return 1;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  // everything allocated so far, on every device, goes back through the allocator that made it
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < 64; ++d)
    if ((g_dev_used >> d) & 1) {
      cudaSetDevice(d);
      release_device(d);
    }
  cudaSetDevice(cur);
  g_alloc_fn = alloc;
  g_release_fn = release;
  g_alloc_ctx = ctx;
  return 0;
}

const char* se1p_last_error(void) { return g_err.c_str(); }

const char* se1p_version(void) { return "se1p-b200 0.1 (sm_100a, fp64)"; }

}  // extern "C"
