// tiles.cu -- gridding (Alg. 1 step 2, Eq. (spread_1p)) and gather (Alg. 1 step 6,
// Eq. (se1p_complete_discretized)) as output-stationary tile contractions on the
// FP64 tensor pipe (mma.sync f64 -> SASS DMMA).  See tiles.cuh.
//
// Fast Gaussian Gridding: k_records stores per sorted particle only the stencil
// starts, q and per axis the two FGG factors A = e^{-alpha d0^2}, E = e^{-2 alpha h d0} (d0 the
// offset of the first stencil node); the window weight of stencil node t is A E^t f1[t],
// f1[t] = e^{-alpha h^2 t^2}.  Tiles move these 80-byte records and expand the weights they need
// in shared memory -- multiplications instead of exponentials.
//
// One CTA per tile X0..X0+15 x Y0..Y0+15 x Z0..Z0+TZ-1 (periodic in z), 25 warps:
//   producer (1 warp): walks the tile's candidate runs (bins: x band of 4 cells, z cell, y cell;
//     a run = one x band, one z cell, the tile's y range) z-major, 32 runs at a time: a warp scan
//     places them in the batch stream and every lane moves its run's records with one bulk copy
//     (cp.async.bulk, SASS UBLKCP) into a ring of NB batches of BM records (mbarrier `raw`,
//     transaction bytes).
//   expanders (kEW warps): per batch, the tile windows wx[16], wy[16], wz[TZ] of every particle
//     (zero outside the stencil, z wraps periodically, gridding folds q into wx) in 16-entry
//     segments (one FGG recurrence each, started by binary powering of E), and per particle the
//     mask of consumer warps its stencil meets with its z-block mask; then `full`.  Gather: they
//     also reduce finished batches' per-warp partials into the slots (lag 2, then `freeb`).
//   consumers (16 warps): warp w owns the 4 x 4 column block (4 (w&3), 4 (w>>2)) over all TZ
//     nodes; per batch it lists the particles whose mask names it (order preserving) and runs
//       gridding  C[16 cols x 8 z]        += A[16 cols x 16 particles] B[16 particles x 8 z]
//                 A = (q wx) wy, B = wz                                   (m16n8k16)
//       gather    T[16 particles x 8 cols] = A[16 particles x 8 z] (wz) B[8 z x 8 cols] (H~)
//                 per col half, then phi_p += sum_cols wx wy T             (m16n8k8)
//     skipping 8-node z blocks no particle of the k-step reaches; then arrives on `empty`.
//   Field modes (FM, gather only): 1 phi and the x, y column moments, 2 d/dz through the
//   z-derivative window (two passes), 3 all four in one pass (build knob).
// Device-side bounds checks set bits of an error word (1 runs, 2 lists, 4 slots, 8 slot map).
// No floating-point atomics: gridding writes its tile once; the gather writes one partial per
// (particle, tile) into a fixed slot and k_gather_finish sums the slots in a fixed order, so
// results are bitwise reproducible.
#include <cstdint>
#include <cstdlib>

#include "tiles.cuh"

namespace se1p {

constexpr int kCW = 16;                          // consumer warps
// expander warps: 8, or 4 for the field gather (32-particle batches, more consumer registers).
// ptxas budgets registers for the thread count rounded up to 4 warps: 25 warps -> 72 registers,
// 24 -> 80, 20 -> 96.  Measured (C5): 7/3 and 6/2 expander warps are 8-20% slower, field 5-8 equal.
#ifndef SE1P_EXP_WARPS
#define SE1P_EXP_WARPS 8
#endif
// z extent of the gather's DMMA blocks: 4 (m16n8k4), 8 (m16n8k8) or 16 (m16n8k16)
#ifndef SE1P_GATHER_KZ
#define SE1P_GATHER_KZ 8
#endif
#ifndef SE1P_GATHER_KZ_FIELD
#define SE1P_GATHER_KZ_FIELD 4
#endif
#ifndef SE1P_FIELD_ONE_PASS
#define SE1P_FIELD_ONE_PASS 0
#endif
#ifndef SE1P_EXP_WARPS_FIELD
#define SE1P_EXP_WARPS_FIELD 4
#endif
// Field modes of the gather (FM): 0 potential; the field E = -grad phi in two passes over the same
// tiles, 1: phi, d/dx, d/dy (x, y window derivatives in the epilogue) and 2: d/dz (the expanders
// write the z-derivative window 2 alpha (node - z_p) wz in place of wz); 3: all four in one pass
// (a second z window and accumulator set).
__host__ __device__ constexpr int n_exp_warps(int fm) { return fm == 3 ? SE1P_EXP_WARPS_FIELD : SE1P_EXP_WARPS; }
__host__ __device__ constexpr int n_threads(int fm) { return (kCW + 1 + n_exp_warps(fm)) * 32; }
__host__ __device__ constexpr int fm_outputs(int fm) { return fm == 0 ? 1 : (fm == 1 ? 3 : (fm == 2 ? 1 : 4)); }
constexpr int kMaxNB = 6;
// doubles per compact record: {s4, q, index, (A, E) per axis} (80 B); the field gather adds the
// particle position (112 B)
__host__ __device__ constexpr int rec_len(int field) { return field ? 14 : 10; }
constexpr int kMaxP = 64;
constexpr int kEntZ = 16;                        // gridding list entry: smem row offset (16 bits), z mask

// Expanded row: 16-entry window segments wx, wy, wz[0:16), wz[16:32) at offsets 0, 17, 34, 51
// (17 apart: when 8 particles x 4 segments are written by one warp, the 32 lanes fall into
// distinct bank pairs); row stride = 4 (mod 16) doubles, so the 4 particles of a consumer
// k-step start 4 banks apart.
// The field gather appends the z-derivative window wz'[j] = 2 alpha (node - z_p) wz[j] at 68 and 85.
__host__ __device__ constexpr int exp_stride(int TZ, int fm = 0) {
  return fm == 3 ? (TZ == 32 ? 116 : 68) : (TZ == 32 ? 68 : 52);
}
constexpr int kEX = 0, kEY = 17, kEZ = 34;
__host__ __device__ constexpr int zoff(int j) { return kEZ + j + (j >= 16 ? 1 : 0); }   // wz[j]
__host__ __device__ constexpr int zoffd(int TZ, int j) { return (TZ == 32 ? 68 : 51) + j + (j >= 16 ? 1 : 0); }

struct TileArgs {
  KDev dv;
  const double* rec;      // compact records [N][rec_len]
  const int* bin_start;
  const double* f1;
  double* grid;
  double* gpart;
  int ntz, nty, tx_lo;   // launched tiles: tx in [tx_lo, tx_lo + gridDim/(nty ntz))
  int order;             // 1: the launch's first and last x columns and y rows (light edge tiles) go last
  int BM, NB;
};

struct TileSmem {
  int off_lists, off_rel, off_acc, off_raw, off_exp, total;
};

__host__ __device__ inline TileSmem tile_smem(int BM, int NB, int TZ, bool gather, int fm = 0) {
  TileSmem s;
  int o = 4 * kMaxNB * 8 + kMaxNB * 4 + kMaxP * 8;   // barriers, counts, f1
  o = (o + 15) & ~15;
  s.off_lists = o;
  o += kCW * (BM + 32) * 4;
  o = (o + 15) & ~15;
  s.off_rel = o;   // per batch particle: consumer-warp mask (16 bits) | z-block mask << 16
  o += NB * BM * 4;
  o = (o + 15) & ~15;
  s.off_acc = o;
  if (gather) o += NB * BM * (kCW + 1) * fm_outputs(fm) * 8;
  o = (o + 127) & ~127;
  s.off_raw = o;
  o += NB * BM * rec_len(fm) * 8;
  o = (o + 127) & ~127;
  s.off_exp = o;
  o += NB * (BM + 1) * exp_stride(TZ, fm) * 8;
  s.total = o;
  return s;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// SE1P_MBAR_WAIT: 0 try_wait (the hardware may suspend the warp until the phase flips),
// 1 test_wait spin (no suspension), 2 try_wait with a suspend-time hint (ns)
#ifndef SE1P_MBAR_WAIT
#define SE1P_MBAR_WAIT 0
#endif
#ifndef SE1P_MBAR_HINT_NS
#define SE1P_MBAR_HINT_NS 64
#endif
__device__ __forceinline__ bool mbar_test_wait(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity), "n"(SE1P_MBAR_HINT_NS)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
#if SE1P_MBAR_WAIT == 1
  while (!mbar_test_wait(b, parity)) {
  }
#elif SE1P_MBAR_WAIT == 2
  while (!mbar_try_wait_hint(b, parity)) {
  }
#else
  while (!mbar_try_wait(b, parity)) {
  }
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// bits of the 8-node z blocks covering tile offsets [lo, hi), hi > lo
__device__ __forceinline__ int zbits(int lo, int hi) { return ((1 << ((hi + 7) >> 3)) - 1) & ~((1 << (lo >> 3)) - 1); }

// the same for 4-node blocks (the gather's m16n8k4 granularity)
__device__ __forceinline__ int zbits4(int lo, int hi) { return ((1 << ((hi + 3) >> 2)) - 1) & ~((1 << (lo >> 2)) - 1); }

// z tiles (extent TZ) hit by the stencil nodes a, a+1, ..., a+P-1 (mod M), a in [0,M): first the
// tiles of [a, min(a+P,M)), then those of the wrapped part [0, a+P-M) not already listed.
// zslot gives the canonical position of tile tz (-1: not hit); k_gather_finish walks the same list.
__device__ __forceinline__ int zslot(int a, int P, int M, int TZ, int tz) {
  const int t1a = a / TZ, t1b = (min(a + P, M) - 1) / TZ;
  if (tz >= t1a && tz <= t1b) return tz - t1a;
  if (a + P > M && tz <= min((a + P - M - 1) / TZ, t1a - 1)) return (t1b - t1a + 1) + tz;
  return -1;
}
__device__ __forceinline__ int zcount(int a, int P, int M, int TZ) {
  const int t1a = a / TZ, t1b = (min(a + P, M) - 1) / TZ;
  int n = t1b - t1a + 1;
  if (a + P > M) n += min((a + P - M - 1) / TZ, t1a - 1) + 1;
  return n;
}

// 8-node z blocks of tile (Z0, TZ) met by the stencil starting at a (mod M); d = (Z0 - a) mod M.
// The stencil covers tile offsets [0, P-d) and [M-d, M-d+P), intersected with [0, min(TZ, M-Z0)).
__device__ __forceinline__ int zmask_of(int d, int P, int M, int jmax) {
  int zm = 0;
  if (d < P) zm |= zbits(0, min(P - d, jmax));
  const int lo2 = M - d;
  if (lo2 < jmax) zm |= zbits(lo2, min(lo2 + P, jmax));
  return zm;
}
__device__ __forceinline__ int zbits16(int lo, int hi) { return ((1 << ((hi + 15) >> 4)) - 1) & ~((1 << (lo >> 4)) - 1); }
__device__ __forceinline__ int zmask16_of(int d, int P, int M, int jmax) {
  int zm = 0;
  if (d < P) zm |= zbits16(0, min(P - d, jmax));
  const int lo2 = M - d;
  if (lo2 < jmax) zm |= zbits16(lo2, min(lo2 + P, jmax));
  return zm;
}
__device__ __forceinline__ int zmask4_of(int d, int P, int M, int jmax) {
  int zm = 0;
  if (d < P) zm |= zbits4(0, min(P - d, jmax));
  const int lo2 = M - d;
  if (lo2 < jmax) zm |= zbits4(lo2, min(lo2 + P, jmax));
  return zm;
}

// FIELD (gather only): also the field E = -grad phi at the particles -- the gradient of the
// gather (Eq. (force_se1p)): d/dx_p e^{-alpha (node - x_p)^2} = 2 alpha (node - x_p) w.
template <int TZ, bool GATHER, int FM = 0>
__global__ void __launch_bounds__(n_threads(FM), 1) k_tiles(const TileArgs A) {
  constexpr int NZB = TZ / 8;
  constexpr bool FIELD = FM == 3;     // one-pass field: second z window and accumulators
  constexpr int RSE = exp_stride(TZ, FM);
  constexpr int kEW = n_exp_warps(FM), kThreads = n_threads(FM), kRec = rec_len(FM);
  constexpr int NC = fm_outputs(FM);  // gather outputs per particle of this pass
  constexpr int NCT = FM ? 4 : 1;     // values per gather slot: phi (and d/dx, d/dy, d/dz)
  constexpr int COFF = FM == 2 ? 3 : 0;   // first slot value this pass writes
  constexpr int KZ = FIELD ? SE1P_GATHER_KZ_FIELD : SE1P_GATHER_KZ;   // gather DMMA z extent
  extern __shared__ __align__(128) unsigned char smem[];
  const KDev& dv = A.dv;
  const int BM = A.BM, NB = A.NB, P = dv.P, M = dv.M, Mt = dv.Mt;
  const TileSmem L = tile_smem(BM, NB, TZ, GATHER, FM);
  uint64_t* rawb = reinterpret_cast<uint64_t*>(smem);
  uint64_t* full = rawb + kMaxNB;
  uint64_t* empty = full + kMaxNB;
  uint64_t* freeb = empty + kMaxNB;   // gather: batch reduced, buffers reusable
  int* cnt = reinterpret_cast<int*>(freeb + kMaxNB);
  double* f1 = reinterpret_cast<double*>(cnt + kMaxNB);
  int* lists = reinterpret_cast<int*>(smem + L.off_lists);
  int* relm = reinterpret_cast<int*>(smem + L.off_rel);
  double* acc = reinterpret_cast<double*>(smem + L.off_acc);
  double* raws = reinterpret_cast<double*>(smem + L.off_raw);
  double* exps = reinterpret_cast<double*>(smem + L.off_exp);
  const int ES = (BM + 1) * RSE;   // doubles per expanded batch (row BM: all zero)

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int tz = blockIdx.x % A.ntz, t2 = blockIdx.x / A.ntz;
  int ty = t2 % A.nty, tx = t2 / A.nty;
  if (A.order) {   // interior first: i -> i+1 for i < n-2, then 0 and n-1 (edge tiles fill the tail)
    const int ntx = gridDim.x / (A.ntz * A.nty);
    auto perm = [](int i, int n) { return n < 3 ? i : (i < n - 2 ? i + 1 : (i == n - 2 ? 0 : n - 1)); };
    tx = perm(tx, ntx);
    ty = perm(ty, A.nty);
  }
  tx += A.tx_lo;
  const int X0 = tx * kTXY, Y0 = ty * kTXY, Z0 = tz * TZ;
  const int jmax = min(TZ, M - Z0);

  if (tid == 0) {
    for (int b = 0; b < kMaxNB; ++b) {
      mbar_init(&rawb[b], 1);
      mbar_init(&full[b], kEW);
      mbar_init(&empty[b], kCW);
      mbar_init(&freeb[b], kEW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = tid; k < P; k += kThreads) f1[k] = A.f1[k];
  for (int b = 0; b < NB; ++b)
    for (int k = tid; k < RSE; k += kThreads) exps[b * ES + BM * RSE + k] = 0.0;
  if (GATHER)
    for (int k = tid; k < NB * BM * (kCW + 1) * NC; k += kThreads) acc[k] = 0.0;
  __syncthreads();

// gather: sum the per-warp partials of batch buffer b into the particles' slots (expander warps)
auto reduce = [&](int b, int rt) {
    const int c = cnt[b];
    const double* rb = raws + b * BM * kRec;
    for (int p = rt; p < c; p += 32 * kEW) {
      const int4 s = *reinterpret_cast<const int4*>(rb + p * kRec);
      double* ap = acc + (b * BM + p) * (kCW + 1) * NC;
      const bool hx = s.x <= X0 + kTXY - 1 && s.x + P - 1 >= X0 && s.y <= Y0 + kTXY - 1 && s.y + P - 1 >= Y0;
      const int sz = hx ? zslot(s.w, P, M, TZ, tz) : -1;
      if (sz >= 0) {
        const int sx = tx - fdiv(s.x, kTXY), sy = ty - fdiv(s.y, kTXY);
        const int64_t i = __double_as_longlong(rb[p * kRec + 3]);   // sorted index (k_records)
        if (sx < 0 || sx >= dv.nsxy || sy < 0 || sy >= dv.nsxy || sz >= dv.nsz || i < 0 || i >= dv.N)
          atomicOr(dv.err, 4);                                          // bounds check: slot map
        double sum[NC];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          sum[cc] = 0.0;
#pragma unroll
          for (int v = 0; v < kCW; ++v) {
            sum[cc] += ap[v * NC + cc];
            ap[v * NC + cc] = 0.0;
          }
        }
        if (FM == 1) {   // column moments -> d/dx, d/dy: 2 alpha (h S + delta phi)
          const double ta = 2.0 * dv.alpha;
          const double dxp = ((double)X0 - 0.5 * P) * dv.h - rb[p * kRec + 10];
          const double dyp = ((double)Y0 - 0.5 * P) * dv.h - rb[p * kRec + 11];
          sum[1] = ta * fma(dv.h, sum[1], dxp * sum[0]);
          sum[2] = ta * fma(dv.h, sum[2], dyp * sum[0]);
        }
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
          A.gpart[(int64_t)(((sx * dv.nsxy + sy) * dv.nsz + sz) * NCT + COFF + cc) * dv.N + i] = sum[cc];
      } else if (hx) {
        for (int v = 0; v < kCW * NC; ++v)
          if (ap[v] != 0.0) atomicOr(dv.err, 8);   // consumer listed a particle the slot map lacks
      }
    }
  };


  if (w == kCW) {
    // ================================================================ producer
    int k = 0, fill = 0, b = 0;
    bool have = false;
    auto acquire = [&]() {
      b = k % NB;
      if (k >= NB) mbar_wait(GATHER ? &freeb[b] : &empty[b], (unsigned)(((k - NB) / NB) & 1));
      have = true;
    };
    auto publish = [&](int c) {
      __threadfence_block();
      __syncwarp();
      if (lane == 0) {
        cnt[b] = c;
        mbar_arrive(&rawb[b]);
      }
      __syncwarp();
      ++k;
      fill = 0;
      have = false;
    };

    // Candidate runs: z cells czs .. czs+span-1 (unwrapped, z-major), x bands bx0..bx1, and in
    // each the contiguous y-cell range cy0..cy1 of the sorted order (bins: x band, z, y).
    const int bx0 = max(0, fdiv(X0 - P, kBin)), bx1 = min(dv.nbx - 1, fdiv(X0 + kTXY - 2, kBin));
    const int cy0 = max(0, Y0 - P), cy1 = min(dv.Mfree - 1, Y0 + kTXY - 2);
    const int nbx = bx1 - bx0 + 1;
    int czs = Z0 - P / 2 - 1, span = TZ + P + 2;   // cells whose stencils may reach the tile
    if (span >= M) {
      czs = 0;
      span = M;
    }
    const int npc = (cy1 >= cy0 && nbx > 0) ? span * nbx : 0;
    auto load_run = [&](int q, int& s, int& e) {
      s = e = 0;
      if (q < npc) {
        const int zz = q / nbx, bx = bx0 + (q - zz * nbx);
        const int row = (bx * M + pmod(czs + zz, M)) * dv.Mfree;
        s = A.bin_start[row + cy0];
        e = A.bin_start[row + cy1 + 1];
      }
    };
    // Runs are issued 32 at a time: lane l owns run q0 + l; a warp scan places the runs in the
    // batch stream (batch k holds stream positions [k BM, (k+1) BM)) and every lane bulk-copies
    // the part of its run that falls into the open batch, in parallel.
    int sN, eN;
    load_run(lane, sN, eN);
    int pos = 0;   // stream position of the next record (= k BM + fill)
    for (int q0 = 0; q0 < npc; q0 += 32) {
      const int sC = sN, nC = eN - sN;
      if (nC < 0 || sC < 0 || (int64_t)sC + nC > dv.N) atomicOr(dv.err, 1);   // bounds check: run outside [0, N)
      load_run(q0 + 32 + lane, sN, eN);   // prefetch the next 32 runs
      int incl = nC;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      const int rlo = pos + incl - nC, rhi = pos + incl;   // this lane's run in stream positions
      const int end = pos + tot;
      while (pos < end) {
        if (!have) acquire();
        const int blo = k * BM, bhi = blo + BM;
        const int lo = max(rlo, blo), hi = min(rhi, bhi);
        if (hi > lo && !(dv.dbg & 16)) {
          const unsigned bytes = (unsigned)((hi - lo) * kRec * 8);
          mbar_expect_tx(&rawb[b], bytes);
          bulk_g2s(raws + (b * BM + (lo - blo)) * kRec, A.rec + (int64_t)(sC + (lo - rlo)) * kRec, bytes, &rawb[b]);
        }
        const int upto = min(end, bhi);
        fill = upto - blo;
        pos = upto;
        if (fill == BM) publish(BM);
      }
    }
    if (fill > 0) publish(fill);
    acquire();
    publish(-1);   // end marker
    return;
  }

  if (w > kCW) {
    // ================================================================ expanders
    // Windows are cut into 16-entry segments: x, y and TZ/16 z segments per particle.  Lane l of
    // an expander warp takes segment kind l & 3 of particle (group base) + (l >> 2), so one warp
    // writes 8 particles x 4 segments with conflict-free stores.  Segment entry i holds stencil
    // node t: free axes t = i + (X0 - jx0); z t = (i + 16 s + (Z0 - a)) mod M.  Inside the
    // stencil the value is A E^t f1[t]: the start power by binary powering, then E^(t+1) = E^t E.
    // Gather: after expanding batch j the expanders reduce batch j-2 (once the consumers released
    // it) and free its buffers for the producer.
    constexpr int NSEG = 2 + TZ / 16;
    const int ew = w - (kCW + 1), kind = lane & 3;
    auto reduce_batch = [&](int j) {
      const int bj = j % NB;
      mbar_wait(&empty[bj], (unsigned)((j / NB) & 1));
      if (!(dv.dbg & 4)) reduce(bj, tid - (kCW + 1) * 32);
      __syncwarp();
      if (lane == 0) mbar_arrive(&freeb[bj]);
    };
    for (int b = 0, ph = 0, j = 0;; b = (b + 1 == NB) ? 0 : b + 1, ph ^= (b == 0), ++j) {
      mbar_wait(&rawb[b], (unsigned)ph);
      const int cn = cnt[b];
      if (cn > 0 && kind < NSEG && !((dv.dbg & 8) && kind > 0)) {
        const double* rb = raws + b * BM * kRec;
        double* eb = exps + b * ES;
        for (int p = 8 * ew + (lane >> 2); p < cn; p += 8 * kEW) {
          const double* r = rb + p * kRec;
          const int4 s = *reinterpret_cast<const int4*>(r);
          if (kind == 0) {
            // which consumer warps (4 x 4 column blocks of 4 x 4 columns) the stencil meets, and its
            // z blocks: computed once here instead of by each of the 16 consumer warps
            const int bx0 = max(fdiv(s.x - X0, 4), 0), bx1 = min(fdiv(s.x - X0 + P - 1, 4), 3);
            const int by0 = max(fdiv(s.y - Y0, 4), 0), by1 = min(fdiv(s.y - Y0 + P - 1, 4), 3);
            int d = Z0 - s.w;
            if (d < 0) d += M;
            const int zm = !GATHER ? zmask_of(d, P, M, jmax)
                                   : (KZ == 4 ? zmask4_of(d, P, M, jmax)
                                              : (KZ == 16 ? zmask16_of(d, P, M, jmax) : zmask_of(d, P, M, jmax)));
            int wm = 0;
            if (zm != 0 && bx0 <= bx1 && by0 <= by1) {
              const int xb = ((1 << (bx1 + 1)) - 1) & ~((1 << bx0) - 1);
              for (int by = by0; by <= by1; ++by) wm |= xb << (4 * by);
            }
            relm[b * BM + p] = wm | (zm << 16);
          }
          const int ax = kind < 2 ? kind : 2;
          const double A0 = (ax == 0 && !GATHER) ? r[4] * r[2] : r[4 + 2 * ax];   // gridding: q in wx
          const double E = r[5 + 2 * ax];
          int t, lim, Mw;
          double* o = eb + p * RSE;
          double* od = nullptr;   // field: z-derivative window 2 alpha (node - z_p) wz
          if (ax < 2) {
            t = ax == 0 ? X0 - s.x : Y0 - s.y;
            lim = 16;
            Mw = 1 << 30;
            o += ax == 0 ? kEX : kEY;
          } else {
            const int i0 = 16 * (kind - 2);
            t = Z0 + i0 - s.w;
            if (t < 0) t += M;
            if (t >= M) t -= M;
            lim = jmax - i0;
            Mw = M;
            if (FIELD) od = o + zoffd(TZ, i0);
            o += zoff(i0);
          }
          // two interleaved chains of 8 entries: entries 0..7 from node t, 8..15 from node t + 8
          int tc[2] = {t, t + 8};
          if (tc[1] >= Mw) tc[1] -= Mw;
          double g[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int tt = tc[c];
            double gg = A0, e = E;
#pragma unroll
            for (int k = 0; k < 6; ++k) {   // binary powering: A E^tt, tt < P <= 64
              if ((tt >> k) & 1) gg *= e;
              e *= e;
            }
            g[c] = (tt > 0 && tt < P) ? gg : A0;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int tt = tc[c];
              double v = 0.0;
              if (tt >= 0 && tt < P && 8 * c + i < lim) {
                v = g[c] * f1[tt];
                g[c] *= E;
              }
              if (FM == 2 && ax == 2)   // pass 2: the z-derivative window in place of wz
                o[8 * c + i] = 2.0 * dv.alpha * ((double)(s.z + tt) * dv.h - r[12]) * v;
              else
                o[8 * c + i] = v;
              if (FIELD && od) od[8 * c + i] = 2.0 * dv.alpha * ((double)(s.z + tt) * dv.h - r[12]) * v;
              if (++tc[c] == Mw) {   // periodic wrap: the stencil restarts at node 0
                tc[c] = 0;
                g[c] = A0;
              }
            }
          }
        }
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);
      if (GATHER) {
        if (j >= 2) reduce_batch(j - 2);
        if (cn < 0 && j >= 1) reduce_batch(j - 1);
      }
      if (cn < 0) break;
    }
    return;
  }

  // ================================================================ consumers
  // list entry per relevant particle: p | zmask << 8 (8-node z blocks of the tile it meets)
  const int gid = lane >> 2, tig = lane & 3;
  const int X0b = X0 + 4 * (w & 3), Y0b = Y0 + 4 * (w >> 2);
  const int xo = 4 * (w & 3), yo = 4 * (w >> 2);   // warp block inside the tile windows
  int* wl = lists + w * (BM + 32);
  const int dummy = BM;

  // gridding accumulators: C[16 cols x 8 z] per 8-node block; col r -> (r & 3, r >> 2) of the block
  double c[GATHER ? 1 : NZB][4];
  // gather operands: H~[8 z x 8 cols] per (z block, col half); col n of half h -> (n & 3, (n >> 2) + 2h)
  double hB[GATHER ? NZB : 1][2][2];
  if (!GATHER) {
#pragma unroll
    for (int zb = 0; zb < NZB; ++zb) c[zb][0] = c[zb][1] = c[zb][2] = c[zb][3] = 0.0;
  } else {
    const int x = X0b + (gid & 3);
#pragma unroll
    for (int zb = 0; zb < NZB; ++zb)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int y = Y0b + (gid >> 2) + 2 * h, z = Z0 + 8 * zb + tig + 4 * kk;
          hB[zb][h][kk] = (z < M && x < Mt && y < Mt) ? A.grid[((int64_t)x * Mt + y) * M + z] : 0.0;
        }
  }

  if (!GATHER) {
    // Gridding, batches in order.  Entries left over after the last full k-step of a batch (< 16)
    // are carried into the next batch's list (entries name their buffer), so k-steps are padded
    // only at the end of the tile; a batch is released (empty) once no carried entry refers to it.
    const int cx = xo + (gid & 3), cy = yo + (gid >> 2);
    auto ksteps = [&](int k0, int k1) {
      for (int k = k0; k < k1; k += 16) {
        int e[4], zm = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          e[j] = wl[k + tig + 4 * j];
          zm |= e[j];
        }
        zm = (zm >> kEntZ) & 0xff;
        zm |= __shfl_xor_sync(0xffffffffu, zm, 1);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 2);
        double a[8];
        const double* rz[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double* r = exps + (e[j] & 0xffff);   // the entry holds its expanded row's offset
          const double wq = r[kEX + cx];
          a[2 * j] = wq * r[kEY + cy];
          a[2 * j + 1] = wq * r[kEY + cy + 2];
          rz[j] = r + gid;
        }
#pragma unroll
        for (int zb = 0; zb < NZB; ++zb)
          if ((zm >> zb) & 1)
            dmma_16x8x16(c[zb], a, rz[0][zoff(8 * zb)], rz[1][zoff(8 * zb)], rz[2][zoff(8 * zb)], rz[3][zoff(8 * zb)]);
      }
    };
    int held = 0, bprev = -1;
    for (int b = 0, ph = 0;; b = (b + 1 == NB) ? 0 : b + 1, ph ^= (b == 0)) {
      mbar_wait(&full[b], (unsigned)ph);
      const int cn = cnt[b];
      if (cn < 0) {
        if (held > 0) {   // flush the carried entries, padded to 16
          if (lane < 16 - held) wl[held + lane] = BM * RSE;   // the all-zero row of buffer 0
          __syncwarp();
          ksteps(0, 16);
        }
        __syncwarp();
        if (lane == 0 && bprev >= 0) mbar_arrive(&empty[bprev]);
        break;
      }
      int n = held;
      for (int p0 = 0; p0 < cn; p0 += 32) {
        const int p = p0 + lane;
        const int r = p < cn ? relm[b * BM + p] : 0;   // expander-computed relevance (see above)
        const bool rel = (r >> w) & 1;
        const int e = (b * ES + p * RSE) | ((r >> 16) << kEntZ);
        const unsigned bal = __ballot_sync(0xffffffffu, rel);
        if (rel) wl[n + __popc(bal & ((1u << lane) - 1u))] = e;
        n += __popc(bal);
      }
      if (lane == 0 && n > BM + 16) atomicOr(dv.err, 2);   // bounds check: list capacity BM + 32
      __syncwarp();
      int kend = n & ~15;
      if (kend < held) {   // fewer than 16 entries and some carried: flush everything (padded)
        kend = (n + 15) & ~15;
        if (lane < kend - n) wl[n + lane] = BM * RSE;
        __syncwarp();
      }
      if (!(dv.dbg & 2)) ksteps(0, kend);
      const int rest = n > kend ? n - kend : 0;   // carry the rest (all from this batch)
      const int mv = lane < rest ? wl[kend + lane] : 0;
      __syncwarp();
      if (lane < rest) wl[lane] = mv;
      __syncwarp();
      held = rest;
      if (lane == 0 && bprev >= 0) mbar_arrive(&empty[bprev]);
      bprev = b;
    }
  } else {
  // Gather, batches in order.  As in gridding, list entries left over after the last full k-step
  // of a batch are carried into the next batch's list (an entry names its buffer: p | zmask << 8
  // | buffer << 16), so k-steps are padded only at the end of the tile; a batch is released
  // (empty -> the expanders reduce it) once no carried entry refers to it.
  int held = 0, bprev = -1;
  for (int b = 0, ph = 0;; b = (b + 1 == NB) ? 0 : b + 1, ph ^= (b == 0)) {
    mbar_wait(&full[b], (unsigned)ph);
    const int cn = cnt[b];
    // particles of the batch meeting this warp's 4 x 4 column block (order preserving)
    int n = held;
    // z blocks of KZ nodes: a 24-node window meets 6-7 4-node, 3-4 8-node or 2-3 16-node blocks
    // (89%, 77%, 60% of the issued work inside the stencil); measured, the instruction count binds,
    // not the DMMA work: at C5 KZ = 4 / 16 are 34% / 14% slower than 8 for the potential; the
    // field (twice the DMMAs per list entry) gains 5% at 4
    for (int p0 = 0; p0 < cn; p0 += 32) {
      const int p = p0 + lane;
      const int r = p < cn ? relm[b * BM + p] : 0;   // expander-computed relevance
      const bool rel = (r >> w) & 1;
      const int e = p | ((r >> 16) << 8) | (b << 16);
      const unsigned bal = __ballot_sync(0xffffffffu, rel);
      if (rel) wl[n + __popc(bal & ((1u << lane) - 1u))] = e;
      n += __popc(bal);
    }
    if (lane == 0 && n > BM + 16) atomicOr(dv.err, 2);   // bounds check: list capacity BM + 32
    __syncwarp();
    int npad = n & ~15;
    if (cn < 0 || npad < held) {   // the end, or fewer than 16 with carried ones: flush all (padded)
      npad = (n + 15) & ~15;
      if (lane < npad - n) wl[n + lane] = dummy;
      __syncwarp();
    }
    // the carried entries (< 16) all sit in the first k-step: the previous batch is released
    // right after it (at once if nothing was carried), so the ring keeps its prefetch depth
    bool pend = bprev >= 0;
    if (pend && held == 0) {
      if (lane == 0) mbar_arrive(&empty[bprev]);
      pend = false;
    }

    if (dv.dbg & 2) {
    } else {
      // T[16 particles x 8 cols] = A[16 particles x 8 z] (wz) B[8 z x 8 cols] (H~), per col half;
      // particle of row gid (gid + 8) is list entry k + gid (k + gid + 8)
      const int cx0 = xo + 2 * (tig & 1), cy0 = yo + (tig >> 1);   // this thread's cols (x +0/+1, y +0/+2)
      for (int k = 0; k < npad; k += 16) {
        const int e0 = wl[k + gid], e1 = wl[k + gid + 8];
        int zm = ((e0 | e1) >> 8) & 0xff;
        zm |= __shfl_xor_sync(0xffffffffu, zm, 4);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 8);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 16);
        const int b0 = (e0 >> 16) & 7, b1 = (e1 >> 16) & 7;
        const double* r0 = exps + b0 * ES + (e0 & 0xff) * RSE;
        const double* r1 = exps + b1 * ES + (e1 & 0xff) * RSE;
        const double* z0 = r0 + tig;
        const double* z1 = r1 + tig;
        double t0[4] = {0.0, 0.0, 0.0, 0.0}, t1[4] = {0.0, 0.0, 0.0, 0.0};
        double u0[4] = {0.0, 0.0, 0.0, 0.0}, u1[4] = {0.0, 0.0, 0.0, 0.0};   // field: wz' H~
        if (KZ == 16) {
#pragma unroll
        for (int zq = 0; zq < NZB / 2; ++zq)
          if ((zm >> zq) & 1) {
            double a[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              a[2 * i] = z0[zoff(16 * zq + 4 * i)];
              a[2 * i + 1] = z1[zoff(16 * zq + 4 * i)];
            }
            dmma_16x8x16(t0, a, hB[2 * zq][0][0], hB[2 * zq][0][1], hB[2 * zq + 1][0][0], hB[2 * zq + 1][0][1]);
            dmma_16x8x16(t1, a, hB[2 * zq][1][0], hB[2 * zq][1][1], hB[2 * zq + 1][1][0], hB[2 * zq + 1][1][1]);
            if (FIELD) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                a[2 * i] = z0[zoffd(TZ, 16 * zq + 4 * i)];
                a[2 * i + 1] = z1[zoffd(TZ, 16 * zq + 4 * i)];
              }
              dmma_16x8x16(u0, a, hB[2 * zq][0][0], hB[2 * zq][0][1], hB[2 * zq + 1][0][0], hB[2 * zq + 1][0][1]);
              dmma_16x8x16(u1, a, hB[2 * zq][1][0], hB[2 * zq][1][1], hB[2 * zq + 1][1][0], hB[2 * zq + 1][1][1]);
            }
          }
        } else if (KZ == 4) {
#pragma unroll
        for (int zb = 0; zb < NZB; ++zb)
#pragma unroll
          for (int s = 0; s < 2; ++s)
            if ((zm >> (2 * zb + s)) & 1) {
              const double a[2] = {z0[zoff(8 * zb + 4 * s)], z1[zoff(8 * zb + 4 * s)]};
              dmma_16x8x4(t0, a, hB[zb][0][s]);
              dmma_16x8x4(t1, a, hB[zb][1][s]);
              if (FIELD) {
                const double ad[2] = {z0[zoffd(TZ, 8 * zb + 4 * s)], z1[zoffd(TZ, 8 * zb + 4 * s)]};
                dmma_16x8x4(u0, ad, hB[zb][0][s]);
                dmma_16x8x4(u1, ad, hB[zb][1][s]);
              }
            }
        } else {
#pragma unroll
        for (int zb = 0; zb < NZB; ++zb) {
          if ((zm >> zb) & 1) {
            const double a[4] = {z0[zoff(8 * zb)], z1[zoff(8 * zb)], z0[zoff(8 * zb + 4)], z1[zoff(8 * zb + 4)]};
            dmma_16x8x8(t0, a, hB[zb][0][0], hB[zb][0][1]);
            dmma_16x8x8(t1, a, hB[zb][1][0], hB[zb][1][1]);
            if (FIELD) {
              const double ad[4] = {z0[zoffd(TZ, 8 * zb)], z1[zoffd(TZ, 8 * zb)], z0[zoffd(TZ, 8 * zb + 4)],
                                    z1[zoffd(TZ, 8 * zb + 4)]};
              dmma_16x8x8(u0, ad, hB[zb][0][0], hB[zb][0][1]);
              dmma_16x8x8(u1, ad, hB[zb][1][0], hB[zb][1][1]);
            }
          }
        }
        }
        // phi_p = sum_cols wx wy T; field: d/dx uses wx' = 2 alpha (node_x - x_p) wx, d/dy likewise,
        // d/dz the wz'-transformed U (the particles' positions sit in their raw records)
        double v[2][NC];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double* r = h ? r1 : r0;
          const double* tt0 = t0 + 2 * h;
          const double* tt1 = t1 + 2 * h;
          const double wx0 = r[kEX + cx0], wx1 = r[kEX + cx0 + 1], wy0 = r[kEY + cy0], wy2 = r[kEY + cy0 + 2];
          const double A0 = fma(wx0, tt0[0], wx1 * tt0[1]), A1 = fma(wx0, tt1[0], wx1 * tt1[1]);
          v[h][0] = fma(wy0, A0, wy2 * A1);
          if (FM == 1) {
            // x, y derivatives: with node - x_p = (tile column) h + delta_x, delta_x = (X0 - P/2) h - x_p
            // per particle and tile, sum (node - x_p) wx wy T = h S_x + delta_x phi; the column moments
            // S_x = sum cx wx wy T, S_y likewise go through the reduction, delta in the slot reduce
            const double cxa = (double)cx0, cya = (double)cy0;
            v[h][1] = fma(wy0, fma(cxa * wx0, tt0[0], (cxa + 1.0) * wx1 * tt0[1]),
                          wy2 * fma(cxa * wx0, tt1[0], (cxa + 1.0) * wx1 * tt1[1]));
            v[h][2] = fma(cya * wy0, A0, (cya + 2.0) * wy2 * A1);
          }
          if (FM == 3) {
            const int ph = (h ? e1 : e0) & 0xff;
            const double* rr = raws + ((h ? b1 : b0) * BM + (ph < BM ? ph : 0)) * kRec;
            const double px = rr[10], py = rr[11];
            const double nx0 = ((double)(X0 + cx0) - 0.5 * P) * dv.h - px, ny0 = ((double)(Y0 + cy0) - 0.5 * P) * dv.h - py;
            const double ta = 2.0 * dv.alpha;
            const double wxd0 = ta * nx0 * wx0, wxd1 = ta * (nx0 + dv.h) * wx1;
            const double wyd0 = ta * ny0 * wy0, wyd2 = ta * (ny0 + 2.0 * dv.h) * wy2;
            v[h][1] = wy0 * fma(wxd0, tt0[0], wxd1 * tt0[1]) + wy2 * fma(wxd0, tt1[0], wxd1 * tt1[1]);
            v[h][2] = wyd0 * fma(wx0, tt0[0], wx1 * tt0[1]) + wyd2 * fma(wx0, tt1[0], wx1 * tt1[1]);
            if (FIELD) {
              const double* uu0 = u0 + 2 * h;
              const double* uu1 = u1 + 2 * h;
              v[h][NC - 1] = wy0 * fma(wx0, uu0[0], wx1 * uu0[1]) + wy2 * fma(wx0, uu1[0], wx1 * uu1[1]);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            v[h][cc] += __shfl_xor_sync(0xffffffffu, v[h][cc], 1);
            v[h][cc] += __shfl_xor_sync(0xffffffffu, v[h][cc], 2);
          }
        if (tig == 0) {
          const int pa = e0 & 0xff, pb = e1 & 0xff;
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            if (pa < BM) acc[((b0 * BM + pa) * (kCW + 1) + w) * NC + cc] = v[0][cc];
            if (pb < BM) acc[((b1 * BM + pb) * (kCW + 1) + w) * NC + cc] = v[1][cc];
          }
        }
        if (pend) {
          __threadfence_block();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[bprev]);
          pend = false;
        }
      }
      __threadfence_block();
    }
    if (pend) {   // (debug mode: no k-steps ran)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[bprev]);
    }
    const int rest = n > npad ? n - npad : 0;   // carry the rest (all from this batch)
    const int mv = lane < rest ? wl[npad + lane] : 0;
    __syncwarp();
    if (lane < rest) wl[lane] = mv;
    __syncwarp();
    held = rest;
    if (cn < 0) break;
    bprev = b;
  }
  }

  if (!GATHER) {
    const int cx = gid & 3, cy = gid >> 2;
#pragma unroll
    for (int zb = 0; zb < NZB; ++zb)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int x = X0b + cx, y = Y0b + cy + 2 * (v >> 1), z = Z0 + 8 * zb + 2 * tig + (v & 1);
        if (x < Mt && y < Mt && z < M) A.grid[((int64_t)x * Mt + y) * M + z] = c[zb][v];
      }
  }
}

// Sum the per-tile partials of every particle in a fixed order and scatter to user order.
// Only x tiles in [txlo, txhi) are summed (one slab of the distributed path; all tiles otherwise).
// FIELD: the slots hold (phi, dphi/dx, dphi/dy, dphi/dz); field = -grad phi (3 per particle).
template <int TZ, bool FIELD>
__global__ void k_gather_finish(KDev dv, const int4* __restrict__ S4, const int* __restrict__ perm,
                                const double* __restrict__ gpart, int64_t N, double* __restrict__ phi,
                                double* __restrict__ field, int txlo, int txhi) {
  constexpr int NC = FIELD ? 4 : 1;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int4 st = S4[p];
  const int P = dv.P;
  const int nx = fdiv(st.x + P - 1, kTXY) - fdiv(st.x, kTXY) + 1;
  const int ny = fdiv(st.y + P - 1, kTXY) - fdiv(st.y, kTXY) + 1;
  const int nz = zcount(st.w, P, dv.M, TZ);
  // slot-major partials [slot][value][particle]: a tile's consecutive particles write, and the
  // finish's consecutive threads read, consecutive addresses
  const double* g = gpart + p;
  double s[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) s[c] = 0.0;
  const int tx0 = fdiv(st.x, kTXY);
  for (int a = 0; a < nx; ++a) {
    if (tx0 + a < txlo || tx0 + a >= txhi) continue;
    for (int b = 0; b < ny; ++b)
      for (int z = 0; z < nz; ++z)
#pragma unroll
        for (int c = 0; c < NC; ++c) s[c] += g[(int64_t)(((a * dv.nsxy + b) * dv.nsz + z) * NC + c) * N];
  }
  const int64_t u = perm[p];
  if (phi) phi[u] = s[0];
  if (FIELD)
#pragma unroll
    for (int c = 0; c < 3; ++c) field[3 * u + c] = -s[1 + c];
}

// Compact records of the sorted particles: {jx0, jy0, lz0, lz0 mod M} (reading R-3), q, the
// sorted index, and per axis the Fast Gaussian Gridding factors of the first stencil
// node offset d0:  A = e^{-alpha d0^2},  E = e^{-2 alpha h d0}   (node t: A E^t f1[t]);
// FIELD records add the particle position.
template <bool FIELD>
__global__ void k_records(KDev dv, const double4* __restrict__ P4, const int4* __restrict__ S4, int64_t N,
                          double* __restrict__ rec) {
  constexpr int kRec = rec_len(FIELD);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double4 pp = P4[i];
  const int4 s = S4[i];
  const double P2 = 0.5 * dv.P;
  const double d0[3] = {((double)s.x - P2) * dv.h - pp.x, ((double)s.y - P2) * dv.h - pp.y, (double)s.z * dv.h - pp.z};
  double r[kRec];
  r[2] = pp.w;
  r[3] = __longlong_as_double((long long)i);   // the gather's slot index
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    r[4 + 2 * ax] = exp(-dv.alpha * d0[ax] * d0[ax]);
    r[5 + 2 * ax] = exp(-2.0 * dv.alpha * dv.h * d0[ax]);
  }
  if (FIELD) {
    r[10] = pp.x;
    r[11] = pp.y;
    r[12] = pp.z;
    r[kRec - 1] = 0.0;
  }
  double2* out = reinterpret_cast<double2*>(rec + i * kRec);
  out[0] = make_double2(__hiloint2double(s.y, s.x), __hiloint2double(s.w, s.z));
#pragma unroll
  for (int k = 1; k < kRec / 2; ++k) out[k] = make_double2(r[2 * k], r[2 * k + 1]);
}

int tile_tz(int M) { return M >= 64 ? 32 : 16; }
int rec_doubles(int P) { return (void)P, rec_len(true); }

// Slots of the gather partials: x and y tiles per stencil, then z tiles (<= ceil(P/TZ)+2 once
// the stencil wraps around the periodic axis).
void slot_geometry(KDev& dv) {
  const int TZ = tile_tz(dv.M), ntz = (int)ceil_div(dv.M, TZ);
  dv.nsxy = (dv.P - 1 + kTXY - 1) / kTXY + 1;
  dv.nsz = std::min((dv.P + TZ - 1) / TZ + 2, ntz);
  dv.nslot = dv.nsxy * dv.nsxy * dv.nsz;
}

int64_t gather_slots(const KDev& dv) {
  KDev d = dv;
  slot_geometry(d);
  return d.nslot;
}

void k_records_stage(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, bool field) {
  if (field)
    k_records<true><<<(unsigned)ceil_div(N, 128), 128, 0, st>>>(pl.dv, (const double4*)w.xs, (const int4*)w.s4, N,
                                                                 w.rec);
  else
    k_records<false><<<(unsigned)ceil_div(N, 128), 128, 0, st>>>(pl.dv, (const double4*)w.xs, (const int4*)w.s4, N,
                                                                  w.rec);
  SE1P_LAUNCH_CHECK();
}

template <int TZ, bool GATHER, int FM>
static void launch_tiles(const KPlan& pl, KWork& w, int64_t N, int tx_lo, int tx_hi, cudaStream_t st) {
  TileArgs a;
  a.dv = pl.dv;
  KDev& dv = a.dv;
  if (dv.P > kMaxP) throw Error{4, "P > 64 is not supported by the tile kernels"};
  slot_geometry(dv);
  dv.err = w.flag + 1;
  dv.N = N;
  {
    const char* e = getenv("SE1P_TILE_DBG");   // experiment bits (tools/tile_experiments.sh); 0 = normal
    dv.dbg = e ? atoi(e) : 0;
  }
  a.ntz = (int)ceil_div(dv.M, TZ);
  a.nty = (int)ceil_div(dv.Mt, kTXY);
  a.tx_lo = tx_lo;
  {
    // edge tiles last when the launch is a few waves (C4: 400 tiles, -4.6 %); at C5 (2592 tiles,
    // 17.5 waves) the in-order launch is 0.3 % faster
    static int n_sm = 0;
    if (!n_sm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
      if (n_sm <= 0) n_sm = 148;
    }
    const int64_t tiles = (int64_t)(tx_hi - tx_lo) * a.nty * a.ntz;
    const char* e = getenv("SE1P_TILE_ORDER");
    a.order = e ? atoi(e) : (tiles < 8 * (int64_t)n_sm ? 1 : 0);
  }
  const int ntx = tx_hi - tx_lo;
  if (ntx <= 0) return;
  a.rec = w.rec;
  a.bin_start = w.bin_start;
  a.f1 = pl.d_f1;
  a.grid = w.grid;
  a.gpart = GATHER ? w.gpart : nullptr;
  int BM = 0, NB = 0;
  const int limit = 227 * 1024 - 1024;
  for (int bm : {64, 32, 16}) {   // the gather's lag-2 reduction needs NB >= 3
    if (FM == 3 && bm > 32) continue;
    for (int nb = kMaxNB; nb >= (GATHER ? 3 : 2) && !BM; --nb)
      if (tile_smem(bm, nb, TZ, GATHER, FM).total <= limit) {
        BM = bm;
        NB = nb;
      }
    if (BM) break;
  }
  if (!BM) throw Error{4, "tile kernels do not fit in shared memory"};
  {   // experiment override (tools/): batch size and ring depth, if they fit
    const char* eb = getenv(GATHER ? "SE1P_GATHER_BM" : "SE1P_SPREAD_BM");
    const char* en = getenv(GATHER ? "SE1P_GATHER_NB" : "SE1P_SPREAD_NB");
    const int bm = eb ? atoi(eb) : BM, nb = en ? atoi(en) : NB;
    if ((eb || en) && bm >= 16 && bm <= 128 && nb >= (GATHER ? 3 : 2) && nb <= kMaxNB &&
        tile_smem(bm, nb, TZ, GATHER, FM).total <= limit) {
      BM = bm;
      NB = nb;
    }
  }
  a.BM = BM;
  a.NB = NB;
  const size_t smem = (size_t)tile_smem(BM, NB, TZ, GATHER, FM).total;
  SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_tiles<TZ, GATHER, FM>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned nblk = (unsigned)(ntx * a.nty * a.ntz);
  k_tiles<TZ, GATHER, FM><<<nblk, n_threads(FM), smem, st>>>(a);
  SE1P_LAUNCH_CHECK();
}

template <bool GATHER, int FM>
static void dispatch_tiles(const KPlan& pl, KWork& w, int64_t N, int tx_lo, int tx_hi, cudaStream_t st) {
  if (tx_hi < 0) tx_hi = (int)ceil_div(pl.dv.Mt, kTXY);
  if (tile_tz(pl.dv.M) == 32) launch_tiles<32, GATHER, FM>(pl, w, N, tx_lo, tx_hi, st);
  else launch_tiles<16, GATHER, FM>(pl, w, N, tx_lo, tx_hi, st);
}

void k_spread_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo, int tx_hi) {
  dispatch_tiles<false, 0>(pl, w, N, tx_lo, tx_hi, st);
}

void k_gather_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo, int tx_hi, bool field) {
  if (field) {
#if SE1P_FIELD_ONE_PASS
    dispatch_tiles<true, 3>(pl, w, N, tx_lo, tx_hi, st);
#else
    dispatch_tiles<true, 1>(pl, w, N, tx_lo, tx_hi, st);   // phi, d/dx, d/dy
    dispatch_tiles<true, 2>(pl, w, N, tx_lo, tx_hi, st);   // d/dz
#endif
  } else {
    dispatch_tiles<true, 0>(pl, w, N, tx_lo, tx_hi, st);
  }
}

void k_gather_finish_stage(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st, int tx_lo, int tx_hi,
                           double* field) {
  KDev dv = pl.dv;
  slot_geometry(dv);
  if (tx_hi < 0) tx_hi = (int)ceil_div(dv.Mt, kTXY);
  const unsigned nb = (unsigned)ceil_div(N, 256);
  const int4* s4 = (const int4*)w.s4;
  if (tile_tz(dv.M) == 32) {
    if (field) k_gather_finish<32, true><<<nb, 256, 0, st>>>(dv, s4, w.perm, w.gpart, N, phi, field, tx_lo, tx_hi);
    else k_gather_finish<32, false><<<nb, 256, 0, st>>>(dv, s4, w.perm, w.gpart, N, phi, field, tx_lo, tx_hi);
  } else {
    if (field) k_gather_finish<16, true><<<nb, 256, 0, st>>>(dv, s4, w.perm, w.gpart, N, phi, field, tx_lo, tx_hi);
    else k_gather_finish<16, false><<<nb, 256, 0, st>>>(dv, s4, w.perm, w.gpart, N, phi, field, tx_lo, tx_hi);
  }
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
