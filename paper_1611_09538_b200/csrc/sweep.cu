// sweep.cu -- gridding (Alg. 1 step 2, Eq. (spread_1p)) and gather (Alg. 1 step 6,
// Eq. (se1p_complete_discretized)) as z-aligned column sweeps on the FP64 tensor
// pipe (mma.sync m16n8k8 f64 -> SASS DMMA; tcgen05.mma has no f64 kind).  See tiles.cuh.
//
// Work item = (16 x 16 column tile of the extended free grid, chunk [Z0, Z0+Ck) of the periodic
// axis).  Persistent CTAs fetch items heavy-first from a work counter.  Inside an item the CTA
// sweeps the stencil-start layers a = Z0 .. Z0+Ck-1 in order.  A "group" is the set of candidate
// particles whose periodic stencil starts at node a (bins: x band, a, y cell, so a group is one
// contiguous run of the sorted order per x band).  Every particle of a group has its P z-weights
// on the SAME nodes a .. a+P-1, so in the frame of the group the z-window is dense:
//   gridding  C[16 cols x 8 z] += A[16 cols x 8 particles] B[8 particles x 8 z]   per 8-node block
//             A = (q wx) wy, B = wz (relative to a): no z block is partly outside the stencil,
//   gather    T[16 cols x 8 particles] += H~[16 cols x 8 z] wz^T[8 z x 8 particles],
//             phi_p += sum_cols wx wy T.
// The z window depends on the particle only, so k_records stores it with the particle's record
// (Fast Gaussian Gridding factors, for the free axes).  Roles (21 warps):
//   producer (1 warp): fetches items, walks their groups (one candidate run per x band: bin_start)
//     and cuts them into batches of <= BM candidates, whose records (with the z windows) it moves
//     into a ring of NB shared-memory slots with bulk copies (cp.async.bulk, SASS UBLKCP;
//     completion by transaction bytes on the slot's mbarrier).
//   expanders (4 warps): per candidate the tile's x and y windows from the FGG factors -- the
//     record holds per free axis A = e^{-alpha d0^2}, E = e^{-2 alpha h d0} (node t weighs
//     A E^t f1[t]) with E^-1 and E^8 for short power trees -- and the 16-bit mask of consumer
//     warps whose 4 x 4 column block the stencil meets; then `full`.  Gather: they also sum the
//     consumers' per-warp partials of finished batches into the particle's slot (fixed order).
//   consumers (16 warps): warp w owns the 4 x 4 column block (w & 3, w >> 2) of the tile; per
//     batch it lists (ballot) the candidates meeting it and runs 8-particle k-steps.  Entries left
//     over (< 8) are carried into the next batch of the same group; a group's last batch pads.
//     Gridding accumulates each group's frame (16 cols x 8 NZB nodes) in a per-warp ring of
//     positions in shared memory (load frame, k-steps, store frame); position u is complete once
//     group u is done, and completed 8-position blocks are written to the grid.  The P-1 positions
//     past the chunk end go to an overhang buffer that k_overhang adds to the next chunk.
// No floating-point atomics: each grid point is written by one warp; the gather's partials go
// to fixed slots summed in a fixed order (k_gather_finish) -> bitwise reproducible.
#include <cstdint>
#include <type_traits>
#include <vector>

#include "tiles.cuh"

namespace se1p {

constexpr int kCW = 16;                 // consumer warps (16 blocks of 4 x 4 columns)
constexpr int kEG = 2;                  // expander groups (alternate batches)
constexpr int kGW = 4;                  // warps per expander group
constexpr int kSW = kEG * kGW;          // expander warps
constexpr int kSweepThreads = (kCW + 1 + kSW) * 32;
constexpr int kMaxNB = 4;
// batch ring depth (shared-memory slots): even, so that a row slot is always reused by the
// expander group that filled it
#ifndef SE1P_SWEEP_NB
#define SE1P_SWEEP_NB 4
#endif
constexpr int kNB = SE1P_SWEEP_NB;
// gather k-steps issued together (1 or 2)
#ifndef SE1P_SWEEP_GU
#define SE1P_SWEEP_GU 1
#endif
constexpr int kGU = SE1P_SWEEP_GU;
// gather k-step of 16 particles with the operands swapped (w_z^T as A, the frame as B; 1) or of
// 8 particles with the frame as A (0)
#ifndef SE1P_GATHER_T16
#define SE1P_GATHER_T16 1
#endif
constexpr int kMaxP = 64;

// header flags of a batch
constexpr int kFirst = 1, kLast = 2, kItemEnd = 4, kKernelEnd = 8;

__host__ __device__ constexpr int sw_nzb(int P) { return P <= 16 ? 2 : (P <= 24 ? 3 : (P <= 32 ? 4 : 8)); }
// record (k_records): {jx0, jy0}, q, x: A E E^-1 E^8, y: A E E^-1 E^8, d0 x y z, sorted index, pad,
// then the z window wz[0 .. 8 NZB) (zero past P); stride = 8 (mod 16) doubles so that the
// consumers' loads of 4 or 8 records spread over the banks
constexpr int kRq = 1, kRx = 2, kRy = 6, kRd = 10, kRi = 13, kRz = 16;
__host__ __device__ constexpr int rec_stride(int NZB) { return kRz + 8 * NZB + ((NZB & 1) ? 0 : 8); }
// rows: x[0:16) y[0:16) (XOR-swizzled, see xy_key), then the z window (copied from the record);
// stride 8 (mod 16) doubles
constexpr int kZ = 32;
__host__ __device__ constexpr int row_stride(int NZB) { return kZ + 8 * NZB + ((NZB & 1) ? 0 : 8); }
#ifndef SE1P_SWEEP_NR
#define SE1P_SWEEP_NR 2
#endif
constexpr int kNR = SE1P_SWEEP_NR;   // record ring depth (batches, a multiple of kEG): released once expanded
// gridding ring: R positions (>= 8 NZB + 8), column stride S = 4 (mod 16) doubles
__host__ __device__ constexpr int sw_R(int NZB) { return 8 * NZB + 8; }
__host__ __device__ constexpr int sw_S(int NZB) { return sw_R(NZB) + ((4 - sw_R(NZB)) % 16 + 16) % 16; }
__host__ __device__ constexpr int sw_nc(int FM) { return FM == 1 ? 3 : 1; }   // gather outputs per pass
// Swizzles (row stride 8 mod 16 doubles, so row e starts at bank pair 8 (e & 1)), with k = e & 6:
// x node i (0..15) of the row of ring slot e sits at i ^ k, y node i at 16 + (ypos(i) ^ k ^ 1) with
// ypos swapping bits 1 and 2 of i, z node n (0..7) of block j at kZ + 8 j + (n ^ (k & 2)).  A warp's
// list is mostly runs of consecutive slots, and for any 4 consecutive slots these make the
// consumers' loads conflict-free: the gridding z loads (4 particles x 8 nodes), x loads (4 x 2 nodes)
// and y loads (4 x 4 nodes), the gather's z pairs; the 8 consecutive slots x 2 axes of one expander
// half-warp's stores hit 16 distinct bank pairs.
__host__ __device__ __forceinline__ int ypos(int i) { return (i & ~6) | ((i & 2) << 1) | ((i & 4) >> 1); }

struct SweepArgs {
  KDev dv;
  const double* rec;
  const int* bin_start;
  const double* f1;
  double* grid;       // gridding: H (written); gather: H~ (read)
  double* over;       // gridding: overhang [nzc][Mt][Mt][P-1]
  double* gpart;      // gather partials [slot][value][N]
  const int* items;   // packed items (tx | ty << 10 | zc << 20), heavy first
  int* counter;       // work counter (zeroed by k_items)
  int n_items, C, nzc, BM, NB;
};

// list capacity per (slot, consumer warp): a batch's entries plus the k-step padding
__host__ __device__ constexpr int sw_ls(int BM) { return BM + 16; }

struct SweepSmem {
  int off_meta, off_mask, off_lists, off_lcnt, off_cb, off_raw, off_rows, off_acc, off_ring, total;
};

// barriers: full, empty, (unused) [kMaxNB], rawb, rawfree [kNR]; headers hdr [kMaxNB], bhdr [kNR]
constexpr int kSmemHead = (3 * kMaxNB + 2 * kNR) * 8 + (kMaxNB + kNR) * 16;

__host__ __device__ inline SweepSmem sweep_smem(int BM, int NB, int NZB, bool gather, int FM) {
  SweepSmem s;
  int o = kSmemHead + kMaxP * 8;                              // + f1
  o = (o + 15) & ~15;
  s.off_meta = o;
  o += (NB * BM + 1) * 16;
  s.off_mask = o;
  o += (NB * BM + 1) * 4;
  o = (o + 15) & ~15;
  s.off_lists = o;   // per-slot consumer lists, written by the expanders
  o += NB * kCW * sw_ls(BM) * 2;
  o = (o + 15) & ~15;
  s.off_lcnt = o;
  o += NB * kCW * 4;
  s.off_cb = o;      // per-warp carry lists (two, alternating)
  o += kCW * 32 * 2;
  o = (o + 127) & ~127;
  s.off_raw = o;
  o += kNR * BM * rec_stride(NZB) * 8;
  s.off_rows = o;
  o += (NB * BM + 1) * row_stride(NZB) * 8;
  s.off_acc = o;
  if (gather) o += (NB * BM + 1) * (kCW * sw_nc(FM) + 1) * 8;
  o = (o + 127) & ~127;
  s.off_ring = o;
  if (!gather) o += kCW * 16 * sw_S(NZB) * 8;
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
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
// SE1P_SWEEP_WATCHDOG (debug builds): report and trap a wait that never completes
#ifndef SE1P_SWEEP_WATCHDOG
#define SE1P_SWEEP_WATCHDOG 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity, int tag = 0) {
#if SE1P_SWEEP_WATCHDOG
  const long long t0 = clock64();
  while (!mbar_try_wait(b, parity)) {
    if (clock64() - t0 > 4000000000ll) {
      printf("sweep watchdog: block %d warp %d tag %d parity %u\n", blockIdx.x, threadIdx.x >> 5, tag, parity);
      __trap();
    }
  }
#else
  (void)tag;
  while (!mbar_try_wait(b, parity)) {
  }
#endif
}

// SE1P_SWEEP_TRACE (experiment builds): CTA 0's per-batch timeline (clock64): producer post,
// expander sees the records / a free slot / arrives full, consumer warp 0 sees full / arrives empty,
// its k-steps and the batch size, then consumer checkpoints; read with se1p_sweep_trace
#ifndef SE1P_SWEEP_TRACE
#define SE1P_SWEEP_TRACE 0
#endif
#if SE1P_SWEEP_TRACE
constexpr int kTraceN = 8192, kTraceF = 12;
__device__ long long g_trace[2][kTraceN][kTraceF];   // [gridding, gather]
#define SW_TRACE(k, i, v) \
  if (blockIdx.x == 0 && (k) < kTraceN) g_trace[GATHER][k][i] = (v)
#define SW_CTRACE(i) \
  if (w == 0 && lane == 0) SW_TRACE(kc, i, clock64())
#else
#define SW_TRACE(k, i, v)
#define SW_CTRACE(i)
#endif

template <bool GATHER, int FM, int NZB>
__global__ void __launch_bounds__(kSweepThreads, 1) k_sweep(const SweepArgs A) {
  constexpr int RD = rec_stride(NZB), RS = row_stride(NZB), R = sw_R(NZB), S = sw_S(NZB);
  constexpr int NC = sw_nc(FM);                   // values this pass writes per particle
  constexpr int NCT = FM ? 4 : 1;                 // values per gather slot
  constexpr int COFF = FM == 2 ? 3 : 0;           // first slot value of this pass
  constexpr int ACS = kCW * NC + 1;               // acc doubles per candidate (odd: conflict-free reduce)
  constexpr bool XL = GATHER;                     // consumer lists built by the expanders
  constexpr bool T16 = GATHER && SE1P_GATHER_T16;   // 16-particle gather k-steps
  constexpr int KS = T16 ? 16 : 8;                 // particles per k-step
  extern __shared__ __align__(128) unsigned char smem[];
  const KDev& dv = A.dv;
  const int BM = A.BM, NB = A.NB, P = dv.P, M = dv.M, Mt = dv.Mt;
  const SweepSmem L = sweep_smem(BM, NB, NZB, GATHER, FM);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxNB;
  uint64_t* rawb = empty + kMaxNB + kMaxNB;
  uint64_t* rawfree = rawb + kNR;
  int4* hdr = reinterpret_cast<int4*>(rawfree + kNR);
  int4* bhdr = hdr + kMaxNB;
  double* f1 = reinterpret_cast<double*>(smem + kSmemHead);
  int4* meta = reinterpret_cast<int4*>(smem + L.off_meta);
  int* mask = reinterpret_cast<int*>(smem + L.off_mask);
  unsigned short* lists = reinterpret_cast<unsigned short*>(smem + L.off_lists);
  int* lcnt = reinterpret_cast<int*>(smem + L.off_lcnt);
  const int LS = sw_ls(BM);
  double* raw = reinterpret_cast<double*>(smem + L.off_raw);
  double* rows = reinterpret_cast<double*>(smem + L.off_rows);
  double* acc = reinterpret_cast<double*>(smem + L.off_acc);
  double* ring = reinterpret_cast<double*>(smem + L.off_ring);
  const int dummy = NB * BM;   // the all-zero slot

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int b = 0; b < kMaxNB; ++b) {
      mbar_init(&full[b], kGW);
      mbar_init(&empty[b], kCW);
    }
    for (int r = 0; r < kNR; ++r) {
      mbar_init(&rawb[r], 1);
      mbar_init(&rawfree[r], kGW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = tid; k < kMaxP; k += kSweepThreads) f1[k] = k < P ? A.f1[k] : 0.0;
  for (int k = tid; k < RS; k += kSweepThreads) rows[dummy * RS + k] = 0.0;
  if (tid < 4) reinterpret_cast<int*>(&meta[dummy])[tid] = 0;
  if (tid == 0) mask[dummy] = 0;
  if (!GATHER)
    for (int k = tid; k < kCW * 16 * S; k += kSweepThreads) ring[k] = 0.0;
  __syncthreads();

  auto item_geom = [&](int it, int& X0, int& Y0, int& Z0, int& Ck, int& zc) {
    const int pk = A.items[it];
    const int tx = pk & 1023, ty = (pk >> 10) & 1023;
    zc = pk >> 20;
    X0 = tx * kTXY;
    Y0 = ty * kTXY;
    Z0 = zc * A.C;
    Ck = min(A.C, M - Z0);
  };

  if (w == kCW) {
    // ================================================================ producer
    int k = 0;   // batch sequence number
    auto acquire = [&](int b) {   // record slot b free: its previous batch expanded
      if (k >= kNR) mbar_wait(&rawfree[b], (unsigned)(((k - kNR) / kNR) & 1), 100 + k);
    };
    auto post = [&](int b, int4 h) {   // after every lane's copies: header, then the arrival
      __syncwarp();
      if (lane == 0) {
        bhdr[b] = h;
        mbar_arrive(&rawb[b]);
        SW_TRACE(k, 0, clock64());
      }
      __syncwarp();
      ++k;
    };
    for (;;) {
      int it = 0;
      if (lane == 0) it = atomicAdd(A.counter, 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= A.n_items) {   // one end marker per expander group
        for (int gq = 0; gq < kEG; ++gq) {
          const int b = k % kNR;
          acquire(b);
          post(b, make_int4(-1, gq, 0, kKernelEnd));
        }
        break;
      }
      int X0, Y0, Z0, Ck, zc;
      item_geom(it, X0, Y0, Z0, Ck, zc);
      // candidate runs of layer a: x bands covering cells [X0 - P, X0 + 14], y cells [cy0, cy1]
      const int b0 = max(0, fdiv(X0 - P, kBin)), b1 = min(dv.nbx - 1, fdiv(X0 + kTXY - 2, kBin));
      const int cy0 = max(0, Y0 - P), cy1 = min(dv.Mfree - 1, Y0 + kTXY - 2);
      const int nruns = (cy1 >= cy0) ? max(0, b1 - b0 + 1) : 0;
      // run bounds of layer u + 1 are loaded while layer u's batches are issued
      auto load_runs = [&](int u, int& s0, int& e0) {
        s0 = e0 = 0;
        if (u < Ck && lane < nruns) {
          const int row = ((b0 + lane) * M + Z0 + u) * dv.Mfree;
          s0 = __ldg(A.bin_start + row + cy0);
          e0 = __ldg(A.bin_start + row + cy1 + 1);
        }
      };
      int sN, eN;
      load_runs(0, sN, eN);
      for (int u = 0; u < Ck; ++u) {
        const int s0 = sN, len = eN - sN;
        load_runs(u + 1, sN, eN);
        if (len < 0 || s0 < 0 || (int64_t)s0 + len > dv.N) atomicOr(dv.err, 1);
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        const int pre = incl - len;
        for (int lo = 0; lo < tot; lo += BM) {
          const int b = k % kNR;
          acquire(b);
          const int cnt = min(BM, tot - lo);
          const int a0 = max(pre, lo), a1 = min(pre + len, lo + cnt);
          if (a1 > a0) {
            const unsigned bytes = (unsigned)((a1 - a0) * RD * 8);
            mbar_expect_tx(&rawb[b], bytes);
            bulk_g2s(raw + ((int64_t)b * BM + (a0 - lo)) * RD, A.rec + ((int64_t)s0 + (a0 - pre)) * RD, bytes,
                     &rawb[b]);
          }
          post(b, make_int4(it, u, cnt, (lo == 0 ? kFirst : 0) | (lo + BM >= tot ? kLast : 0)));
        }
      }
      const int b = k % kNR;
      acquire(b);
      post(b, make_int4(it, Ck, 0, kItemEnd));
    }
    return;
  }

  if (w > kCW) {
    // ================================================================ expanders
    // group gi expands batches k = gi, gi + kEG, ...; record slot k % kNR = gi; with kNB even the
    // row slot k % kNB returns to the same group, which first reduces (gather) its previous batch
    const int ew = w - kCW - 1, gi = ew / kGW, gw = ew % kGW, gl = gw * 32 + lane;
    // gather: sum batch j's per-warp partials into the slots (fixed warp order)
    auto reduce_batch = [&](int j) {
      const int bj = j % NB;
      mbar_wait(&empty[bj], (unsigned)((j / NB) & 1), 200000 + j);
      const int4 h = hdr[bj];
      if (h.z > 0) {
        int X0, Y0, Z0, Ck, zc;
        item_geom(h.x, X0, Y0, Z0, Ck, zc);
        const int tx = X0 / kTXY, ty = Y0 / kTXY;
        for (int p = gl; p < h.z; p += kGW * 32) {
          const int4 m = meta[bj * BM + p];
          const int wm = mask[bj * BM + p];
          if (wm == 0) continue;
          const double* ap = acc + (int64_t)(bj * BM + p) * ACS;
          double sm[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) sm[c] = 0.0;
          for (int v = 0; v < kCW; ++v)
            if ((wm >> v) & 1)
#pragma unroll
              for (int c = 0; c < NC; ++c) sm[c] += ap[v * NC + c];
          if (FM == 1) {   // column moments -> d/dx, d/dy: 2 alpha (h S + delta phi), delta = d0 + (X0 - j0) h
            const double* rr = A.rec + (int64_t)m.w * RD;
            const double ta = 2.0 * dv.alpha;
            const double dx = rr[kRd] + (double)(X0 - m.y) * dv.h, dy = rr[kRd + 1] + (double)(Y0 - m.z) * dv.h;
            sm[1] = ta * fma(dv.h, sm[1], dx * sm[0]);
            sm[2] = ta * fma(dv.h, sm[2], dy * sm[0]);
          }
          const int sx = tx - fdiv(m.y, kTXY), sy = ty - fdiv(m.z, kTXY);
          if (sx < 0 || sx >= dv.nsxy || sy < 0 || sy >= dv.nsxy || m.w < 0 || m.w >= dv.N) {
            atomicOr(dv.err, 4);
#if SE1P_SWEEP_WATCHDOG
            printf("slot check: blk %d j %d bj %d p %d h=(%d %d %d %d) wm %x meta=(%d %d %d %d) X0 %d Y0 %d\n", blockIdx.x, j,
                   bj, p, h.x, h.y, h.z, h.w, wm, m.x, m.y, m.z, m.w, X0, Y0);
#endif
            continue;
          }
#pragma unroll
          for (int c = 0; c < NC; ++c)
            A.gpart[(int64_t)((sx * dv.nsxy + sy) * NCT + COFF + c) * dv.N + m.w] = sm[c];
        }
      }
    };
    for (int k = gi;; k += kEG) {
      const int b = k % NB, r = k % kNR;
      mbar_wait(&rawb[r], (unsigned)((k / kNR) & 1), 300000 + k);
      if (gw == 0 && lane == 0) SW_TRACE(k, 1, clock64());
      const int4 h = bhdr[r];
      if (h.w & kKernelEnd) {   // drain this group's unreduced batches; end marker 0 goes to the consumers
        if (GATHER)
          for (int j = max(gi, k - NB); j < k; j += kEG) reduce_batch(j);
        else if (k >= NB)
          mbar_wait(&empty[b], (unsigned)(((k - NB) / NB) & 1), 600000 + k);
        if (h.y == 0) {
          if (gw == 0 && lane == 0) hdr[b] = h;
          __threadfence_block();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[b]);
        }
        break;
      }
      if (k >= NB) {
        if (GATHER) {
          reduce_batch(k - NB);
          // the group's 4 warps reduced disjoint candidates of the slot: all done before it is refilled
          asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "n"(kGW * 32) : "memory");
        } else {
          mbar_wait(&empty[b], (unsigned)(((k - NB) / NB) & 1), 600000 + k);
        }
      }
      if (gw == 0 && lane == 0) SW_TRACE(k, 2, clock64());
      if (h.z > 0) {
        int X0, Y0, Z0, Ck, zc;
        item_geom(h.x, X0, Y0, Z0, Ck, zc);
        // tasks: 2 per candidate (the tile's 16 x nodes, 16 y nodes)
        for (int t = gl; t < h.z * 2; t += kGW * 32) {
          const int cand = t >> 1, ax = t & 1, e = b * BM + cand;
          const double* rr = raw + (int64_t)(r * BM + cand) * RD;
          const int2 jj = *reinterpret_cast<const int2*>(rr);
          // v[i] = A E^(t0+i) f1[t0+i] on the stencil nodes 0 <= t0+i < P, else 0, as base E^i with
          // base = A E^t0 from a power tree (short dependency chains: the FP64 pipe is shared with
          // the consumers' DMMAs); nodes 8..15 from base E^8
          const double* ra = rr + (ax == 0 ? kRx : kRy);
          const int t0 = ax == 0 ? X0 - jj.x : Y0 - jj.y;
          const double E = ra[1], E8 = ra[3];
          const bool neg = t0 < 0;
          const int n = min(neg ? -t0 : t0, 63);
          const double b1 = neg ? ra[2] : E;
          const double b2 = b1 * b1, b4 = b2 * b2;
          const double e8 = neg ? b4 * b4 : E8, e16 = e8 * e8, e32 = e16 * e16;
          const double f01 = ((n & 1) ? b1 : 1.0) * ((n & 2) ? b2 : 1.0);
          const double f23 = ((n & 4) ? b4 : 1.0) * ((n & 8) ? e8 : 1.0);
          const double a0 = (!GATHER && ax == 0) ? ra[0] * rr[kRq] : ra[0];   // gridding: q folded into wx
          const double base = (a0 * (((n & 16) ? e16 : 1.0) * ((n & 32) ? e32 : 1.0))) * (f01 * f23);
          const double base8 = base * E8;
          const double E2 = neg ? E * E : b2, E4 = neg ? E2 * E2 : b4;
          const double E3 = E2 * E;
          const double pw[8] = {1.0, E, E2, E3, E4, E4 * E, E4 * E2, E4 * E3};
          double* o = rows + (int64_t)e * RS + 16 * ax;
          const int key = (e & 6) | ax;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int tt = t0 + q;
            o[(ax ? ypos(q) : q) ^ key] = (tt >= 0 && tt < P) ? ((q < 8 ? base : base8) * f1[tt]) * pw[q & 7] : 0.0;
          }
          if (ax == 0) {
            // consumer warps whose 4 x 4 block the stencil meets
            const int bx0 = max(fdiv(jj.x - X0, 4), 0), bx1 = min(fdiv(jj.x - X0 + P - 1, 4), 3);
            const int by0 = max(fdiv(jj.y - Y0, 4), 0), by1 = min(fdiv(jj.y - Y0 + P - 1, 4), 3);
            int wm = 0;
            if (bx0 <= bx1 && by0 <= by1) {
              const int xb = ((1 << (bx1 + 1)) - 1) & ~((1 << bx0) - 1);
              for (int by = by0; by <= by1; ++by) wm |= xb << (4 * by);
            }
            meta[e] = make_int4(0, jj.x, jj.y, (int)__double_as_longlong(rr[kRi]));
            mask[e] = wm;
          }
          // the z window: 16-byte chunks ax, ax + 2, ..., rotated by 3 steps for every other pair of
          // candidates (conflict-free 16-byte stores)
          const double2* zs = reinterpret_cast<const double2*>(rr + kRz);
          double2* zd = reinterpret_cast<double2*>(rows + (int64_t)e * RS + kZ);
          const int nz2 = 2 * NZB, rot = ((cand >> 1) & 1) * 3, zk = (e >> 1) & 1;
#pragma unroll
          for (int i = 0; i < nz2; ++i) {
            int i2 = i + rot;
            if (i2 >= nz2) i2 -= nz2;
            const int sc = 2 * i2 + ax;   // source chunk (node pair) -> block sc >> 2, pair (sc & 3) ^ zk
            zd[(sc & ~3) | ((sc & 3) ^ zk)] = zs[sc];
          }
        }
        // gather: the consumer lists of this batch (candidate order), warp gw builds those of
        // consumers gw, gw + 4, gw + 8, gw + 12 once the group's masks are all written (gridding:
        // the consumers build their own, the expanders being the slower side there)
        if (XL) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "n"(kGW * 32) : "memory");
        unsigned short* Lb = lists + b * kCW * LS;
        int nl[4] = {0, 0, 0, 0};
        const unsigned lt = (1u << lane) - 1u;
        for (int p0 = 0; p0 < h.z; p0 += 32) {
          const int p = p0 + lane;
          const int m = p < h.z ? mask[b * BM + p] : 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool rel = (m >> (gw + 4 * i)) & 1;
            const unsigned bal = __ballot_sync(0xffffffffu, rel);
            if (rel) Lb[(gw + 4 * i) * LS + nl[i] + __popc(bal & lt)] = (unsigned short)(b * BM + p);
            nl[i] += __popc(bal);
          }
        }
        if (lane < 4) lcnt[b * kCW + gw + 4 * lane] = lane == 0 ? nl[0] : lane == 1 ? nl[1] : lane == 2 ? nl[2] : nl[3];
        }
      }
      if (gw == 0 && lane == 0) hdr[b] = h;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&rawfree[r]);
        mbar_arrive(&full[b]);
        if (gw == 0) SW_TRACE(k, 3, clock64());
      }
    }
    return;
  }

  // ================================================================== consumers
  const int g = lane >> 2, tg = lane & 3;
  const int bxw = w & 3, byw = w >> 2;
  const int xa = 4 * bxw + (g >> 2), yb = 4 * byw + (g & 3);   // this lane's columns g, g+8 -> x xa, xa+2; y yb
  // row offsets (see ypos): x node xa (xa + 2) at xa ^ k, y node yb at 16 + (yq ^ k), k = e & 6
  const int yq = ypos(yb) ^ 1;
  // gridding: B lane g holds frame node sg = (g >> 1) + 4 (g & 1), so C lane tg holds nodes tg, tg + 4;
  // gather: K index tg (tg + 4) of block j is node 2 tg (2 tg + 1): one 16-byte pair of the record
  const int sg = (g >> 1) + 4 * (g & 1);
  // carried entries: two buffers per warp, so a batch's left-overs are copied out before its
  // k-steps (the copy then does not wait behind the k-steps' shared-memory traffic)
  unsigned short* cbw = reinterpret_cast<unsigned short*>(smem + L.off_cb) + w * 32;
  int cbsel = 0;
  double* rg = ring + w * 16 * S;   // gridding ring [16 cols][S]

  int cur = -1, X0 = 0, Y0 = 0, Z0 = 0, Ck = 0, zc = 0;
  int u = 0, flushed = 0;
  bool fr = false;   // frame loaded for group u
  double c[NZB][4];  // gridding frame accumulators / gather frame operand H~[16 cols x 8 z]
#pragma unroll
  for (int j = 0; j < NZB; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;

  // gridding: ring position p -> slot p mod R; lane's frame value (j, v): col g + 8 (v >> 1),
  // node u + 8 j + tg + 4 (v & 1)
  auto frame_io = [&](bool store) {
#pragma unroll
    for (int j = 0; j < NZB; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int col = g + 8 * (v >> 1);
        const int sl = (u + 8 * j + tg + 4 * (v & 1)) % R;
        double* p = rg + col * S + sl;
        if (store) *p = c[j][v];
        else c[j][v] = *p;
      }
  };
  // gridding: write positions [f, f + 8) of the warp's 16 columns (grid, or overhang past Ck), zero them
  auto flush_block = [&](int f) {
    const int col = lane >> 1, hh = lane & 1;
    const int x = X0 + 4 * bxw + (col >> 2), y = Y0 + 4 * byw + (col & 3);
    double* p = rg + col * S + (f % R) + 4 * hh;
    const double2 v0 = *reinterpret_cast<double2*>(p), v1 = *reinterpret_cast<double2*>(p + 2);
    *reinterpret_cast<double2*>(p) = make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(p + 2) = make_double2(0.0, 0.0);
    if (x < Mt && y < Mt) {
      const double vv[4] = {v0.x, v0.y, v1.x, v1.y};
      const int p0 = f + 4 * hh;
      if (p0 + 4 <= Ck) {
        double* gp = A.grid + ((int64_t)x * Mt + y) * M + Z0 + p0;
        *reinterpret_cast<double2*>(gp) = v0;
        *reinterpret_cast<double2*>(gp + 2) = v1;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int pp = p0 + i;
          if (pp < Ck) A.grid[((int64_t)x * Mt + y) * M + Z0 + pp] = vv[i];
          else if (pp < Ck + P - 1)
            A.over[(((int64_t)zc * Mt + x) * Mt + y) * (P - 1) + (pp - Ck)] = vv[i];
        }
      }
    }
  };
  // gather: the frame operand A[j] = H~[cols g, g+8][nodes a + 8j + 2 tg (+1)]
  // (column pointers gp0, gp1 of cols g, g + 8 set per item; null outside the grid)
  const double* gp0 = nullptr;
  const double* gp1 = nullptr;
  auto frame_load_gather = [&]() {
    const int zb = Z0 + u + 2 * tg;
#pragma unroll
    for (int j = 0; j < NZB; ++j)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        int z = zb + 8 * j + s;
        z = z >= M ? z - M : z;   // z < 2 M
        c[j][2 * s] = gp0 ? __ldg(gp0 + z) : 0.0;
        c[j][2 * s + 1] = gp1 ? __ldg(gp1 + z) : 0.0;
      }
  };

  auto ksteps = [&](const unsigned short* wl, int k0, int k1) {
#ifdef SE1P_SWEEP_EXP_NO_KSTEPS   // experiment build: the staging and bookkeeping floor
    return;
#endif
    if (!GATHER) {
      for (int k = k0; k < k1; k += 8) {
        const int e0 = wl[k + tg], e1 = wl[k + tg + 4];
        const double* r0 = rows + e0 * RS;
        const double* r1 = rows + e1 * RS;
        const int k0 = e0 & 6, k1 = e1 & 6;
        const double y0 = r0[16 + (yq ^ k0)], y1 = r1[16 + (yq ^ k1)];
        const double a[4] = {r0[xa ^ k0] * y0, r0[(xa + 2) ^ k0] * y0, r1[xa ^ k1] * y1, r1[(xa + 2) ^ k1] * y1};
        const double* z0 = r0 + kZ + (sg ^ (k0 & 2));
        const double* z1 = r1 + kZ + (sg ^ (k1 & 2));
#pragma unroll
        for (int j = 0; j < NZB; ++j) dmma_16x8x8(c[j], a, z0[8 * j], z1[8 * j]);
      }
    } else {
      // U k-steps at once (independent chains); T[col g (+8)][particle 2tg (+1)] of k-step u gives
      // the particle's column partial wy (wx T + wx' T'), summed over the 8 g lanes by a
      // transposing butterfly: each round halves the values a lane holds, so lane g < 2U ends
      // with the full sum of particle 2tg + (g & 1) of k-step g >> 1
      auto gstep = [&](auto uc, int k) {
        constexpr int U = decltype(uc)::value;
        double t[U][4];
        int ee[U][2];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          const int e = wl[k + 8 * uu + g];
          const double* z = rows + e * RS + kZ + ((2 * tg) ^ (e & 2));
          t[uu][0] = t[uu][1] = t[uu][2] = t[uu][3] = 0.0;
#pragma unroll
          for (int j = 0; j < NZB; ++j) {
            const double2 bb = *reinterpret_cast<const double2*>(z + 8 * j);
            dmma_16x8x8(t[uu], c[j], bb.x, bb.y);
          }
          ee[uu][0] = wl[k + 8 * uu + 2 * tg];
          ee[uu][1] = wl[k + 8 * uu + 2 * tg + 1];
        }
        double v[U][2][NC];
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
#pragma unroll
          for (int pb = 0; pb < 2; ++pb) {
            const int ep = ee[uu][pb];
            const double* rp = rows + ep * RS;
            const int sp = ep & 6;
            const double wx = rp[xa ^ sp], wx2 = rp[(xa + 2) ^ sp], wy = rp[16 + (yq ^ sp)];
            const double tp = t[uu][pb], tp2 = t[uu][pb + 2];
            v[uu][pb][0] = wy * fma(wx, tp, wx2 * tp2);
            if (FM == 1) {   // column moments in tile coordinates (x: xa, xa + 2; y: yb)
              const double cx = (double)xa;
              v[uu][pb][1] = wy * fma(cx * wx, tp, (cx + 2.0) * wx2 * tp2);
              v[uu][pb][2] = (double)yb * v[uu][pb][0];
            }
          }
        // round 1 (lanes g ^ 1): keep particle (g & 1) of each k-step
        const bool b1 = g & 1;
        double r1[U][NC];
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            const double send = b1 ? v[uu][0][cc] : v[uu][1][cc];
            const double keep = b1 ? v[uu][1][cc] : v[uu][0][cc];
            r1[uu][cc] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
          }
        double x[NC];
        if (U == 2) {   // round 2 (lanes g ^ 2): keep k-step (g >> 1) & 1
          const bool b2 = (g >> 1) & 1;
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) {
            const double send = b2 ? r1[0][cc] : r1[U - 1][cc];
            const double keep = b2 ? r1[U - 1][cc] : r1[0][cc];
            x[cc] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) x[cc] = r1[0][cc] + __shfl_xor_sync(0xffffffffu, r1[0][cc], 8);
        }
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) x[cc] += __shfl_xor_sync(0xffffffffu, x[cc], 16);
        if (g < 2 * U) {
          const int uu = g >> 1;
          const int ep = (uu == 0) ? (b1 ? ee[0][1] : ee[0][0]) : (b1 ? ee[U - 1][1] : ee[U - 1][0]);
#pragma unroll
          for (int cc = 0; cc < NC; ++cc) acc[(int64_t)ep * ACS + w * NC + cc] = x[cc];
        }
      };
      // 16 particles per k-step with the operands swapped: D_nb[16 particles x 8 cols] =
      // w_z^T[16 particles x 8 nodes] (A: the particles' z pairs, 16-byte loads) x H~^T (B: the
      // same frame registers, column half nb); a lane then holds particles g, g + 8 at columns
      // 2tg, 2tg + 1 of both halves, so the column sum is a 2-round butterfly over the quad
      // (every lane of the quad reads the same 4 weights of a particle: x nodes xA, xA + 2,
      // y nodes yA, yA + 1)
      auto gstep16 = [&](int k) {
        const int eg = wl[k + g], eg8 = wl[k + 8 + g];
        const double* zg = rows + eg * RS + kZ + ((2 * tg) ^ (eg & 2));
        const double* zg8 = rows + eg8 * RS + kZ + ((2 * tg) ^ (eg8 & 2));
        double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NZB; ++j) {
          const double2 za = *reinterpret_cast<const double2*>(zg + 8 * j);
          const double2 zb = *reinterpret_cast<const double2*>(zg8 + 8 * j);
          const double a[4] = {za.x, zb.x, za.y, zb.y};
          dmma_16x8x8(d0, a, c[j][0], c[j][2]);
          dmma_16x8x8(d1, a, c[j][1], c[j][3]);
        }
        const int xA = 4 * bxw + (tg >> 1), yA = 4 * byw + 2 * (tg & 1);
        const int qA = ypos(yA) ^ 1, qB = ypos(yA + 1) ^ 1;
        double v[2][NC];
#pragma unroll
        for (int pb = 0; pb < 2; ++pb) {
          const int ep = pb ? eg8 : eg;
          const double* rp = rows + ep * RS;
          const int sp = ep & 6;
          const double wxA = rp[xA ^ sp], wxB = rp[(xA + 2) ^ sp];
          const double wyA = rp[16 + (qA ^ sp)], wyB = rp[16 + (qB ^ sp)];
          const double sA = fma(wyA, d0[2 * pb], wyB * d0[2 * pb + 1]);   // x node xA
          const double sB = fma(wyA, d1[2 * pb], wyB * d1[2 * pb + 1]);   // x node xA + 2
          v[pb][0] = fma(wxA, sA, wxB * sB);
          if (FM == 1) {   // column moments in tile coordinates
            v[pb][1] = fma((double)xA * wxA, sA, (double)(xA + 2) * wxB * sB);
            const double yAd = (double)yA;
            const double tA = fma(yAd * wyA, d0[2 * pb], (yAd + 1.0) * wyB * d0[2 * pb + 1]);
            const double tB = fma(yAd * wyA, d1[2 * pb], (yAd + 1.0) * wyB * d1[2 * pb + 1]);
            v[pb][2] = fma(wxA, tA, wxB * tB);
          }
        }
        const bool b1 = tg & 1;
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const double send = b1 ? v[0][cc] : v[1][cc];
          double x = (b1 ? v[1][cc] : v[0][cc]) + __shfl_xor_sync(0xffffffffu, send, 1);
          x += __shfl_xor_sync(0xffffffffu, x, 2);
          if (tg < 2) acc[(int64_t)(b1 ? eg8 : eg) * ACS + w * NC + cc] = x;
        }
      };
      if (T16) {
        for (int k = k0; k < k1; k += 16) gstep16(k);
      } else {
        int k = k0;
        for (; k + 16 <= k1 && kGU == 2; k += 16) gstep(std::integral_constant<int, kGU>(), k);
        for (; k < k1; k += 8) gstep(std::integral_constant<int, 1>(), k);
      }
    }
  };

  int held = 0, bprev = -1;
#if SE1P_SWEEP_TRACE
  int kc = -1;
#endif
  for (int b = 0, ph = 0;; b = (b + 1 == NB) ? 0 : b + 1, ph ^= (b == 0)) {
    mbar_wait(&full[b], (unsigned)ph, 400000 + b);
#if SE1P_SWEEP_TRACE
    ++kc;
#endif
    SW_CTRACE(4);
    const int4 h = hdr[b];
    if (h.w & kKernelEnd) {
      __syncwarp();
      if (lane == 0) {
        if (bprev >= 0) mbar_arrive(&empty[bprev]);
        mbar_arrive(&empty[b]);
      }
      break;
    }
    if (h.x != cur) {
      cur = h.x;
      item_geom(cur, X0, Y0, Z0, Ck, zc);
      flushed = 0;
      fr = false;
      if (GATHER) {
        const int x0 = X0 + 4 * bxw + (g >> 2), x1 = x0 + 2, y = Y0 + 4 * byw + (g & 3);
        gp0 = (x0 < Mt && y < Mt) ? A.grid + ((int64_t)x0 * Mt + y) * M : nullptr;
        gp1 = (x1 < Mt && y < Mt) ? A.grid + ((int64_t)x1 * Mt + y) * M : nullptr;
      }
    }
    if (h.w & kItemEnd) {
      if (!GATHER) {
        __syncwarp();
        for (; flushed < Ck + P - 1; flushed += 8) flush_block(flushed);
        __syncwarp();
      }
      if (lane == 0) {
        if (bprev >= 0) mbar_arrive(&empty[bprev]);
        mbar_arrive(&empty[b]);
      }
      bprev = -1;
      continue;
    }
    if (h.w & kFirst) {
      u = h.y;
      if (!GATHER) {
        __syncwarp();
        for (; flushed + 8 <= u; flushed += 8) flush_block(flushed);
        __syncwarp();
      }
      fr = false;
    }
    // this warp's list of the batch (built by the expanders), after the held entries: positions
    // [0, held) are cb, [held, tot) are L
    SW_CTRACE(8);
    unsigned short* Lw = lists + (b * kCW + w) * LS;
    int n = 0;
    if (XL) {
      n = lcnt[b * kCW + w];
    } else {
      for (int p0 = 0; p0 < h.z; p0 += 32) {
        const int p = p0 + lane;
        const bool rel = p < h.z && ((mask[b * BM + p] >> w) & 1);
        const unsigned bal = __ballot_sync(0xffffffffu, rel);
        if (rel) Lw[n + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)(b * BM + p);
        n += __popc(bal);
      }
      __syncwarp();
    }
    const int tot = held + n;
    SW_CTRACE(9);
    // k-steps of 8 entries; the group's last batch pads and runs everything, and so does a batch
    // that cannot fill one k-step on top of held entries (at most one batch is ever held)
    int kend = tot & ~(KS - 1);
    if ((h.w & kLast) || (held > 0 && kend == 0)) {
      kend = (tot + KS - 1) & ~(KS - 1);
      if (lane < kend - tot) Lw[n + lane] = (unsigned short)dummy;
      __syncwarp();
    }
    unsigned short* cb = cbw + 16 * cbsel;         // this batch's held entries (from bprev)
    unsigned short* cbn = cbw + 16 * (cbsel ^ 1);  // its own left-overs for the next batch
    const int rest = max(tot - kend, 0);   // < KS, all from this batch (none after padding)
    if (lane < rest) cbn[lane] = Lw[kend - held + lane];
    if (kend > 0) {
      if (!fr) {
        if (GATHER) frame_load_gather();
        else frame_io(false);
        fr = true;
      }
      if (held > 0) {   // one mixed k-step: the held entries (batch bprev), then this batch's first
        if (lane >= held && lane < KS) cb[lane] = Lw[lane - held];
        __syncwarp();
        ksteps(cb, 0, KS);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[bprev]);
        bprev = -1;
        ksteps(Lw + KS - held, 0, kend - KS);
      } else {
        ksteps(Lw, 0, kend);
      }
    }
    SW_CTRACE(10);
    if (rest > 0) cbsel ^= 1;
    held = rest;
    if (h.w & kLast) {
      if (!GATHER && fr) {
        __syncwarp();
        frame_io(true);
      }
      fr = false;
    }
    SW_CTRACE(11);
    __syncwarp();
    if (held == 0) {
      if (lane == 0) mbar_arrive(&empty[b]);
    } else {
      bprev = b;
    }
#if SE1P_SWEEP_TRACE
    if (w == 0 && lane == 0) {
      SW_TRACE(kc, 5, clock64());
      SW_TRACE(kc, 6, kend / KS);
      SW_TRACE(kc, 7, h.z);
    }
#endif
  }
}

#if SE1P_SWEEP_TRACE
extern "C" int se1p_sweep_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
}
#endif

// Overhang: the P-1 positions past each chunk belong to the next chunk (periodic in z); every
// position receives at most one overhang (chunks hold >= P-1 nodes), so the adds do not race.
__global__ void k_overhang(const double* __restrict__ over, double* __restrict__ grid, int Mt, int M, int P, int C,
                           int nzc, int x_lo, int x_hi) {
  // one thread per (chunk, column, overhang node): contiguous reads of the overhang, runs of
  // consecutive z in the grid column
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ncol = (int64_t)(x_hi - x_lo) * Mt;
  if (i >= ncol * nzc * (P - 1)) return;
  const int64_t cc = i / (P - 1);
  const int t = (int)(i - cc * (P - 1));
  const int zc = (int)(cc / ncol);
  const int64_t col = (int64_t)x_lo * Mt + (cc - (int64_t)zc * ncol);
  const int Z0 = zc * C, Ck = min(C, M - Z0);
  int z = Z0 + Ck + t;
  while (z >= M) z -= M;
  grid[col * M + z] += over[((int64_t)zc * Mt * Mt + col) * (P - 1) + t];
}

// Items (tx | ty << 10 | zc << 20) ordered by candidate count, heaviest first (ties: index order).
// (weights staged in shared memory when they fit: SW)
template <bool SW>
__global__ void k_items(int ntx, int tx_lo, int nty, int nzc, int Mfree, int P, int* __restrict__ items,
                        int* __restrict__ counter) {
  extern __shared__ int wsm[];
  const int n = ntx * nty * nzc;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) counter[0] = 0;
  auto wt = [&](int j) {
    const int zc = j % nzc, t2 = j / nzc, ty = t2 % nty, tx = t2 / nty + tx_lo;
    (void)zc;
    const int X0 = tx * kTXY, Y0 = ty * kTXY;
    const int wx = max(0, min(X0 + kTXY - 1, Mfree) - max(X0 - P + 1, 1) + 1);
    const int wy = max(0, min(Y0 + kTXY - 1, Mfree) - max(Y0 - P + 1, 1) + 1);
    return wx * wy;
  };
  if (SW) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) wsm[j] = wt(j);
    __syncthreads();
  }
  if (i >= n) return;
  const int wi = SW ? wsm[i] : wt(i);
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    const int wj = SW ? wsm[j] : wt(j);
    rank += (wj > wi) || (wj == wi && j < i);
  }
  const int zc = i % nzc, t2 = i / nzc, ty = t2 % nty, tx = t2 / nty + tx_lo;
  items[rank] = tx | (ty << 10) | (zc << 20);
}

// Records of the sorted particles, stride rec_stride(NZB): {jx0, jy0} (reading R-3),
// q, per free axis the Fast Gaussian Gridding factors of the first stencil node offset d0,
// A = e^{-alpha d0^2}, E = e^{-2 alpha h d0} (node t: A E^t f1[t]) with E^-1 and E^8 for the
// sweeps' power trees, d0 per axis, the record's own sorted index, and the periodic-axis window
// wz[t] = e^{-alpha (d0z + t h)^2} for t < P (zero up to 8 NZB).
__global__ void __launch_bounds__(128) k_records(KDev dv, const double4* __restrict__ P4, const int4* __restrict__ S4,
                                                int64_t N, int RD, double* __restrict__ rec) {
  extern __shared__ double srec[];   // 128 records, written out by the block with coalesced stores
  const int64_t i0 = (int64_t)blockIdx.x * 128, i = i0 + threadIdx.x;
  const int nrec = (int)(N - i0 < 128 ? N - i0 : 128);
  if (i < N) {
    const double4 pp = P4[i];
    const int4 s = S4[i];
    const double P2 = 0.5 * dv.P;
    const double d0[3] = {((double)s.x - P2) * dv.h - pp.x, ((double)s.y - P2) * dv.h - pp.y,
                          (double)s.z * dv.h - pp.z};
    const double ah = 2.0 * dv.alpha * dv.h;
    double* r = srec + threadIdx.x * (RD + 1);   // odd stride: conflict-free per-thread rows
    r[0] = __hiloint2double(s.y, s.x);
    r[kRq] = pp.w;
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      double* ra = r + (ax == 0 ? kRx : kRy);
      ra[0] = exp(-dv.alpha * d0[ax] * d0[ax]);
      ra[1] = exp(-ah * d0[ax]);
      ra[2] = exp(ah * d0[ax]);
      ra[3] = exp(-8.0 * ah * d0[ax]);
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) r[kRd + ax] = d0[ax];
    r[kRi] = __longlong_as_double((long long)i);   // the sorted index (gather slots)
    r[kRi + 1] = r[kRi + 2] = 0.0;
    // z window by the FGG recurrence: e^{-alpha (d0 + t h)^2} = A E^t f1[t], with
    // E^t f1[t] = prod_{s<t} E e^{-alpha h^2 (2s+1)}
    const double g2 = exp(-2.0 * dv.alpha * dv.h * dv.h);
    double wv = exp(-dv.alpha * d0[2] * d0[2]), step = exp(-ah * d0[2]) * exp(-dv.alpha * dv.h * dv.h);
    for (int t = 0; t < RD - kRz; ++t) {
      r[kRz + t] = (t < dv.P) ? wv : 0.0;
      wv *= step;
      step *= g2;
    }
  }
  __syncthreads();
  double2* dst = reinterpret_cast<double2*>(rec + i0 * RD);
  for (int k = threadIdx.x; k < nrec * RD / 2; k += 128) {
    const int row = (2 * k) / RD, col = 2 * k - row * RD;   // RD even: a pair never straddles rows
    const double* sp = srec + row * (RD + 1) + col;
    dst[k] = make_double2(sp[0], sp[1]);
  }
}

// The field's second gather pass: the z windows become 2 alpha (node - z_p) wz (d/dz_p of the
// window, Eq. (force_se1p)), in place.
__global__ void k_records_zderiv(KDev dv, int64_t N, int RD, double* __restrict__ rec) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double* r = rec + i * RD;
  const double dz = r[kRd + 2], ta = 2.0 * dv.alpha;
  for (int t = 0; t < RD - kRz; ++t) r[kRz + t] *= ta * fma((double)t, dv.h, dz);
}

// Sum the per-tile partials of every particle in a fixed order and scatter to user order.
// Only x tiles in [txlo, txhi) are summed (one slab of the distributed path; all tiles otherwise).
// FIELD: the slots hold (phi, dphi/dx, dphi/dy, dphi/dz); field = -grad phi (3 per particle).
template <bool FIELD>
__global__ void k_gather_finish(KDev dv, const int4* __restrict__ S4, const int* __restrict__ perm,
                                const double* __restrict__ gpart, int64_t N, double* __restrict__ phi,
                                double* __restrict__ field, int txlo, int txhi) {
  constexpr int NC = FIELD ? 4 : 1;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int4 st = S4[p];
  const int P = dv.P;
  const int tx0 = fdiv(st.x, kTXY), ty0 = fdiv(st.y, kTXY);
  const int nx = fdiv(st.x + P - 1, kTXY) - tx0 + 1;
  const int ny = fdiv(st.y + P - 1, kTXY) - ty0 + 1;
  // slot-major partials [slot][value][particle]: consecutive particles at consecutive addresses
  const double* gq = gpart + p;
  double s[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) s[c] = 0.0;
  for (int a = 0; a < nx; ++a) {
    if (tx0 + a < txlo || tx0 + a >= txhi) continue;
    for (int b = 0; b < ny; ++b)
#pragma unroll
      for (int c = 0; c < NC; ++c) s[c] += gq[(int64_t)((a * dv.nsxy + b) * NC + c) * N];
  }
  const int64_t u = perm[p];
  if (phi) phi[u] = s[0];
  if (FIELD)
#pragma unroll
    for (int c = 0; c < 3; ++c) field[3 * u + c] = -s[1 + c];
}

// ------------------------------------------------------------------ host side
int rec_doubles(int P) { return rec_stride(sw_nzb(P)); }

void slot_geometry(KDev& dv) {
  dv.nsxy = (dv.P - 1 + kTXY - 1) / kTXY + 1;
  dv.nsz = 1;
  dv.nslot = dv.nsxy * dv.nsxy;
}

int64_t gather_slots(const KDev& dv) {
  KDev d = dv;
  slot_geometry(d);
  return d.nslot;
}

// chunking of the periodic axis: enough items for ~4 per SM, chunks of >= max(P, 16) nodes,
// multiples of 8 (the flush blocks)
static void sweep_chunks(const KDev& dv, int ncol, int& C, int& nzc) {
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  const int M = dv.M, P = dv.P;
  nzc = 1;
  C = M;
  for (int z = 2; z <= 64; ++z) {
    if ((int64_t)ncol * nzc >= 4 * (int64_t)n_sm) break;
    const int c = (int)ceil_div(ceil_div(M, z), 8) * 8;
    if (c < std::max(P, 16)) break;
    const int nz = (int)ceil_div(M, c);
    if (M - (nz - 1) * c < P - 1) continue;   // the last chunk must hold an overhang
    if (nz > nzc) {
      nzc = nz;
      C = c;
    }
  }
}

// the largest chunk count sweep_chunks can pick: chunks of >= max(P, 16) nodes
static int64_t sweep_nzc_max(const KDev& dv) { return dv.M / std::max(dv.P, 16) + 1; }
int64_t sweep_overhang_doubles(const KDev& dv) {
  return sweep_nzc_max(dv) * dv.Mt * dv.Mt * std::max(dv.P - 1, 1);
}
int64_t sweep_items_max(const KDev& dv) {
  const int64_t nt = ceil_div(dv.Mt, kTXY);
  return nt * nt * sweep_nzc_max(dv) + 2;
}

void k_records_stage(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, bool field) {
  (void)field;
  const int nz = sw_nzb(pl.dv.P);
  const int RD = rec_stride(nz);
  const size_t sm = 128 * (RD + 1) * sizeof(double);
  if (sm > 48 * 1024)
    SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_records, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_records<<<(unsigned)ceil_div(N, 128), 128, sm, st>>>(pl.dv, (const double4*)w.xs, (const int4*)w.s4, N, RD,
                                                         w.rec);
  SE1P_LAUNCH_CHECK();
}

template <bool GATHER, int FM, int NZB>
static void launch_sweep_t(const KPlan& pl, KWork& w, int64_t N, int tx_lo, int tx_hi, cudaStream_t st) {
  SweepArgs a;
  a.dv = pl.dv;
  KDev& dv = a.dv;
  slot_geometry(dv);
  dv.err = w.flag + 1;
  dv.N = N;
  const int nty = (int)ceil_div(dv.Mt, kTXY), ntx = tx_hi - tx_lo;
  if (ntx <= 0) return;
  sweep_chunks(dv, ntx * nty, a.C, a.nzc);
  a.n_items = ntx * nty * a.nzc;
  // item table (heavy first); k_items also zeroes the work counter
  if (w.items_cap < a.n_items + 2) throw Error{6, "sweep item table not allocated"};
  if ((size_t)a.n_items * sizeof(int) <= 48 * 1024)
    k_items<true><<<(unsigned)ceil_div(a.n_items, 256), 256, (size_t)a.n_items * sizeof(int), st>>>(
        ntx, tx_lo, nty, a.nzc, dv.Mfree, dv.P, w.items, w.items + a.n_items);
  else
    k_items<false><<<(unsigned)ceil_div(a.n_items, 256), 256, 0, st>>>(ntx, tx_lo, nty, a.nzc, dv.Mfree, dv.P,
                                                                       w.items, w.items + a.n_items);
  SE1P_LAUNCH_CHECK();
  a.items = w.items;
  a.counter = w.items + a.n_items;
  a.rec = w.rec;
  a.bin_start = w.bin_start;
  a.f1 = pl.d_f1;
  a.grid = w.grid;
  a.over = w.over;
  a.gpart = GATHER ? w.gpart : nullptr;
  int BM = 0, NB = 0;
  const int limit = 227 * 1024 - 512;
  for (int nb : {kNB, 2})
    for (int bm = 128; bm >= 8 && !BM; bm -= 8)
      if (sweep_smem(bm, nb, NZB, GATHER, FM).total <= limit) {
        BM = bm;
        NB = nb;
      }
  if (!BM) throw Error{4, "sweep kernels do not fit in shared memory"};
  a.BM = BM;
  a.NB = NB;
  const size_t smem = (size_t)sweep_smem(BM, NB, NZB, GATHER, FM).total;
  SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_sweep<GATHER, FM, NZB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  const unsigned nblk = (unsigned)std::min(a.n_items, n_sm);
  k_sweep<GATHER, FM, NZB><<<nblk, kSweepThreads, smem, st>>>(a);
  SE1P_LAUNCH_CHECK();
  if (!GATHER && dv.P > 1) {
    const int x_lo = tx_lo * kTXY, x_hi = std::min(tx_hi * kTXY, dv.Mt);
    const int64_t n = (int64_t)a.nzc * (x_hi - x_lo) * dv.Mt * (dv.P - 1);
    k_overhang<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(w.over, w.grid, dv.Mt, dv.M, dv.P, a.C, a.nzc, x_lo, x_hi);
    SE1P_LAUNCH_CHECK();
  }
}

template <bool GATHER, int FM>
static void launch_sweep(const KPlan& pl, KWork& w, int64_t N, int tx_lo, int tx_hi, cudaStream_t st) {
  if (pl.dv.P > kMaxP) throw Error{4, "P > 64 is not supported by the sweep kernels"};
  if (tx_hi < 0) tx_hi = (int)ceil_div(pl.dv.Mt, kTXY);
  switch (sw_nzb(pl.dv.P)) {
    case 2: launch_sweep_t<GATHER, FM, 2>(pl, w, N, tx_lo, tx_hi, st); break;
    case 3: launch_sweep_t<GATHER, FM, 3>(pl, w, N, tx_lo, tx_hi, st); break;
    case 4: launch_sweep_t<GATHER, FM, 4>(pl, w, N, tx_lo, tx_hi, st); break;
    default: launch_sweep_t<GATHER, FM, 8>(pl, w, N, tx_lo, tx_hi, st); break;
  }
}

void k_spread_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo, int tx_hi) {
  launch_sweep<false, 0>(pl, w, N, tx_lo, tx_hi, st);
}

void k_gather_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo, int tx_hi, bool field) {
  if (field) {
    launch_sweep<true, 1>(pl, w, N, tx_lo, tx_hi, st);   // phi, d/dx, d/dy
    k_records_zderiv<<<(unsigned)ceil_div(N, 128), 128, 0, st>>>(pl.dv, N, rec_stride(sw_nzb(pl.dv.P)), w.rec);
    SE1P_LAUNCH_CHECK();
    launch_sweep<true, 2>(pl, w, N, tx_lo, tx_hi, st);   // d/dz
  } else {
    launch_sweep<true, 0>(pl, w, N, tx_lo, tx_hi, st);
  }
}

void k_gather_finish_stage(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st, int tx_lo, int tx_hi,
                           double* field) {
  KDev dv = pl.dv;
  slot_geometry(dv);
  if (tx_hi < 0) tx_hi = (int)ceil_div(dv.Mt, kTXY);
  const unsigned nb = (unsigned)ceil_div(N, 256);
  const int4* s4 = (const int4*)w.s4;
  if (field) k_gather_finish<true><<<nb, 256, 0, st>>>(dv, s4, w.perm, w.gpart, N, phi, field, tx_lo, tx_hi);
  else k_gather_finish<false><<<nb, 256, 0, st>>>(dv, s4, w.perm, w.gpart, N, phi, field, tx_lo, tx_hi);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
