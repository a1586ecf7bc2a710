// tiles.cu -- gridding (Alg. 1 step 2, Eq. (spread_1p)) and gather (Alg. 1 step 6,
// Eq. (se1p_complete_discretized)) as output-stationary tile contractions on the
// FP64 tensor pipe (mma.sync m16n8k8 f64 -> SASS DMMA).  See tiles.cuh.
//
// Weights: k_records evaluates every sorted particle's 3 x P one-dimensional window weights
// e^{-alpha d^2} once per call into a record row (tiles.cuh), so that the P^3 stencil is the
// outer product of three staged vectors (the separability that Fast Gaussian Gridding, P:807-817,
// exploits on the CPU).
//
// One CTA per tile X0..X0+15 x Y0..Y0+15 x Z0..Z0+TZ-1 (periodic in z), 17 warps:
//   producer warp: walks the tile's candidate bins (xy columns of 4 x 4 cells, z-sorted) in
//     z windows of kWinCells cells, columns concatenated inside a window, and moves the records
//     of each contiguous run with one bulk copy (cp.async.bulk, SASS UBLKCP) into a ring of NB
//     shared-memory batches of BM rows; completion is signalled by transaction bytes on the
//     batch's `full` mbarrier.  Gather: it also reduces the finished batches' per-warp partials.
//   16 consumer warps: warp w owns the 4 x 4 column block (4 (w&3), 4 (w>>2)) over all TZ
//     nodes; per batch it keeps the particles meeting its block (order preserving) and runs
//       gridding  C[16 cols x 8 z]        += A[16 cols x 8 particles] B[8 particles x 8 z]
//                 A = q wx wy (built from the staged rows), B = wz
//       gather    T[16 cols x 8 particles] = A[16 cols x 8 z] (H~, registers) B[8 z x 8 particles]
//                 phi_p += sum_cols wx wy T
//     skipping 8-node z blocks no particle of the k-step reaches; then arrives on `empty`.
// No floating-point atomics: gridding writes its tile once; the gather writes one partial per
// (particle, tile) into a fixed slot and k_gather_finish sums the slots in a fixed order, so
// results are bitwise reproducible.
#include <cstdint>
#include <cstdlib>

#include "tiles.cuh"

namespace se1p {

constexpr int kCW = 16;                      // consumer warps
constexpr int kThreads = (kCW + 1) * 32;     // + 1 producer warp
constexpr int kMaxNB = 4;

struct TileArgs {
  KDev dv;
  const double* rec;
  const int* bin_start;
  double* grid;
  double* gpart;
  int ntz, nty, tx_lo;   // launched tiles: tx in [tx_lo, tx_lo + gridDim/(nty ntz))
  int BM, NB, RS;
};

struct TileSmem {
  int off_pidx, off_lists, off_acc, off_buf, total;
};

__host__ __device__ inline TileSmem tile_smem(int BM, int NB, int RS, bool gather) {
  TileSmem s;
  int o = 2 * kMaxNB * 8 + kMaxNB * 4;   // barriers, counts
  s.off_pidx = o;
  o += kMaxNB * BM * 4;
  o = (o + 15) & ~15;
  s.off_lists = o;
  o += kCW * (BM + 16) * 8;
  o = (o + 15) & ~15;
  s.off_acc = o;
  if (gather) o += NB * BM * (kCW + 1) * 8;
  o = (o + 127) & ~127;
  s.off_buf = o;
  o += NB * (BM + 1) * RS * 8;
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
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  while (!mbar_try_wait(b, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ int clampw(int t, int P) { return min(max(t, -1), P); }
// bits of the 8-node z blocks covering tile offsets [lo, hi), hi > lo
__device__ __forceinline__ int zbits(int lo, int hi) { return ((1 << ((hi + 7) >> 3)) - 1) & ~((1 << (lo >> 3)) - 1); }

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

template <int TZ, bool GATHER, bool WRAP2>
__global__ void __launch_bounds__(kThreads, 1) k_tiles(const TileArgs A) {
  constexpr int NZB = TZ / 8;
  extern __shared__ __align__(128) unsigned char smem[];
  const KDev& dv = A.dv;
  const int BM = A.BM, NB = A.NB, RS = A.RS, P = dv.P, M = dv.M, Mt = dv.Mt;
  const int WXo = rec_wx(), WYo = rec_wy(P), WZo = rec_wz(P);
  const TileSmem L = tile_smem(BM, NB, RS, GATHER);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxNB;
  int* cnt = reinterpret_cast<int*>(empty + kMaxNB);
  int* pidx = reinterpret_cast<int*>(smem + L.off_pidx);
  int2* lists = reinterpret_cast<int2*>(smem + L.off_lists);
  double* acc = reinterpret_cast<double*>(smem + L.off_acc);
  double* bufs = reinterpret_cast<double*>(smem + L.off_buf);
  const int BS = (BM + 1) * RS;   // doubles per batch buffer (row BM: all zero)

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int tz = blockIdx.x % A.ntz, t2 = blockIdx.x / A.ntz;
  const int ty = t2 % A.nty, tx = A.tx_lo + t2 / A.nty;
  const int X0 = tx * kTXY, Y0 = ty * kTXY, Z0 = tz * TZ;
  const int jmax = min(TZ, M - Z0);

  if (tid == 0) {
    for (int b = 0; b < kMaxNB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int b = 0; b < NB; ++b)
    for (int k = tid; k < RS; k += kThreads) bufs[b * BS + BM * RS + k] = 0.0;
  if (GATHER)
    for (int k = tid; k < NB * BM * (kCW + 1); k += kThreads) acc[k] = 0.0;
  __syncthreads();

  if (w == kCW) {
    // ================================================================ producer
    const int nslot = dv.nslot;
    auto reduce = [&](int b) {   // gather: sum the per-warp partials of batch buffer b
      const int c = cnt[b];
      const double* bb = bufs + b * BS;
      for (int p = lane; p < c; p += 32) {
        const int4 s = *reinterpret_cast<const int4*>(bb + p * RS);
        double* ap = acc + (b * BM + p) * (kCW + 1);
        const bool hx = s.x <= X0 + kTXY - 1 && s.x + P - 1 >= X0 && s.y <= Y0 + kTXY - 1 && s.y + P - 1 >= Y0;
        const int sz = hx ? zslot(s.w, P, M, TZ, tz) : -1;
        if (sz >= 0) {
          double sum = 0.0;
#pragma unroll
          for (int v = 0; v < kCW; ++v) {
            sum += ap[v];
            ap[v] = 0.0;
          }
          const int sx = tx - fdiv(s.x, kTXY), sy = ty - fdiv(s.y, kTXY);
          A.gpart[(int64_t)pidx[b * BM + p] * nslot + (sx * dv.nsxy + sy) * dv.nsz + sz] = sum;
        } else if (hx) {
          for (int v = 0; v < kCW; ++v)
            if (ap[v] != 0.0) atomicOr(dv.err, 8);   // consumer listed a particle the slot map lacks
        }
      }
      __syncwarp();
    };

    int k = 0, fill = 0, b = 0;
    bool have = false;
    auto acquire = [&]() {
      b = k % NB;
      if (k >= NB) {
        mbar_wait(&empty[b], (unsigned)(((k - NB) / NB) & 1));
        if (GATHER) reduce(b);
      }
      have = true;
    };
    auto publish = [&](int c) {
      __threadfence_block();
      __syncwarp();
      if (lane == 0) {
        cnt[b] = c;
        mbar_arrive(&full[b]);
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
    int sN, eN;
    load_run(lane, sN, eN);
    for (int q0 = 0; q0 < npc; q0 += 32) {
      const int sC = sN, eC = eN;
      load_run(q0 + 32 + lane, sN, eN);   // prefetch the next 32 runs
      const int nq = min(32, npc - q0);
      for (int i = 0; i < nq; ++i) {
        int s = __shfl_sync(0xffffffffu, sC, i);
        int n = __shfl_sync(0xffffffffu, eC, i) - s;
        while (n > 0) {
          if (!have) acquire();
          const int take = min(n, BM - fill);
          double* dst = bufs + b * BS + fill * RS;
          if (lane == 0) {
            const unsigned bytes = (unsigned)(take * RS * 8);
            mbar_expect_tx(&full[b], bytes);
            bulk_g2s(dst, A.rec + (int64_t)s * RS, bytes, &full[b]);
          }
          for (int l = lane; l < take; l += 32) pidx[b * BM + fill + l] = s + l;
          fill += take;
          s += take;
          n -= take;
          if (fill == BM) publish(BM);
        }
      }
    }
    if (fill > 0) publish(fill);
    acquire();
    publish(-1);   // end marker
    if (GATHER) {
      const int kend = k;   // batches 0 .. kend-2 are real; those < kend-NB were reduced already
      for (int j = max(0, kend - NB); j <= kend - 2; ++j) {
        mbar_wait(&empty[j % NB], (unsigned)((j / NB) & 1));
        reduce(j % NB);
      }
    }
    return;
  }

  // ================================================================ consumers
  // List entry per relevant particle: x = p | zmask << 8 | (ox + 8) << 16 | (oy + 8) << 24 with
  // ox = X0b - jx0, oy = Y0b - jy0 (window offsets of the warp block), y = the z offset:
  //   WRAP2:  d = (Z0 - a) mod M, stencil index of tile node j is (d + j) mod M
  //   else:   e = signed tile offset of the stencil start, stencil index of node j is j - e
  const int gid = lane >> 2, tig = lane & 3;
  const int X0b = X0 + 4 * (w & 3), Y0b = Y0 + 4 * (w >> 2);
  int2* wl = lists + w * (BM + 16);
  const int2 dummy = make_int2(BM | (8 << 16) | (8 << 24), WRAP2 ? 0 : -P);
  auto zidx = [&](int y, int j) -> int {   // stencil index of tile node j, clamped onto a guard
    if (WRAP2) {
      int t = y + j;
      t -= (t >= M) ? M : 0;
      return min(t, P);
    }
    return clampw(j - y, P);
  };

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

  for (int b = 0, ph = 0;; b = (b + 1 == NB) ? 0 : b + 1, ph ^= (b == 0)) {
    mbar_wait(&full[b], (unsigned)ph);
    const int cn = cnt[b];
    if (cn < 0) break;
    const double* bb = bufs + b * BS;
    // particles of the batch meeting this warp's 4 x 4 column block (order preserving)
    int n = 0;
    for (int p0 = 0; p0 < ((dv.dbg & 4) ? 0 : cn); p0 += 32) {
      const int p = p0 + lane;
      bool rel = false;
      int2 e = dummy;
      if (p < cn) {
        const int4 s = *reinterpret_cast<const int4*>(bb + p * RS);
        const int ox = X0b - s.x, oy = Y0b - s.y;
        if (ox >= -3 && ox <= P - 1 && oy >= -3 && oy <= P - 1) {
          int d = Z0 - s.w;
          if (d < 0) d += M;
          const int zm = zmask_of(d, P, M, jmax);
          rel = zm != 0;
          e = make_int2(p | (zm << 8) | ((ox + 8) << 16) | ((oy + 8) << 24), WRAP2 ? d : (d < P ? -d : M - d));
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, rel);
      if (rel) wl[n + __popc(bal & ((1u << lane) - 1u))] = e;
      n += __popc(bal);
    }
    const int npad = (n + 15) & ~15;
    if (lane < npad - n) wl[n + lane] = dummy;
    __syncwarp();

    if (dv.dbg & 2) {
    } else if (!GATHER) {
      // C[16 cols x 8 z] += A[16 cols x 16 particles] B[16 particles x 8 z]; particle of k-slot
      // tig + 4j is list entry k + tig + 4j (A and B agree on it)
      const int cx = gid & 3, cy = gid >> 2;
      for (int k = 0; k < npad; k += 16) {
        int2 e[4];
        int zm = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          e[j] = wl[k + tig + 4 * j];
          zm |= e[j].x;
        }
        zm = (zm >> 8) & 0xff;
        zm |= __shfl_xor_sync(0xffffffffu, zm, 1);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 2);
        double a[8];
        const double* rz[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double* r = bb + (e[j].x & 0xff) * RS;
          const int ox = ((e[j].x >> 16) & 0xff) - 8, oy = ((unsigned)e[j].x >> 24) - 8;
          const double wq = r[2] * r[WXo + clampw(ox + cx, P)];
          a[2 * j] = wq * r[WYo + clampw(oy + cy, P)];
          a[2 * j + 1] = wq * r[WYo + clampw(oy + cy + 2, P)];
          rz[j] = r + WZo;
        }
#pragma unroll
        for (int zb = 0; zb < NZB; ++zb) {
          if (((zm >> zb) & 1) && !(dv.dbg & 1)) {
            const int jz = 8 * zb + gid;
            dmma_16x8x16(c[zb], a, rz[0][zidx(e[0].y, jz)], rz[1][zidx(e[1].y, jz)], rz[2][zidx(e[2].y, jz)],
                         rz[3][zidx(e[3].y, jz)]);
          }
        }
      }
    } else {
      // T[16 particles x 8 cols] = A[16 particles x 8 z] (wz) B[8 z x 8 cols] (H~), per col half;
      // particle of row gid (gid + 8) is list entry k + gid (k + gid + 8)
      for (int k = 0; k < npad; k += 16) {
        const int2 e0 = wl[k + gid], e1 = wl[k + gid + 8];
        int zm = ((e0.x | e1.x) >> 8) & 0xff;
        zm |= __shfl_xor_sync(0xffffffffu, zm, 4);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 8);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 16);
        const double* r0 = bb + (e0.x & 0xff) * RS;
        const double* r1 = bb + (e1.x & 0xff) * RS;
        double t0[4] = {0.0, 0.0, 0.0, 0.0}, t1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int zb = 0; zb < NZB; ++zb) {
          if (((zm >> zb) & 1) && !(dv.dbg & 1)) {
            const int j0 = 8 * zb + tig, j1 = j0 + 4;
            const double a[4] = {r0[WZo + zidx(e0.y, j0)], r1[WZo + zidx(e1.y, j0)], r0[WZo + zidx(e0.y, j1)],
                                 r1[WZo + zidx(e1.y, j1)]};
            dmma_16x8x8(t0, a, hB[zb][0][0], hB[zb][0][1]);
            dmma_16x8x8(t1, a, hB[zb][1][0], hB[zb][1][1]);
          }
        }
        // this thread's cols: x = 2 (tig & 1) + {0, 1}, y = (tig >> 1) + {0 (half 0), 2 (half 1)}
        const int cx0 = 2 * (tig & 1), cy0 = tig >> 1;
        double v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int2 eh = h ? e1 : e0;
          const double* r = h ? r1 : r0;
          const int ox = ((eh.x >> 16) & 0xff) - 8, oy = ((unsigned)eh.x >> 24) - 8;
          const double wx0 = r[WXo + clampw(ox + cx0, P)], wx1 = r[WXo + clampw(ox + cx0 + 1, P)];
          const double wy0 = r[WYo + clampw(oy + cy0, P)], wy2 = r[WYo + clampw(oy + cy0 + 2, P)];
          v[h] = wy0 * fma(wx0, t0[2 * h], wx1 * t0[2 * h + 1]) + wy2 * fma(wx0, t1[2 * h], wx1 * t1[2 * h + 1]);
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        v[1] += __shfl_xor_sync(0xffffffffu, v[1], 1);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
        v[1] += __shfl_xor_sync(0xffffffffu, v[1], 2);
        if (tig == 0) {
          const int pa = e0.x & 0xff, pb = e1.x & 0xff;
          if (pa < BM) acc[(b * BM + pa) * (kCW + 1) + w] = v[0];
          if (pb < BM) acc[(b * BM + pb) * (kCW + 1) + w] = v[1];
        }
      }
      __threadfence_block();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
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
template <int TZ>
__global__ void k_gather_finish(KDev dv, const int4* __restrict__ S4, const int* __restrict__ perm,
                                const double* __restrict__ gpart, int64_t N, double* __restrict__ phi, int txlo,
                                int txhi) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int4 st = S4[p];
  const int P = dv.P;
  const int nx = fdiv(st.x + P - 1, kTXY) - fdiv(st.x, kTXY) + 1;
  const int ny = fdiv(st.y + P - 1, kTXY) - fdiv(st.y, kTXY) + 1;
  const int nz = zcount(st.w, P, dv.M, TZ);
  const double* g = gpart + p * dv.nslot;
  double s = 0.0;
  const int tx0 = fdiv(st.x, kTXY);
  for (int a = 0; a < nx; ++a) {
    if (tx0 + a < txlo || tx0 + a >= txhi) continue;
    for (int b = 0; b < ny; ++b)
      for (int z = 0; z < nz; ++z) s += g[(a * dv.nsxy + b) * dv.nsz + z];
  }
  phi[perm[p]] = s;
}

// Record rows of the sorted particles (layout in tiles.cuh).  Window weights by Fast Gaussian
// Gridding: with d0 the signed distance from the particle to the first stencil node,
//   e^{-alpha (d0 + t h)^2} = e^{-alpha d0^2} (e^{-2 alpha h d0})^t e^{-alpha h^2 t^2},
// i.e. two exponentials per particle and axis plus the particle-independent table f1[t]
// (reading R-3 for the node positions).  kRecPB particles per block are assembled in shared
// memory and written out as one coalesced run.
constexpr int kRecPB = 16;

__global__ void __launch_bounds__(128) k_records(KDev dv, const double4* __restrict__ P4, const int4* __restrict__ S4,
                                                 int64_t N, int RS, const double* __restrict__ f1,
                                                 double* __restrict__ rec) {
  extern __shared__ __align__(16) double srow[];
  const int P = dv.P;
  const int64_t i0 = (int64_t)blockIdx.x * kRecPB;
  const int np = (int)((N - i0 < kRecPB) ? (N - i0) : kRecPB);
  for (int k = threadIdx.x; k < kRecPB * RS; k += blockDim.x) srow[k] = 0.0;
  __syncthreads();
  if (threadIdx.x < 3 * np) {
    const int p = threadIdx.x / 3, ax = threadIdx.x - 3 * p;
    const int64_t i = i0 + p;
    const double4 pp = P4[i];
    const int4 s = S4[i];
    double* row = srow + p * RS;
    double d0;
    int off;
    if (ax == 0) {
      d0 = ((double)s.x - 0.5 * P) * dv.h - pp.x;
      off = rec_wx();
      reinterpret_cast<int4*>(row)[0] = s;
      row[2] = pp.w;
    } else if (ax == 1) {
      d0 = ((double)s.y - 0.5 * P) * dv.h - pp.y;
      off = rec_wy(P);
    } else {
      d0 = (double)s.z * dv.h - pp.z;
      off = rec_wz(P);
    }
    double g = exp(-dv.alpha * d0 * d0);
    const double E = exp(-2.0 * dv.alpha * dv.h * d0);
    for (int t = 0; t < P; ++t) {
      row[off + t] = g * f1[t];
      g *= E;
    }
  }
  __syncthreads();
  const double2* src = reinterpret_cast<const double2*>(srow);
  double2* dst = reinterpret_cast<double2*>(rec + i0 * RS);
  for (int k = threadIdx.x; k < np * RS / 2; k += blockDim.x) dst[k] = src[k];
}

int tile_tz(int M) { return M >= 64 ? 32 : 16; }

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

void k_records_stage(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st) {
  const int RS = rec_stride(pl.dv.P);
  const size_t smem = sizeof(double) * kRecPB * RS;
  if (smem > 48 * 1024)
    SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_records, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_records<<<(unsigned)ceil_div(N, kRecPB), 128, smem, st>>>(pl.dv, (const double4*)w.xs, (const int4*)w.s4, N, RS,
                                                               pl.d_f1, w.rec);
  SE1P_LAUNCH_CHECK();
}

template <int TZ, bool GATHER, bool WRAP2>
static void launch_tiles(const KPlan& pl, KWork& w, int64_t N, int tx_lo, int tx_hi, cudaStream_t st) {
  TileArgs a;
  a.dv = pl.dv;
  KDev& dv = a.dv;
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
  const int ntx = tx_hi - tx_lo;
  if (ntx <= 0) return;
  a.RS = rec_stride(dv.P);
  a.rec = w.rec;
  a.bin_start = w.bin_start;
  a.grid = w.grid;
  a.gpart = GATHER ? w.gpart : nullptr;
  int BM = 0, NB = 0;
  const int limit = 227 * 1024 - 1024;
  for (int bm : {64, 32, 16}) {
    for (int nb = kMaxNB; nb >= 2 && !BM; --nb)
      if (tile_smem(bm, nb, a.RS, GATHER).total <= limit) {
        BM = bm;
        NB = nb;
      }
    if (BM) break;
  }
  if (!BM) throw Error{4, "P too large for the tile kernels (shared memory)"};
  a.BM = BM;
  a.NB = NB;
  const size_t smem = (size_t)tile_smem(BM, NB, a.RS, GATHER).total;
  SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_tiles<TZ, GATHER, WRAP2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  const unsigned nblk = (unsigned)(ntx * a.nty * a.ntz);
  k_tiles<TZ, GATHER, WRAP2><<<nblk, kThreads, smem, st>>>(a);
  SE1P_LAUNCH_CHECK();
}

// WRAP2: a stencil can meet a z tile twice (both ends of the periodic axis) iff TZ + P > M.
template <bool GATHER>
static void dispatch_tiles(const KPlan& pl, KWork& w, int64_t N, int tx_lo, int tx_hi, cudaStream_t st) {
  const int TZ = tile_tz(pl.dv.M);
  const bool wrap2 = TZ + pl.dv.P > pl.dv.M;
  if (tx_hi < 0) tx_hi = (int)ceil_div(pl.dv.Mt, kTXY);
  if (TZ == 32) {
    if (wrap2) launch_tiles<32, GATHER, true>(pl, w, N, tx_lo, tx_hi, st);
    else launch_tiles<32, GATHER, false>(pl, w, N, tx_lo, tx_hi, st);
  } else {
    if (wrap2) launch_tiles<16, GATHER, true>(pl, w, N, tx_lo, tx_hi, st);
    else launch_tiles<16, GATHER, false>(pl, w, N, tx_lo, tx_hi, st);
  }
}

void k_spread_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo, int tx_hi) {
  dispatch_tiles<false>(pl, w, N, tx_lo, tx_hi, st);
}

void k_gather_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo, int tx_hi) {
  dispatch_tiles<true>(pl, w, N, tx_lo, tx_hi, st);
}

void k_gather_finish_stage(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st, int tx_lo, int tx_hi) {
  KDev dv = pl.dv;
  slot_geometry(dv);
  if (tx_hi < 0) tx_hi = (int)ceil_div(dv.Mt, kTXY);
  const unsigned nb = (unsigned)ceil_div(N, 256);
  if (tile_tz(dv.M) == 32)
    k_gather_finish<32><<<nb, 256, 0, st>>>(dv, (const int4*)w.s4, w.perm, w.gpart, N, phi, tx_lo, tx_hi);
  else
    k_gather_finish<16><<<nb, 256, 0, st>>>(dv, (const int4*)w.s4, w.perm, w.gpart, N, phi, tx_lo, tx_hi);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
