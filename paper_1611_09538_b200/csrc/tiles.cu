// tiles.cu -- gridding (Alg. 1 step 2, Eq. (spread_1p)) and gather (Alg. 1 step 6,
// Eq. (se1p_complete_discretized)) as output-stationary tile contractions on the
// FP64 tensor pipe (mma.sync m16n8k4 f64 -> SASS DMMA).  See tiles.cuh for the decomposition.
//
// One CTA per tile X0..X0+15 x Y0..Y0+15 x Z0..Z0+TZ-1 (periodic in z):
//   producer warps (kPW): stream the candidate particles of the tile (bins are xy columns of
//     8 x 8 cells, z-sorted inside), keep those whose P^3 stencil meets the tile (order-
//     preserving compaction) and hand lists of kStage particles to the consumers through a
//     ring of kNL shared-memory lists (named barriers lfull/lempty);
//   consumer warps (kCW = 16): each owns a 4 x 4 column block over all TZ nodes.  Per batch
//     they (a) stage the NEXT batch's tile-restricted Fast Gaussian Gridding weights into the
//     other half of a double buffer -- w = A E^t f1(t) with A, E per particle and axis from
//     k_permute and f1 a table, no exps here -- and (b) run DMMA on the CURRENT
//     batch for the staged particles meeting their block:
//       gridding  C[16 cols x 8 z]        += A[16 cols x 4 particles] B[4 particles x 8 z]
//       gather    T[16 cols x 8 particles] = A[16 cols x 4 z] (H~, registers) B[4 z x 8 particles]
//                 phi_p += sum_cols wx wy T
//     skipping the 8-node z blocks no particle of the k-step reaches; one consumer barrier
//     per batch.  Staging by all 16 warps interleaves with other warps' DMMA issue.
// Gridding writes its tile once (no atomics); the gather writes one partial per (particle,
// tile) into a fixed slot and k_gather_finish sums the slots in a fixed order: results are
// bitwise reproducible.
#include <cstdlib>

#include "tiles.cuh"

namespace se1p {

constexpr int kCW = 16, kPW = 4;
constexpr int kPT = kPW * 32;                 // producer threads
constexpr int kCT = kCW * 32;                 // consumer threads
constexpr int kThreads = kCT + kPT;           // 640
constexpr int kNL = 4;                        // candidate-list ring
constexpr int kBarProd = 1, kBarCons = 2;
__host__ __device__ constexpr int bar_lfull(int b) { return 3 + b; }
__host__ __device__ constexpr int bar_lempty(int b) { return 3 + kNL + b; }

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// z tiles (extent TZ, the last one ragged) hit by the stencil nodes a, a+1, ..., a+P-1 (mod M),
// a in [0,M): first the tiles of [a, min(a+P,M)), then those of the wrapped part [0, a+P-M)
// not already listed.  zslot gives the canonical position of tile tz (-1: not hit).
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

// Does the stencil (jx0, jy0, lz0 mod M = a) meet tile (tx,ty,tz)?  Agrees with the slot
// ranges of k_gather_finish: x tiles fdiv(jx0,16)..fdiv(jx0+P-1,16) (no wrap), z per zslot.
template <int TZ>
__device__ __forceinline__ bool tile_hit(const KDev& dv, const int4& s, int tx, int ty, int tz) {
  const int P = dv.P;
  if (tx < fdiv(s.x, kTXY) || tx > fdiv(s.x + P - 1, kTXY)) return false;
  if (ty < fdiv(s.y, kTXY) || ty > fdiv(s.y + P - 1, kTXY)) return false;
  return zslot(s.w, P, dv.M, TZ, tz) >= 0;
}

template <int TZ>
struct WBuf {   // staged weights of one batch
  static constexpr int SZ = TZ + 4;
  double wx[(kStage + 1) * kSX];
  double wy[(kStage + 1) * kSX];
  double wz[(kStage + 1) * SZ];
  int xr[kStage + 1], yr[kStage + 1], zm[kStage + 1];
  int pad;
};

struct LBuf {   // a candidate list (sorted particle indices)
  int idx[kStage];
  int cnt;      // < 0: end of stream
  int pad[3];
};

template <int TZ>
struct Smem {
  WBuf<TZ> wb[2];
  double acc[3][kStage * (kCW + 1)];   // gather: partial per (particle, warp), ring of 3 batches
  int sidx[3][kStage];
  int scnt[3];
  int pad0;
  LBuf lb[kNL];
  double f1[64];
  int pend[kPT + kStage];
  int pcnt[kPW];
  int wl[kCW][kStage + 8];
};

template <int TZ>
__host__ __device__ constexpr size_t tile_smem_bytes() { return sizeof(Smem<TZ>); }

template <int TZ, bool GATHER>
__global__ void __launch_bounds__(kThreads, 1)
    k_tile_mma(KDev dv, const double4* __restrict__ P4, const int4* __restrict__ S4, const double* __restrict__ F6,
               const int* __restrict__ bin_start, double* __restrict__ grid, double* __restrict__ gpart, int ntz) {
  constexpr int NZB = TZ / 8;
  constexpr int SZ = WBuf<TZ>::SZ;
  constexpr int NK = TZ / 4;
  extern __shared__ __align__(16) char smem_raw[];
  Smem<TZ>& S = *reinterpret_cast<Smem<TZ>*>(smem_raw);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int tz = blockIdx.x % ntz, t2 = blockIdx.x / ntz;
  const int ty = t2 % dv.nty2, tx = t2 / dv.nty2;
  const int X0 = tx * kTXY, Y0 = ty * kTXY, Z0 = tz * TZ;
  const int M = dv.M, P = dv.P;

  if (w >= kCW) {
    // ================================================================ producers: candidate lists
    const int ptid = tid - kCT, pw = w - kCW;
    unsigned long long t_wait = 0, t_all0 = clock64();
    int nlist = 0, npend = 0;
    auto emit = [&](int cnt) {   // hand S.pend[0..cnt) to the consumers (cnt < 0: end marker)
      const int b = nlist % kNL;
      if (nlist >= kNL) {
        const unsigned long long t0 = clock64();
        bar_sync(bar_lempty(b), kThreads);
        if (*(volatile int*)&S.lb[b].cnt == -12345) S.pcnt[0] = 0;   // charge the lazy wait here
        t_wait += clock64() - t0;
      }
      for (int k = ptid; k < cnt; k += kPT) S.lb[b].idx[k] = S.pend[k];
      if (ptid == 0) S.lb[b].cnt = cnt;
      bar_arrive(bar_lfull(b), kThreads);
      ++nlist;
    };
    const int bx0 = max(0, fdiv(X0 - P, kTX)), bx1 = min(dv.nbx - 1, fdiv(X0 + kTXY - 1, kTX));
    const int by0 = max(0, fdiv(Y0 - P, kTY)), by1 = min(dv.nby - 1, fdiv(Y0 + kTXY - 1, kTY));
    // cells whose stencil may reach the tile: nodes lz0..lz0+P-1 with lz0 = floor(z/h - P/2)+1,
    // i.e. cz - (P+1)/2 <= lz0 <= cz - P/2 + 1 (exact test: tile_hit)
    const int cz0 = Z0 - P / 2 - 1, cz1 = Z0 + TZ + (P + 1) / 2;
    int r0s[2], r1s[2], nr;
    if (cz1 - cz0 + 1 >= M) { r0s[0] = 0; r1s[0] = M - 1; nr = 1; }
    else {
      const int a = pmod(cz0, M), c = pmod(cz1, M);
      if (a <= c) { r0s[0] = a; r1s[0] = c; nr = 1; }
      else { r0s[0] = a; r1s[0] = M - 1; r0s[1] = 0; r1s[1] = c; nr = 2; }
    }
    constexpr int kPre = 4;   // candidate records loaded ahead per thread
    for (int bx = bx0; bx <= bx1; ++bx)
      for (int by = by0; by <= by1; ++by) {
        const int base = (bx * dv.nby + by) * M;
        for (int r = 0; r < nr; ++r) {
          const int s = bin_start[base + r0s[r]], e = bin_start[base + r1s[r] + 1];
          for (int c00 = s; c00 < e; c00 += kPre * kPT) {
            bool relv[kPre];
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
              const int idx = c00 + u * kPT + ptid;
              relv[u] = (idx < e) && tile_hit<TZ>(dv, S4[idx], tx, ty, tz);
            }
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
              if (c00 + u * kPT >= e) break;
              const int idx = c00 + u * kPT + ptid;
              const bool rel = relv[u];
              const unsigned bal = __ballot_sync(0xffffffffu, rel);
              if (lane == 0) S.pcnt[pw] = __popc(bal);
              bar_sync(kBarProd, kPT);
              int off = npend, tot = 0;
#pragma unroll
              for (int v = 0; v < kPW; ++v) {
                const int cv = S.pcnt[v];
                if (v < pw) off += cv;
                tot += cv;
              }
              if (rel) S.pend[off + __popc(bal & ((1u << lane) - 1u))] = idx;
              bar_sync(kBarProd, kPT);
              npend += tot;
              while (npend >= kStage) {
                emit(kStage);
                const int rem = npend - kStage;
                const int v = (ptid < rem) ? S.pend[kStage + ptid] : 0;
                bar_sync(kBarProd, kPT);
                if (ptid < rem) S.pend[ptid] = v;
                bar_sync(kBarProd, kPT);
                npend = rem;
              }
            }
          }
        }
      }
    if (npend > 0) emit(npend);
    emit(-1);   // end marker
    // match the consumers' lempty arrivals of the lists still outstanding
    for (int j = max(0, nlist - kNL); j < nlist; ++j) bar_sync(bar_lempty(j % kNL), kThreads);
    if (dv.prof && lane == 0) {
      const unsigned long long tall = clock64() - t_all0;
      atomicAdd(dv.prof + 0, tall);          // producer warp total
      atomicAdd(dv.prof + 1, t_wait);        // waiting for free list slots
      atomicAdd(dv.prof + 3, tall - t_wait); // candidate filtering
      if (pw == 0) atomicAdd(dv.prof + 4, (unsigned long long)(nlist - 1));
    }
    return;
  }

  // ================================================================ consumers
  const int gid = lane >> 2, tig = lane & 3;
  const int bxw = w & 3, byw = w >> 2;
  const int colx = X0 + 4 * bxw + (gid & 3), coly = Y0 + 4 * byw + (gid >> 2);
  for (int t = tid; t < P; t += kCT) S.f1[t] = exp(-dv.alpha * dv.h * dv.h * (double)t * (double)t);
  for (int b = 0; b < 2; ++b) {   // dummy all-zero row (index kStage)
    WBuf<TZ>& B = S.wb[b];
    if (tid < kSX) {
      B.wx[kStage * kSX + tid] = 0.0;
      B.wy[kStage * kSX + tid] = 0.0;
    }
    if (tid < SZ) B.wz[kStage * SZ + tid] = 0.0;
    if (tid == 0) B.xr[kStage] = B.yr[kStage] = B.zm[kStage] = 0;
  }
  bar_sync(kBarCons, kCT);

  double c[NZB][4];
  double hA[GATHER ? NK : 1][2];
#pragma unroll
  for (int zb = 0; zb < NZB; ++zb) c[zb][0] = c[zb][1] = c[zb][2] = c[zb][3] = 0.0;
  if (GATHER) {
#pragma unroll
    for (int s = 0; s < NK; ++s) {
      const int z = Z0 + 4 * s + tig;
      double a0 = 0.0, a1 = 0.0;
      if (z < M && colx < dv.Mt) {
        if (coly < dv.Mt) a0 = grid[((int64_t)colx * dv.Mt + coly) * M + z];
        if (coly + 2 < dv.Mt) a1 = grid[((int64_t)colx * dv.Mt + coly + 2) * M + z];
      }
      hA[s][0] = a0;
      hA[s][1] = a1;
    }
  }

  // Stage list `L` (cnt particles) into weight buffer B; acc/sidx ring slot `slot`.
  // Task = (particle, axis): 3 cnt tasks spread over all warps (lane-major).
  auto stage = [&](const LBuf& L, int cnt, WBuf<TZ>& B, int slot) {
    const int task = lane * kCW + w;
    if (task < 3 * cnt) {
      const int p = task / 3, ax = task - 3 * p;
      const int i = L.idx[p];
      const int4 s = S4[i];
      double A = F6[6 * (int64_t)i + 2 * ax];
      const double E = F6[6 * (int64_t)i + 2 * ax + 1];
      if (!GATHER && ax == 2) A *= P4[i].w;
      // A E^t for t = 4k + j as four independent chains in k
      const double E2 = E * E, E4 = E2 * E2;
      double Ej[4] = {A, A * E, A * E2, A * E2 * E};
      if (ax < 2) {
        double* row = (ax == 0 ? B.wx : B.wy) + p * kSX;
        const int j0 = ax == 0 ? s.x : s.y;
        const int T0 = ax == 0 ? X0 : Y0;
#pragma unroll
        for (int k = 0; k < kTXY; ++k) row[k] = 0.0;
        for (int t0 = 0; t0 < P; t0 += 4) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + j, k = j0 + t - T0;
            if (t < P && k >= 0 && k < kTXY) row[k] = Ej[j] * S.f1[t];
            Ej[j] *= E4;
          }
        }
        (ax == 0 ? B.xr : B.yr)[p] = (max(j0, T0) - T0) | ((min(j0 + P, T0 + kTXY) - T0) << 8);
      } else {
        double* row = B.wz + p * SZ;
#pragma unroll
        for (int k = 0; k < TZ; ++k) row[k] = 0.0;
        int mask = 0;
        for (int t0 = 0; t0 < P; t0 += 4) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + j;
            int g = s.w + t;
            if (g >= M) g -= M;
            const int gl = g - Z0;
            if (t < P && gl >= 0 && gl < TZ) {
              row[gl] = Ej[j] * S.f1[t];
              mask |= 1 << (gl >> 3);
            }
            Ej[j] *= E4;
          }
        }
        B.zm[p] = mask;
        S.sidx[slot][p] = i;
      }
    }
    if (GATHER)
      for (int k = tid; k < cnt * (kCW + 1); k += kCT) S.acc[slot][k] = 0.0;
    if (tid == 0) S.scnt[slot] = cnt;
  };

  // Sum the per-warp partials of a finished gather batch into the fixed slots.
  auto reduce = [&](int slot) {
    const int cnt = S.scnt[slot];
    for (int p = tid; p < cnt; p += kCT) {
      double s = 0.0;
#pragma unroll
      for (int v = 0; v < kCW; ++v) s += S.acc[slot][p * (kCW + 1) + v];
      const int i = S.sidx[slot][p];
      const int4 st = S4[i];
      const int sx = tx - fdiv(st.x, kTXY), sy = ty - fdiv(st.y, kTXY);
      const int sz = zslot(st.w, P, M, TZ, tz);
      gpart[(int64_t)i * dv.nslot + (sx * dv.nsxy + sy) * dv.nsz + sz] = s;
    }
  };

  // Contract the staged batch B (cnt particles) into this warp's accumulators.
  int* wl = S.wl[w];
  unsigned long long c_dmma = 0;
  auto compute = [&](const WBuf<TZ>& B, int cnt, int slot) {
    int n = 0;
    for (int p0 = 0; p0 < cnt; p0 += 32) {
      const int p = p0 + lane;
      bool rel = false;
      if (p < cnt) {
        const int xr = B.xr[p], yr = B.yr[p];
        rel = (xr & 255) < 4 * bxw + 4 && (xr >> 8) > 4 * bxw && (yr & 255) < 4 * byw + 4 && (yr >> 8) > 4 * byw;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, rel);
      if (rel) wl[n + __popc(bal & ((1u << lane) - 1u))] = p;
      n += __popc(bal);
    }
    constexpr int KS = GATHER ? 8 : 4;
    const int npad = (n + KS - 1) / KS * KS;
    if (lane < npad - n) wl[n + lane] = kStage;
    __syncwarp();
    if (dv.dbg & 1) return;
    if (!GATHER) {
      for (int k = 0; k < npad; k += 4) {
        const int p = wl[k + tig];
        const double wxv = B.wx[p * kSX + 4 * bxw + (gid & 3)];
        const double a0 = wxv * B.wy[p * kSX + 4 * byw + (gid >> 2)];
        const double a1 = wxv * B.wy[p * kSX + 4 * byw + (gid >> 2) + 2];
        int zm = B.zm[p];
        zm |= __shfl_xor_sync(0xffffffffu, zm, 1);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 2);
        c_dmma += __popc(zm);
        const double* wzr = B.wz + p * SZ + gid;
#pragma unroll
        for (int zb = 0; zb < NZB; ++zb)
          if ((zm >> zb) & 1) dmma_16x8x4(c[zb], a0, a1, wzr[zb * 8]);
      }
    } else {
      for (int k = 0; k < npad; k += 8) {
        const int pB = wl[k + gid];
        int zm = B.zm[pB];
        zm |= __shfl_xor_sync(0xffffffffu, zm, 4);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 8);
        zm |= __shfl_xor_sync(0xffffffffu, zm, 16);
        c_dmma += 2 * __popc(zm);
        double t0[4] = {0.0, 0.0, 0.0, 0.0}, t1[4] = {0.0, 0.0, 0.0, 0.0};
        const double* wzr = B.wz + pB * SZ + tig;
#pragma unroll
        for (int s = 0; s < NK; s += 2) {      // two accumulators halve the DMMA dependency chain
          if ((zm >> (s >> 1)) & 1) {
            dmma_16x8x4(t0, hA[s][0], hA[s][1], wzr[4 * s]);
            dmma_16x8x4(t1, hA[s + 1][0], hA[s + 1][1], wzr[4 * s + 4]);
          }
        }
        const int pa = wl[k + 2 * tig], pb = wl[k + 2 * tig + 1];
        const int ix = 4 * bxw + (gid & 3), iy = 4 * byw + (gid >> 2);
        double va = B.wx[pa * kSX + ix] * fma(B.wy[pa * kSX + iy], t0[0] + t1[0], B.wy[pa * kSX + iy + 2] * (t0[2] + t1[2]));
        double vb = B.wx[pb * kSX + ix] * fma(B.wy[pb * kSX + iy], t0[1] + t1[1], B.wy[pb * kSX + iy + 2] * (t0[3] + t1[3]));
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          va += __shfl_xor_sync(0xffffffffu, va, off);
          vb += __shfl_xor_sync(0xffffffffu, vb, off);
        }
        if (gid == 0) {
          if (pa < kStage) S.acc[slot][pa * (kCW + 1) + w] = va;
          if (pb < kStage) S.acc[slot][pb * (kCW + 1) + w] = vb;
        }
      }
    }
  };

  unsigned long long c_wait = 0, c_all0 = clock64(), c_stage = 0;
  auto take_list = [&](int k) -> int {   // wait for list k; returns its count
    const unsigned long long t0 = clock64();
    bar_sync(bar_lfull(k % kNL), kThreads);
    const int cnt = *(volatile int*)&S.lb[k % kNL].cnt;
    c_wait += clock64() - t0;
    return cnt;
  };
  int cur = take_list(0);
  if (cur >= 0) stage(S.lb[0], cur, S.wb[0], 0);
  bar_arrive(bar_lempty(0), kThreads);
  bar_sync(kBarCons, kCT);
  int k = 0;
  while (cur >= 0) {
    if (GATHER && k >= 1) reduce((k - 1) % 3);
    const int nxt = take_list(k + 1);
    const unsigned long long ts = clock64();
    if (nxt >= 0) stage(S.lb[(k + 1) % kNL], nxt, S.wb[(k + 1) & 1], (k + 1) % 3);
    c_stage += clock64() - ts;
    bar_arrive(bar_lempty((k + 1) % kNL), kThreads);
    compute(S.wb[k & 1], cur, k % 3);
    bar_sync(kBarCons, kCT);
    cur = nxt;
    ++k;
  }
  if (GATHER && k >= 1) reduce((k - 1) % 3);
  if (dv.prof && lane == 0) {
    const unsigned long long tall = clock64() - c_all0;
    atomicAdd(dv.prof + 8, tall);       // consumer warp total
    atomicAdd(dv.prof + 9, c_wait);     // waiting for candidate lists
    atomicAdd(dv.prof + 10, c_stage);   // staging
    atomicAdd(dv.prof + 11, tall - c_wait - c_stage);   // DMMA k-steps + barriers
    atomicAdd(dv.prof + 12, c_dmma);    // m16n8k4 issued
  }
  if (!GATHER) {
#pragma unroll
    for (int zb = 0; zb < NZB; ++zb)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int x = colx, y = coly + 2 * (v >> 1), z = Z0 + zb * 8 + 2 * tig + (v & 1);
        if (x < dv.Mt && y < dv.Mt && z < M) grid[((int64_t)x * dv.Mt + y) * M + z] = c[zb][v];
      }
  }
}

// Sum the per-tile partials of every particle in a fixed order and scatter to user order.
template <int TZ>
__global__ void k_gather_finish(KDev dv, const int4* __restrict__ S4, const int* __restrict__ perm,
                                const double* __restrict__ gpart, int64_t N, double* __restrict__ phi) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int4 st = S4[p];
  const int P = dv.P;
  const int nx = fdiv(st.x + P - 1, kTXY) - fdiv(st.x, kTXY) + 1;
  const int ny = fdiv(st.y + P - 1, kTXY) - fdiv(st.y, kTXY) + 1;
  const int nz = zcount(st.w, P, dv.M, TZ);
  const double* g = gpart + p * dv.nslot;
  double s = 0.0;
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < ny; ++b)
      for (int z = 0; z < nz; ++z) s += g[(a * dv.nsxy + b) * dv.nsz + z];
  phi[perm[p]] = s;
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

template <int TZ, bool GATHER>
static void launch_tile(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st) {
  KDev dv = pl.dv;
  const int ntz = (int)ceil_div(dv.M, TZ);
  dv.nty2 = (int)ceil_div(dv.Mt, kTXY);
  const int ntx2 = (int)ceil_div(dv.Mt, kTXY);
  slot_geometry(dv);
  dv.prof = w.prof_on ? w.prof + (GATHER ? 16 : 0) : nullptr;
  {
    const char* e = getenv("SE1P_TILE_DBG");
    dv.dbg = e ? atoi(e) : 0;
  }
  const size_t smem = tile_smem_bytes<TZ>();
  SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_tile_mma<TZ, GATHER>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned nblk = (unsigned)(ntx2 * dv.nty2 * ntz);
  k_tile_mma<TZ, GATHER><<<nblk, kThreads, smem, st>>>(dv, (const double4*)w.xs, (const int4*)w.s4, w.f6,
                                                       w.bin_start, w.grid, GATHER ? w.gpart : nullptr, ntz);
  SE1P_LAUNCH_CHECK();
  if (GATHER) {
    k_gather_finish<TZ><<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(dv, (const int4*)w.s4, w.perm, w.gpart, N, phi);
    SE1P_LAUNCH_CHECK();
  }
}

void k_spread_mma(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st) {
  if (tile_tz(pl.dv.M) == 32) launch_tile<32, false>(pl, w, N, nullptr, st);
  else launch_tile<16, false>(pl, w, N, nullptr, st);
}

void k_gather_mma(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st) {
  if (tile_tz(pl.dv.M) == 32) launch_tile<32, true>(pl, w, N, phi, st);
  else launch_tile<16, true>(pl, w, N, phi, st);
}

}  // namespace se1p
