// dmma_tiles.cu -- gridding (Alg. 1 step 2, Eq. (spread_1p)) and gather (Alg. 1
// step 6, Eq. (se1p_complete_discretized)) as output-stationary tile contractions on
// the FP64 tensor pipe (mma.sync m16n8k4 f64 -> SASS DMMA).  See tiles.cuh.
//
// Weights: k_stencil_weights evaluates every particle's 3 x P one-dimensional window weights
// e^{-alpha d^2} once per call (W[i][axis][t], t = stencil offset).  A tile then only COPIES
// the parts of those rows that fall inside it.
//
// One CTA per tile X0..X0+15 x Y0..Y0+15 x Z0..Z0+TZ-1 (periodic in z):
//   producer warps (kPW): stream the candidate particles of the tile (bins are xy columns of
//     8 x 8 cells, z-sorted inside), keep those whose P^3 stencil meets the tile (order-
//     preserving compaction) into a ring of records; every kStage records form a batch,
//     published into one of kNBuf shared-memory weight buffers;
//   staging: per particle one warp unit copies the tile windows of its rows with cp.async
//     (zero-fill outside the stencil); units are claimed through an atomic counter by any free
//     warp (producers after publishing, consumers when they reach the batch);
//   consumer warps (kCW = 16): each owns a 4 x 4 column block over all TZ nodes and runs
//       gridding  C[16 cols x 8 z]        += A[16 cols x 4 particles] B[4 particles x 8 z]
//                 A = q wx wy, B = wz
//       gather    T[16 cols x 8 particles] = A[16 cols x 4 z] (H~, registers) B[4 z x 8 particles]
//                 phi_p += sum_cols wx wy T
//     on the staged particles meeting its block, skipping 8-node z blocks no particle of the
//     k-step reaches.
// Consumers arrive on a named "empty" barrier after a batch; producers sync on it before
// reusing that buffer.  Gridding writes its tile once (no floating-point atomics); the gather
// writes one partial per (particle, tile) into a fixed slot and k_gather_finish sums the slots
// in a fixed order: results are bitwise reproducible.
#include <cstdlib>

#include "tiles.cuh"

namespace se1p {

constexpr int kCW = 16, kPW = 4;
constexpr int kPT = kPW * 32;                 // producer threads
constexpr int kCT = kCW * 32;                 // consumer threads
constexpr int kThreads = kCT + kPT;           // 640
constexpr int kNBuf = 3;
constexpr int kRing = 1024;                   // candidate records (>= (kNBuf + 2) kStage + kPre kPT)
constexpr int kPre = 4;                       // candidates per producer thread per round
constexpr int kWin = 4;                       // z cells per candidate window
constexpr int kBarProd = 1;                   // producer-internal barrier id
__host__ __device__ constexpr int bar_full(int b) { return 2 + b; }
__host__ __device__ constexpr int bar_empty(int b) { return 2 + kNBuf + b; }

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// 8-byte global -> shared async copy; src_bytes = 0 writes zeros (cp.async zero-fill)
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

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

// Does the stencil (jx0, jy0, lz0, a = lz0 mod M) meet tile (tx,ty,tz)?  Agrees with the slot
// ranges of k_gather_finish: x tiles fdiv(jx0,16)..fdiv(jx0+P-1,16) (no wrap), z per zslot.
template <int TZ>
__device__ __forceinline__ bool tile_hit(const KDev& dv, const int4& s, int tx, int ty, int tz) {
  const int P = dv.P;
  if (tx < fdiv(s.x, kTXY) || tx > fdiv(s.x + P - 1, kTXY)) return false;
  if (ty < fdiv(s.y, kTXY) || ty > fdiv(s.y + P - 1, kTXY)) return false;
  return zslot(s.w, P, dv.M, TZ, tz) >= 0;
}

template <int TZ>
struct Buf {   // one staged batch
  static constexpr int SZ = TZ + 4;
  double wx[(kStage + 1) * kSX];
  double wy[(kStage + 1) * kSX];
  double wz[(kStage + 1) * SZ];
  double acc[kStage * (kCW + 1)];
  double q[kStage + 1];
  int64_t slot[kStage];   // gather: destination of each particle's partial in gpart
  int xr[kStage + 1], yr[kStage + 1], zm[kStage + 1];
  int cnt;       // particles (< 0: end of stream)
  int rec;       // ring position of the first record
  int claim;     // staging units claimed
  int done;      // staging units finished
};

template <int TZ>
struct Smem {
  Buf<TZ> buf[kNBuf];
  double pq[kRing];         // charge
  int4 ps[kRing];           // stencil starts
  int pi[kRing];            // sorted particle index
  int pcnt[kPW];
  int cs[64], csz[64], cpre[65];   // candidate window: per-column start, size, exclusive prefix
  int wl[kCW][kStage + 8];
};

template <int TZ>
__host__ __device__ constexpr size_t tile_smem_bytes() { return sizeof(Smem<TZ>); }

template <int TZ, bool GATHER>
__global__ void __launch_bounds__(kThreads, 1)
    k_tile_mma(KDev dv, const double4* __restrict__ P4, const int4* __restrict__ S4, const double* __restrict__ W,
               const int* __restrict__ bin_start, double* __restrict__ grid, double* __restrict__ gpart, int ntz) {
  constexpr int NZB = TZ / 8;
  constexpr int SZ = Buf<TZ>::SZ;
  constexpr int NK = TZ / 4;
  extern __shared__ __align__(16) char smem_raw[];
  Smem<TZ>& S = *reinterpret_cast<Smem<TZ>*>(smem_raw);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int tz = blockIdx.x % ntz, t2 = blockIdx.x / ntz;
  const int ty = t2 % dv.nty2, tx = t2 / dv.nty2;
  const int X0 = tx * kTXY, Y0 = ty * kTXY, Z0 = tz * TZ;
  const int M = dv.M, P = dv.P;

  for (int b = 0; b < kNBuf; ++b) {   // dummy all-zero row (index kStage) of every buffer
    Buf<TZ>& B = S.buf[b];
    for (int k = tid; k < kSX; k += kThreads) {
      B.wx[kStage * kSX + k] = 0.0;
      B.wy[kStage * kSX + k] = 0.0;
    }
    for (int k = tid; k < SZ; k += kThreads) B.wz[kStage * SZ + k] = 0.0;
    if (tid == 0) {
      B.xr[kStage] = B.yr[kStage] = B.zm[kStage] = 0;
      B.q[kStage] = 0.0;
    }
  }
  __syncthreads();

  // ---- staging unit: warp-wide, one particle p of buffer B (async copies, no wait here)
  auto stage_unit = [&](Buf<TZ>& B, int p) {
    const int rr = (B.rec + p) & (kRing - 1);
    const int4 s = S.ps[rr];
    int i = S.pi[rr];
    if ((unsigned)i >= (unsigned)dv.N || (unsigned)p >= (unsigned)kStage) {   // never expected
      atomicOr(dv.err, 1 | (p >= kStage ? 2 : 0));
      i = 0;
    }
    const double* row = W + (int64_t)i * 3 * P;
    {   // x (lanes 0-15) and y (lanes 16-31)
      const int ax = lane >> 4, k = lane & 15;
      const int t = (ax == 0 ? X0 - s.x : Y0 - s.y) + k;
      const bool v = t >= 0 && t < P;
      cp_async8((ax == 0 ? B.wx : B.wy) + p * kSX + k, row + ax * P + (v ? t : 0), v ? 8 : 0);
    }
    bool in = false;
    if (lane < TZ) {   // z: lane = window node
      const int g = Z0 + lane;
      int t = g - s.w;
      if (t < 0) t += M;
      in = (g < M) && (t < P);
      cp_async8(B.wz + p * SZ + lane, row + 2 * P + (in ? t : 0), in ? 8 : 0);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) {
      int mask = 0;
#pragma unroll
      for (int zb = 0; zb < NZB; ++zb) mask |= ((bal >> (8 * zb)) & 0xffu) ? (1 << zb) : 0;
      B.zm[p] = mask;
      B.xr[p] = (max(s.x, X0) - X0) | ((min(s.x + P, X0 + kTXY) - X0) << 8);
      B.yr[p] = (max(s.y, Y0) - Y0) | ((min(s.y + P, Y0 + kTXY) - Y0) << 8);
      if (GATHER) {
        const int sx = tx - fdiv(s.x, kTXY), sy = ty - fdiv(s.y, kTXY);
        const int sz = zslot(s.w, P, M, TZ, tz);
        B.slot[p] = (int64_t)i * dv.nslot + (sx * dv.nsxy + sy) * dv.nsz + sz;
      } else {
        B.q[p] = S.pq[rr];
      }
    }
    if (GATHER && lane < kCW + 1) B.acc[p * (kCW + 1) + lane] = 0.0;
  };
  // claim and process units of B until none is left (warp-uniform), then publish completion
  auto help_stage = [&](Buf<TZ>& B, int cnt) {
    int mine = 0;
    for (;;) {
      int u = 0;
      if (lane == 0) u = atomicAdd(&B.claim, 1);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u >= cnt) break;
      stage_unit(B, u);
      ++mine;
    }
    if (mine) {
      cp_async_wait_all();
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicAdd(&B.done, mine);
    }
  };

  if (w >= kCW) {
    // ================================================================ producers
    const int ptid = tid - kCT, pw = w - kCW;
    unsigned long long t_wait = 0, t_stage = 0, t_all0 = clock64();
    int nbatch = 0, npend = 0, nwaited = 0, head = 0, tail = 0;

    auto reduce = [&](int b) {   // sum the per-warp partials of a finished gather batch
      if (!GATHER) return;
      Buf<TZ>& B = S.buf[b];
      const int cnt = B.cnt;
      for (int p = ptid; p < cnt; p += kPT) {
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < kCW; ++v) s += B.acc[p * (kCW + 1) + v];
        const int64_t sl = B.slot[p];
        if (sl < 0 || sl >= dv.N * dv.nslot) atomicOr(dv.err, 4);   // never expected
        else gpart[sl] = s;
      }
    };
    auto wait_empty = [&](int batch) {   // buffer of `batch` is free again (consumers done)
      const int b = batch % kNBuf;
      const unsigned long long t0 = clock64();
      bar_sync(bar_empty(b), kThreads);
      if (*(volatile int*)&S.buf[b].cnt == -12345) S.pcnt[0] = 0;   // charge the lazy wait here
      t_wait += clock64() - t0;
      reduce(b);
      ++nwaited;
    };
    auto publish = [&](int cnt) {   // records head .. head+cnt-1 form the next batch (cnt < 0: end)
      const int b = nbatch % kNBuf;
      if (nbatch >= kNBuf) wait_empty(nbatch - kNBuf);
      Buf<TZ>& B = S.buf[b];
      bar_sync(kBarProd, kPT);   // every producer finished reading the old batch (reduce)
      if (ptid == 0) {
        B.cnt = cnt;
        B.rec = head & (kRing - 1);
        B.claim = 0;
        B.done = 0;
      }
      bar_arrive(bar_full(b), kThreads);
      const unsigned long long ts = clock64();
      if (cnt > 0 && !(dv.dbg & 2)) help_stage(B, cnt);
      t_stage += clock64() - ts;
      ++nbatch;
      if (cnt > 0) head += cnt;
    };

    // candidate stream, interleaved over the xy bin columns (8x8 cells, z-sorted by cell inside):
    // z windows of kWin cells, and inside a window the columns' ranges concatenated, so every
    // batch spreads over the whole tile (balanced consumer warps) and stays z-coherent.
    const int bx0 = max(0, fdiv(X0 - P, kTX)), bx1 = min(dv.nbx - 1, fdiv(X0 + kTXY - 1, kTX));
    const int by0 = max(0, fdiv(Y0 - P, kTY)), by1 = min(dv.nby - 1, fdiv(Y0 + kTXY - 1, kTY));
    const int nbyc = by1 - by0 + 1, ncol = max(0, (bx1 - bx0 + 1) * nbyc);
    // cells whose stencil may reach the tile: nodes lz0..lz0+P-1 with lz0 = floor(z/h - P/2)+1,
    // i.e. cz - (P+1)/2 <= lz0 <= cz - P/2 + 1 (exact test: tile_hit)
    int czs = Z0 - P / 2 - 1, span = TZ + P + 2;
    if (span >= M) { czs = 0; span = M; }
    for (int w0 = 0; w0 < span;) {
      const int a = pmod(czs + w0, M);
      const int len = min(min(kWin, span - w0), M - a);   // a window never crosses the periodic seam
      w0 += len;
      if (ptid < ncol) {
        const int c = ptid, bx = bx0 + c / nbyc, by = by0 + c - (c / nbyc) * nbyc;
        const int base = (bx * dv.nby + by) * M + a;
        const int s = bin_start[base];
        S.cs[c] = s;
        S.csz[c] = bin_start[base + len] - s;
      }
      bar_sync(kBarProd, kPT);
      if (pw == 0) {   // exclusive prefix of the column sizes (<= 64 columns, 2 per lane)
        const int v0 = (2 * lane < ncol) ? S.csz[2 * lane] : 0, v1 = (2 * lane + 1 < ncol) ? S.csz[2 * lane + 1] : 0;
        int x = v0 + v1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const int ex = x - v0 - v1;
        S.cpre[2 * lane] = ex;
        S.cpre[2 * lane + 1] = ex + v0;
        if (lane == 31) S.cpre[64] = x;
      }
      bar_sync(kBarProd, kPT);
      const int total_w = S.cpre[64];
      for (int c00 = 0; c00 < total_w; c00 += kPre * kPT) {
        int4 sv[kPre];
        bool relv[kPre];
        double qv[kPre];
        int idxv[kPre];
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          const int vi = c00 + u * kPT + ptid;
          relv[u] = false;
          idxv[u] = 0;
          if (vi < total_w) {
            int lo = 0, hi = ncol - 1;   // last column with cpre[c] <= vi
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (S.cpre[mid] <= vi) lo = mid; else hi = mid - 1;
            }
            const int idx = S.cs[lo] + (vi - S.cpre[lo]);
            idxv[u] = idx;
            sv[u] = S4[idx];
            if (!GATHER) qv[u] = P4[idx].w;
            relv[u] = tile_hit<TZ>(dv, sv[u], tx, ty, tz);
          }
        }
        // ordered compaction of the kPre rounds: per-warp counts packed in one int
        unsigned bals[kPre];
        int packed = 0;
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          bals[u] = __ballot_sync(0xffffffffu, relv[u]);
          packed |= __popc(bals[u]) << (8 * u);
        }
        if (lane == 0) S.pcnt[pw] = packed;
        bar_sync(kBarProd, kPT);
        int off[kPre], total = 0;
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          int o = total, t = 0;
#pragma unroll
          for (int v = 0; v < kPW; ++v) {
            const int cv = (S.pcnt[v] >> (8 * u)) & 255;
            if (v < pw) o += cv;
            t += cv;
          }
          off[u] = o;
          total += t;
        }
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          if (relv[u]) {
            const int rr = (tail + off[u] + __popc(bals[u] & ((1u << lane) - 1u))) & (kRing - 1);
            S.pi[rr] = idxv[u];
            S.ps[rr] = sv[u];
            if (!GATHER) S.pq[rr] = qv[u];
          }
        }
        bar_sync(kBarProd, kPT);
        tail += total;
        npend += total;
        while (npend >= kStage) {
          publish(kStage);
          npend -= kStage;
        }
      }
    }
    if (npend > 0) publish(npend);
    const int nreal = nbatch;
    publish(-1);   // end marker
    for (int j = nwaited; j < nreal; ++j) wait_empty(j);
    if (dv.prof && lane == 0) {
      const unsigned long long tall = clock64() - t_all0;
      atomicAdd(dv.prof + 0, tall);                     // producer warp total
      atomicAdd(dv.prof + 1, t_wait);                   // waiting for free buffers
      atomicAdd(dv.prof + 2, t_stage);                  // helping to stage
      atomicAdd(dv.prof + 3, tall - t_wait - t_stage);  // candidate filtering
      if (pw == 0) atomicAdd(dv.prof + 4, (unsigned long long)nreal);
    }
    return;
  }

  // ================================================================ consumers
  const int gid = lane >> 2, tig = lane & 3;
  const int bxw = w & 3, byw = w >> 2;
  const int colx = X0 + 4 * bxw + (gid & 3), coly = Y0 + 4 * byw + (gid >> 2);
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
  int* wl = S.wl[w];
  unsigned long long c_wait = 0, c_stage = 0, c_all0 = clock64(), c_dmma = 0;
  for (int batch = 0;; ++batch) {
    const int b = batch % kNBuf;
    Buf<TZ>& B = S.buf[b];
    unsigned long long t0 = clock64();
    bar_sync(bar_full(b), kThreads);
    const int cnt = *(volatile int*)&B.cnt;
    unsigned long long t1 = clock64();
    c_wait += t1 - t0;
    if (cnt < 0) break;
    help_stage(B, cnt);
    while (*(volatile int*)&B.done < cnt) __nanosleep(32);
    __threadfence_block();
    t0 = clock64();
    c_stage += t0 - t1;
    // staged particles meeting this warp's 4x4 column block (order preserving)
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
    if (dv.dbg & 1) {
      // experiment: no consumer compute
    } else if (!GATHER) {
      for (int k = 0; k < npad; k += 4) {
        const int p = wl[k + tig];
        const double wxv = B.wx[p * kSX + 4 * bxw + (gid & 3)] * B.q[p];
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
        double t0v[4] = {0.0, 0.0, 0.0, 0.0}, t1v[4] = {0.0, 0.0, 0.0, 0.0};
        const double* wzr = B.wz + pB * SZ + tig;
#pragma unroll
        for (int s = 0; s < NK; s += 2) {      // two accumulators halve the DMMA dependency chain
          if ((zm >> (s >> 1)) & 1) {
            dmma_16x8x4(t0v, hA[s][0], hA[s][1], wzr[4 * s]);
            dmma_16x8x4(t1v, hA[s + 1][0], hA[s + 1][1], wzr[4 * s + 4]);
          }
        }
        const int pa = wl[k + 2 * tig], pb = wl[k + 2 * tig + 1];
        const int ix = 4 * bxw + (gid & 3), iy = 4 * byw + (gid >> 2);
        double va = B.wx[pa * kSX + ix] * fma(B.wy[pa * kSX + iy], t0v[0] + t1v[0], B.wy[pa * kSX + iy + 2] * (t0v[2] + t1v[2]));
        double vb = B.wx[pb * kSX + ix] * fma(B.wy[pb * kSX + iy], t0v[1] + t1v[1], B.wy[pb * kSX + iy + 2] * (t0v[3] + t1v[3]));
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          va += __shfl_xor_sync(0xffffffffu, va, off);
          vb += __shfl_xor_sync(0xffffffffu, vb, off);
        }
        if (gid == 0) {
          if (pa < kStage) B.acc[pa * (kCW + 1) + w] = va;
          if (pb < kStage) B.acc[pb * (kCW + 1) + w] = vb;
        }
      }
    }
    bar_arrive(bar_empty(b), kThreads);
  }
  if (dv.prof && lane == 0) {
    const unsigned long long tall = clock64() - c_all0;
    atomicAdd(dv.prof + 8, tall);                      // consumer warp total
    atomicAdd(dv.prof + 9, c_wait);                    // waiting for published batches
    atomicAdd(dv.prof + 10, c_stage);                  // staging + waiting for staging
    atomicAdd(dv.prof + 11, tall - c_wait - c_stage);  // lists + DMMA k-steps
    atomicAdd(dv.prof + 12, c_dmma);                   // m16n8k4 issued
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

// One-dimensional window weights of every sorted particle: W[i][axis][t] = e^{-alpha d_t^2},
// d_t the signed distance to stencil node t (Eq. (spread_1p) factorised per axis, reading R-3).
__global__ void k_stencil_weights(KDev dv, const double4* __restrict__ P4, const int4* __restrict__ S4, int64_t N,
                                  double* __restrict__ W) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int P = dv.P;
  if (id >= N * 3 * P) return;
  const int64_t i = id / (3 * P);
  const int r = (int)(id - i * 3 * P), ax = r / P, t = r - ax * P;
  const double4 pp = P4[i];
  const int4 s = S4[i];
  double d;
  if (ax == 0) d = ((double)(s.x + t) - 0.5 * P) * dv.h - pp.x;
  else if (ax == 1) d = ((double)(s.y + t) - 0.5 * P) * dv.h - pp.y;
  else d = (double)(s.z + t) * dv.h - pp.z;
  W[id] = exp(-dv.alpha * d * d);
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

void k_weights(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st) {
  const int64_t n = N * 3 * pl.dv.P;
  k_stencil_weights<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(pl.dv, (const double4*)w.xs, (const int4*)w.s4, N,
                                                                 w.wts);
  SE1P_LAUNCH_CHECK();
}

template <int TZ, bool GATHER>
static void launch_tile(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st) {
  KDev dv = pl.dv;
  const int ntz = (int)ceil_div(dv.M, TZ);
  dv.nty2 = (int)ceil_div(dv.Mt, kTXY);
  const int ntx2 = (int)ceil_div(dv.Mt, kTXY);
  slot_geometry(dv);
  dv.prof = w.prof_on ? w.prof + (GATHER ? 16 : 0) : nullptr;
  dv.err = w.flag + 1;
  dv.N = N;
  {
    const char* e = getenv("SE1P_TILE_DBG");
    dv.dbg = e ? atoi(e) : 0;
  }
  const size_t smem = tile_smem_bytes<TZ>();
  SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_tile_mma<TZ, GATHER>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned nblk = (unsigned)(ntx2 * dv.nty2 * ntz);
  k_tile_mma<TZ, GATHER><<<nblk, kThreads, smem, st>>>(dv, (const double4*)w.xs, (const int4*)w.s4, w.wts,
                                                       w.bin_start, w.grid, GATHER ? w.gpart : nullptr, ntz);
  SE1P_LAUNCH_CHECK();
  if (GATHER) {
    k_gather_finish<TZ><<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(dv, (const int4*)w.s4, w.perm, w.gpart, N, phi);
    SE1P_LAUNCH_CHECK();
  }
}

void k_spread_mma(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st) {
  k_weights(pl, w, N, st);
  if (tile_tz(pl.dv.M) == 32) launch_tile<32, false>(pl, w, N, nullptr, st);
  else launch_tile<16, false>(pl, w, N, nullptr, st);
}

void k_gather_mma(const KPlan& pl, KWork& w, int64_t N, double* phi, cudaStream_t st) {
  if (tile_tz(pl.dv.M) == 32) launch_tile<32, true>(pl, w, N, phi, st);
  else launch_tile<16, true>(pl, w, N, phi, st);
}

}  // namespace se1p
