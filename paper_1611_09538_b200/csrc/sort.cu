// sort.cu -- deterministic stable sort of particles into bins (cells / tiles).
//
// The gridding and gather kernels visit particles bin by bin; a stable order (by original
// index inside a bin) makes every floating-point reduction order fixed, so results are
// bitwise reproducible without floating-point atomics.
//
//   bin_start: per-bin counts (integer atomics, order independent) -> exclusive scan
//   perm:      LSD radix sort of (key, index) pairs, ceil(log2 nbins) bits in passes of <= 8
//              bits; every pass is stable: per-block digit histograms -> digit-major exclusive
//              scan -> each block scatters its elements in input order (warps in order, 32
//              elements at a time, equal digits ranked with __match_any_sync).
#include <algorithm>

#include "sort.cuh"

namespace se1p {

constexpr int kSortThreads = 256, kSortItems = 8, kSortTile = kSortThreads * kSortItems;
constexpr int kScanThreads = 1024, kScanItems = 4, kScanTile = kScanThreads * kScanItems;

// ------------------------------------------------------------------ exclusive scan (n -> n+1)
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns the block total in *tot
__device__ int block_excl_scan(int v, int* sw, int* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int inc = warp_incl_scan(v, lane);
  if (lane == 31) sw[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int s = (lane < nw) ? sw[lane] : 0;
    const int si = warp_incl_scan(s, lane);
    if (lane < nw) sw[lane] = si - s;
    if (lane == nw - 1) sw[32] = si;
  }
  __syncthreads();
  const int r = sw[w] + inc - v;
  *tot = sw[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const int* __restrict__ in, int64_t n, int* __restrict__ out,
                                                             int* __restrict__ bsum) {
  __shared__ int sw[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems], s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0;
    s += v[k];
  }
  int tot;
  int run = block_excl_scan(s, sw, &tot);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// single block: exclusive scan of the tile sums in place (any count, sequential chunks with a
// carry), total -> out[n]
__global__ void __launch_bounds__(kScanThreads) k_scan_top(int* __restrict__ bsum, int nb, int* __restrict__ out, int64_t n) {
  __shared__ int sw[33];
  int carry = 0;
  for (int c0 = 0; c0 < nb; c0 += kScanThreads) {
    const int i = c0 + threadIdx.x;
    const int v = (i < nb) ? bsum[i] : 0;
    int tot;
    const int r = block_excl_scan(v, sw, &tot);
    if (i < nb) bsum[i] = carry + r;
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(int* __restrict__ out, int64_t n, const int* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  const int add = bsum[blockIdx.x];
  for (int k = threadIdx.x; k < kScanTile; k += kScanThreads)
    if (base + k < n) out[base + k] += add;
}

static void excl_scan(const int* in, int64_t n, int* out, int* bsum, cudaStream_t st) {
  const int nb = (int)ceil_div(n, kScanTile);
  k_scan_tiles<<<nb, kScanThreads, 0, st>>>(in, n, out, bsum);
  SE1P_LAUNCH_CHECK();
  k_scan_top<<<1, kScanThreads, 0, st>>>(bsum, nb, out, n);
  SE1P_LAUNCH_CHECK();
  if (nb > 1) {
    k_scan_add<<<nb, kScanThreads, 0, st>>>(out, n, bsum);
    SE1P_LAUNCH_CHECK();
  }
}

// ------------------------------------------------------------------ bin counts
__global__ void k_bin_count(const int* __restrict__ keys, int64_t N, int* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) atomicAdd(&cnt[keys[i]], 1);
}

// ------------------------------------------------------------------ radix passes
__global__ void __launch_bounds__(kSortThreads) k_rs_up(const int* __restrict__ keys, int64_t N, int shift, int R,
                                                        int nblk, int* __restrict__ ghist) {
  __shared__ int h[256];
  for (int d = threadIdx.x; d < R; d += kSortThreads) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int k = threadIdx.x; k < kSortTile; k += kSortThreads)
    if (base + k < N) atomicAdd(&h[(keys[base + k] >> shift) & (R - 1)], 1);
  __syncthreads();
  for (int d = threadIdx.x; d < R; d += kSortThreads) ghist[(int64_t)d * nblk + blockIdx.x] = h[d];
}

// vals_in == nullptr: the values are the input positions (first pass)
__global__ void __launch_bounds__(kSortThreads) k_rs_down(const int* __restrict__ kin, const int* __restrict__ vin,
                                                          int64_t N, int shift, int R, int nblk,
                                                          const int* __restrict__ goff, int* __restrict__ kout,
                                                          int* __restrict__ vout) {
  constexpr int NW = kSortThreads / 32, PER = kSortTile / NW;
  __shared__ int wofs[NW][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < NW * 256; k += kSortThreads) (&wofs[0][0])[k] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kSortTile + (int64_t)w * PER;
  for (int s = 0; s < PER; s += 32) {   // per-warp digit counts
    const int64_t i = wbase + s + lane;
    if (i < N) atomicAdd(&wofs[w][(kin[i] >> shift) & (R - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < R; d += kSortThreads) {   // warp offsets, warps in order
    int run = goff[(int64_t)d * nblk + blockIdx.x];
    for (int v = 0; v < NW; ++v) {
      const int c = wofs[v][d];
      wofs[v][d] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int s = 0; s < PER; s += 32) {
    const int64_t i = wbase + s + lane;
    const bool act = i < N;
    const unsigned mask = __ballot_sync(0xffffffffu, act);
    if (act) {
      const int key = kin[i];
      const int d = (key >> shift) & (R - 1);
      const unsigned peers = __match_any_sync(mask, d);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int pos = wofs[w][d] + rank;
      kout[pos] = key;
      vout[pos] = vin ? vin[i] : (int)i;
      __syncwarp(mask);
      if (rank == 0) wofs[w][d] += __popc(peers);
    }
    __syncwarp();
  }
}

void exclusive_scan_ints(const int* in, int64_t n, int* out, int* scratch, cudaStream_t st) {
  excl_scan(in, n, out, scratch, st);
}
int64_t scan_scratch_ints(int64_t n) { return ceil_div(n + 1, kScanTile) + 16; }

int64_t sort_scratch_ints(int64_t N, int nbins) {
  const int64_t nblk = ceil_div(N, kSortTile);
  const int64_t gh = 256 * nblk + 1;
  const int64_t scan_max = std::max<int64_t>(gh, (int64_t)nbins + 1);
  return 3 * N + gh + (int64_t)nbins + 1 + ceil_div(scan_max, kScanTile) + 16;
}

void stable_bin_sort(const int* keys, int64_t N, int nbins, int* perm, int* bin_start, int* scratch, cudaStream_t st) {
  const int nblk = (int)ceil_div(N, kSortTile);
  int* kA = scratch;
  int* kB = kA + N;
  int* vA = kB + N;
  int* ghist = vA + N;
  int* cnt = ghist + 256 * (int64_t)nblk + 1;
  int* bsum = cnt + nbins + 1;
  // bin_start
  SE1P_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)nbins, st));
  k_bin_count<<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(keys, N, cnt);
  SE1P_LAUNCH_CHECK();
  excl_scan(cnt, nbins, bin_start, bsum, st);
  // perm: LSD radix passes; the last pass writes perm directly
  int bits = 1;
  while ((1ll << bits) < (long long)nbins) ++bits;
  const int passes = (bits + 7) / 8;
  const int per = (bits + passes - 1) / passes;
  const int* kin = keys;
  const int* vin = nullptr;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * per, R = 1 << std::min(per, bits - shift);
    k_rs_up<<<nblk, kSortThreads, 0, st>>>(kin, N, shift, R, nblk, ghist);
    SE1P_LAUNCH_CHECK();
    excl_scan(ghist, (int64_t)R * nblk, ghist, bsum, st);
    int* kout = (p & 1) ? kB : kA;
    int* vout = ((passes - 1 - p) % 2 == 0) ? perm : vA;   // the last pass lands in perm
    k_rs_down<<<nblk, kSortThreads, 0, st>>>(kin, vin, N, shift, R, nblk, ghist, kout, vout);
    SE1P_LAUNCH_CHECK();
    kin = kout;
    vin = vout;
  }
}

}  // namespace se1p
