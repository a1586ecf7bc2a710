// sort.cu -- deterministic stable counting sort of particles into bins (cells / tiles).
//
// The gridding and gather kernels visit particles bin by bin; a stable order (by original
// index inside a bin) makes every floating-point reduction order fixed, so results are
// bitwise reproducible without atomics on floating point data.
//
//   1. per-chunk histograms  hist[c][b]   (chunk = kChunk consecutive input particles)
//   2. column scan over chunks -> per-(chunk,bin) running offsets, bin totals
//   3. exclusive scan of totals -> bin_start[b]
//   4. scatter: one warp per chunk walks its particles in order, 32 at a time; equal keys
//      inside a group are ranked with __match_any_sync, so positions follow input order.
#include "sort.cuh"

namespace se1p {

__global__ void k_hist(const int* __restrict__ keys, int64_t N, int nbins, int* __restrict__ hist) {
  const int64_t c = blockIdx.x;
  const int64_t lo = c * kChunk, hi = ((N < lo + kChunk) ? N : lo + kChunk);
  int* h = hist + c * (int64_t)nbins;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[keys[i]], 1);
}

__global__ void k_colscan(int* __restrict__ hist, int64_t nchunks, int nbins, int* __restrict__ total) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  int run = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    int v = hist[c * nbins + b];
    hist[c * nbins + b] = run;
    run += v;
  }
  total[b] = run;
}

// Single-block exclusive scan of n ints (n up to a few million, strided passes).
__global__ void k_exscan(const int* __restrict__ in, int n, int* __restrict__ out) {
  __shared__ int part[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    int i = base + threadIdx.x;
    int v = (i < n) ? in[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      int t = (threadIdx.x >= off) ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) out[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void k_scatter(const int* __restrict__ keys, int64_t N, int nbins, int* __restrict__ hist,
                          const int* __restrict__ bin_start, int* __restrict__ perm) {
  // one warp per chunk
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t lo = c * kChunk;
  if (lo >= N) return;
  const int64_t hi = ((N < lo + kChunk) ? N : lo + kChunk);
  int* h = hist + c * (int64_t)nbins;
  for (int64_t g = lo; g < hi; g += 32) {
    const int64_t i = g + lane;
    const bool act = i < hi;
    const unsigned mask = __ballot_sync(0xffffffffu, act);
    if (act) {
      const int key = keys[i];
      const unsigned peers = __match_any_sync(mask, key);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int base = h[key] + bin_start[key];
      perm[base + rank] = (int)i;
      __syncwarp(mask);
      if (rank == 0) h[key] += __popc(peers);
    }
    __syncwarp();
  }
}

void stable_bin_sort(const int* keys, int64_t N, int nbins, int* perm, int* bin_start, int* hist,
                     int* total, cudaStream_t st) {
  const int64_t nchunks = ceil_div(N, kChunk);
  SE1P_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(int) * nchunks * nbins, st));
  k_hist<<<(unsigned)nchunks, 256, 0, st>>>(keys, N, nbins, hist);
  SE1P_LAUNCH_CHECK();
  k_colscan<<<(unsigned)ceil_div(nbins, 256), 256, 0, st>>>(hist, nchunks, nbins, total);
  SE1P_LAUNCH_CHECK();
  k_exscan<<<1, 1024, 0, st>>>(total, nbins, bin_start);
  SE1P_LAUNCH_CHECK();
  k_scatter<<<(unsigned)ceil_div(nchunks, 4), 128, 0, st>>>(keys, N, nbins, hist, bin_start, perm);
  SE1P_LAUNCH_CHECK();
}

int64_t sort_hist_ints(int64_t N, int nbins) { return ceil_div(N, kChunk) * (int64_t)nbins; }

}  // namespace se1p
