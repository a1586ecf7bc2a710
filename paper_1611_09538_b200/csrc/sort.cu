// sort.cu -- deterministic stable counting sort of particles into bins (cells / tiles).
//
// The gridding and gather kernels visit particles bin by bin; a stable order (by original
// index inside a bin) makes every floating-point reduction order fixed, so results are
// bitwise reproducible without atomics on floating point data.
//
//   1. per-chunk histograms  hist[c][b]   (chunk = consecutive input particles; the chunk
//      length adapts so that the histogram matrix stays below kHistBudget ints)
//   2. column scan over chunks -> per-(chunk,bin) running offsets, bin totals
//   3. exclusive scan of totals -> bin_start[b]
//   4. scatter: one warp per chunk walks its particles in order, 32 at a time; equal keys
//      inside a group are ranked with __match_any_sync, so positions follow input order.
#include "sort.cuh"

namespace se1p {

constexpr int64_t kHistBudget = 1 << 23;

int64_t sort_chunk(int64_t N, int nbins) {
  int64_t chunk = kChunk;
  while (ceil_div(N, chunk) * (int64_t)nbins > kHistBudget && chunk < N) chunk *= 2;
  return chunk;
}

__global__ void k_hist(const int* __restrict__ keys, int64_t N, int64_t chunk, int nbins, int* __restrict__ hist) {
  const int64_t c = blockIdx.x;
  const int64_t lo = c * chunk, hi = ((N < lo + chunk) ? N : lo + chunk);
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

// Exclusive scan of n ints in one block: each thread scans a contiguous span, the 1024 span
// totals are scanned in shared memory, then each span is rewritten with its offset.
__global__ void k_exscan(const int* __restrict__ in, int n, int* __restrict__ out) {
  __shared__ int part[1024];
  const int span = (n + 1023) / 1024;
  const int lo = min(n, (int)threadIdx.x * span), hi = min(n, lo + span);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += in[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    int t = (threadIdx.x >= off) ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  int run = part[threadIdx.x] - s;
  for (int i = lo; i < hi; ++i) {
    const int v = in[i];
    out[i] = run;
    run += v;
  }
  if (threadIdx.x == 1023) out[n] = part[1023];
}

__global__ void k_scatter(const int* __restrict__ keys, int64_t N, int64_t chunk, int nbins, int* __restrict__ hist,
                          const int* __restrict__ bin_start, int* __restrict__ perm) {
  // one warp per chunk
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t lo = c * chunk;
  if (lo >= N) return;
  const int64_t hi = ((N < lo + chunk) ? N : lo + chunk);
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
  const int64_t chunk = sort_chunk(N, nbins);
  const int64_t nchunks = ceil_div(N, chunk);
  SE1P_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(int) * nchunks * nbins, st));
  k_hist<<<(unsigned)nchunks, 256, 0, st>>>(keys, N, chunk, nbins, hist);
  SE1P_LAUNCH_CHECK();
  k_colscan<<<(unsigned)ceil_div(nbins, 256), 256, 0, st>>>(hist, nchunks, nbins, total);
  SE1P_LAUNCH_CHECK();
  k_exscan<<<1, 1024, 0, st>>>(total, nbins, bin_start);
  SE1P_LAUNCH_CHECK();
  k_scatter<<<(unsigned)ceil_div(nchunks, 4), 128, 0, st>>>(keys, N, chunk, nbins, hist, bin_start, perm);
  SE1P_LAUNCH_CHECK();
}

int64_t sort_hist_ints(int64_t N, int nbins) { return ceil_div(N, sort_chunk(N, nbins)) * (int64_t)nbins; }

}  // namespace se1p
