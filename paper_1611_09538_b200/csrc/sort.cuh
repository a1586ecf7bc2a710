// sort.cuh -- deterministic stable bin sort (see sort.cu).
#pragma once
#include "common.cuh"

namespace se1p {

// keys[i] in [0, nbins).  perm[pos] = original index of the particle at sorted position pos;
// bin_start[b] .. bin_start[b+1] is bin b (bin_start has nbins+1 entries).
// scratch: sort_scratch_ints(N, nbins) ints.
void stable_bin_sort(const int* keys, int64_t N, int nbins, int* perm, int* bin_start, int* scratch,
                     cudaStream_t st);
int64_t sort_scratch_ints(int64_t N, int nbins);
// out[0..n]: exclusive prefix sums of in[0..n) and the total at out[n]; scratch: scan_scratch_ints(n)
void exclusive_scan_ints(const int* in, int64_t n, int* out, int* scratch, cudaStream_t st);
int64_t scan_scratch_ints(int64_t n);

}  // namespace se1p
