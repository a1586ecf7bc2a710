// particles.cu -- binning of the particles for the gridding/gather sweeps (sweep.cu) and the
// particle selection of the distributed path.
//
// Stencil (reading R-3): free axes use the P nodes j = floor(x/h)+1 .. floor(x/h)+P,
// node j at coordinate (j - P/2) h; the periodic axis uses nodes l = floor(z/h - P/2)+1 ..
// +P (unwrapped, distance l h - z, index l mod M).  Window e^{-alpha d^2}, alpha = 2 xi^2/eta.
// Constants ((2xi^2/(pi eta))^{3/2} twice and 4 pi h^3) are folded into the mode multipliers.
#include "kspace.cuh"
#include "sort.cuh"

namespace se1p {

__device__ __forceinline__ int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
__device__ __forceinline__ int imod(int a, int m) { int r = a % m; return r < 0 ? r + m : r; }

// ------------------------------------------------------------------ binning
__global__ void k_keys(KDev dv, const double* __restrict__ x, int64_t N, int* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double px = x[3 * i], py = x[3 * i + 1];
  double pz = x[3 * i + 2];
  pz -= dv.L3 * floor(pz / dv.L3);
  if (pz >= dv.L3) pz -= dv.L3;
  int cx = (int)floor(px * dv.inv_h), cy = (int)floor(py * dv.inv_h);
  cx = min(max(cx, 0), dv.Mfree - 1);
  cy = min(max(cy, 0), dv.Mfree - 1);
  // periodic stencil start a = lz0 mod M (the same arithmetic as k_permute)
  const int lz0 = (int)floor(pz * dv.inv_h - 0.5 * dv.P) + 1;
  int a = lz0 % dv.M;
  if (a < 0) a += dv.M;
  // bins: (x band of kBin cells, stencil start a, y cell), y fastest -- a sweep layer's candidates
  // in one x band are one contiguous run of the sorted order
  keys[i] = ((cx / kBin) * dv.M + a) * dv.Mfree + cy;
}

// Sorted particles: position/charge and stencil starts (reading R-3).
__global__ void k_permute(KDev dv, const double* __restrict__ x, const double* __restrict__ q,
                          const int* __restrict__ perm, int64_t N, double4* __restrict__ out,
                          int4* __restrict__ s4) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= N) return;
  const int64_t i = perm[s];
  double pz = x[3 * i + 2];
  pz -= dv.L3 * floor(pz / dv.L3);
  if (pz >= dv.L3) pz -= dv.L3;
  const double px = x[3 * i], py = x[3 * i + 1];
  out[s] = make_double4(px, py, pz, q[i]);
  int cx = (int)floor(px * dv.inv_h), cy = (int)floor(py * dv.inv_h);
  cx = min(max(cx, 0), dv.Mfree - 1);
  cy = min(max(cy, 0), dv.Mfree - 1);
  const int jx0 = cx + 1, jy0 = cy + 1, lz0 = (int)floor(pz * dv.inv_h - 0.5 * dv.P) + 1;
  int a = lz0 % dv.M;
  if (a < 0) a += dv.M;
  s4[s] = make_int4(jx0, jy0, lz0, a);
}

// Distributed path: the particles whose x stencil rows [jx0, jx0 + P) meet the slab rows
// [row_lo, row_hi) (reading R-3: jx0 = floor(x/h) + 1), compacted in their original order.
__global__ void k_slab_flags(KDev dv, const double* __restrict__ x, int64_t N, int row_lo, int row_hi,
                             int* __restrict__ flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int cx = (int)floor(x[3 * i] * dv.inv_h);
  cx = min(max(cx, 0), dv.Mfree - 1);
  const int j0 = cx + 1;
  flags[i] = (j0 + dv.P > row_lo && j0 < row_hi) ? 1 : 0;
}

__global__ void k_slab_compact(const double* __restrict__ x, const double* __restrict__ q, int64_t N,
                               const int* __restrict__ flags, const int* __restrict__ pos, double* __restrict__ xc,
                               double* __restrict__ qc, int* __restrict__ idmap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N || !flags[i]) return;
  const int p = pos[i];
  xc[3 * (int64_t)p] = x[3 * i];
  xc[3 * (int64_t)p + 1] = x[3 * i + 1];
  xc[3 * (int64_t)p + 2] = x[3 * i + 2];
  qc[p] = q[i];
  idmap[p] = (int)i;
}

__global__ void k_scatter_partial(const double* __restrict__ phic, const int* __restrict__ idmap, int64_t n,
                                  double* __restrict__ phi) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) phi[idmap[p]] = phic[p];
}

void k_slab_select(const KPlan& pl, const double* x, const double* q, int64_t N, int row_lo, int row_hi, int* flags,
                   int* pos, int* scan_scratch, double* xc, double* qc, int* idmap, cudaStream_t st) {
  const unsigned nb = (unsigned)ceil_div(N, 256);
  k_slab_flags<<<nb, 256, 0, st>>>(pl.dv, x, N, row_lo, row_hi, flags);
  SE1P_LAUNCH_CHECK();
  exclusive_scan_ints(flags, N, pos, scan_scratch, st);
  k_slab_compact<<<nb, 256, 0, st>>>(x, q, N, flags, pos, xc, qc, idmap);
  SE1P_LAUNCH_CHECK();
}

void k_scatter_partial_stage(const double* phic, const int* idmap, int64_t n, double* phi, cudaStream_t st) {
  if (n <= 0) return;
  k_scatter_partial<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(phic, idmap, n, phi);
  SE1P_LAUNCH_CHECK();
}

void k_bin_particles(const KPlan& pl, KWork& w, const double* x, const double* q, int64_t N, cudaStream_t st) {
  const KDev& dv = pl.dv;
  const int nbins = dv.nbx * dv.M * dv.Mfree;
  const unsigned nb = (unsigned)ceil_div(N, 256);
  k_keys<<<nb, 256, 0, st>>>(dv, x, N, w.keys);
  SE1P_LAUNCH_CHECK();
  stable_bin_sort(w.keys, N, nbins, w.perm, w.bin_start, w.scratch, st);
  k_permute<<<nb, 256, 0, st>>>(dv, x, q, w.perm, N, (double4*)w.xs, (int4*)w.s4);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
