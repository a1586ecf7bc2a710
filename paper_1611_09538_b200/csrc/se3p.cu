// se3p.cu -- the SE3P baseline: the triply periodic k-space sum through the
// same gridding/gather tiles as SE1P.  The 1P tile plan grids onto the extended free axes
// (M~ = M_free + P rows, node j at (j - P/2) h, reading R-3); with every axis periodic the node
// j is the periodic node (j - P/2) mod M_free (P even), so folding the overhanging rows onto the
// periodic grid gives the SE3P gridding, and unfolding H~ gives the grid the gather reads.
#include "kspace.cuh"

namespace se1p {

// per[i][j][k] = sum of ext[x][y][k] over x = i + P/2 + a Mf, y = j + P/2 + b Mf inside [0, Mt)
__global__ void k_fold(int Mt, int Mf, int M, int off, const double* __restrict__ ext, double* __restrict__ per) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)Mf * Mf * M) return;
  const int k = (int)(id % M);
  const int64_t ij = id / M;
  const int j = (int)(ij % Mf), i = (int)(ij / Mf);
  // the smallest x >= 0 congruent to i + off (mod Mf)
  const int x0 = (i + off) % Mf, y0 = (j + off) % Mf;
  double s = 0.0;
  for (int x = x0; x < Mt; x += Mf)
    for (int y = y0; y < Mt; y += Mf) s += ext[((int64_t)x * Mt + y) * M + k];
  per[id] = s;
}

__global__ void k_unfold(int Mt, int Mf, int M, int off, const double* __restrict__ per, double* __restrict__ ext) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)Mt * Mt * M) return;
  const int k = (int)(id % M);
  const int64_t xy = id / M;
  const int y = (int)(xy % Mt), x = (int)(xy / Mt);
  const int i = ((x - off) % Mf + Mf) % Mf, j = ((y - off) % Mf + Mf) % Mf;
  ext[id] = per[((int64_t)i * Mf + j) * M + k];
}

void k_fold_3p(const KPlan& e, const double* grid_ext, double* grid_per, cudaStream_t st) {
  const KDev& d = e.dv;
  const int64_t n = (int64_t)d.Mfree * d.Mfree * d.M;
  k_fold<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d.Mt, d.Mfree, d.M, d.P / 2, grid_ext, grid_per);
  SE1P_LAUNCH_CHECK();
}

void k_unfold_3p(const KPlan& e, const double* grid_per, double* grid_ext, cudaStream_t st) {
  const KDev& d = e.dv;
  const int64_t n = (int64_t)d.Mt * d.Mt * d.M;
  k_unfold<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d.Mt, d.Mfree, d.M, d.P / 2, grid_per, grid_ext);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
