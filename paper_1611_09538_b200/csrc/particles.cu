// particles.cu -- binning, gridding (Alg. 1 step 2, Eq. (spread_1p)) and gather
// (Alg. 1 step 6, Eq. (se1p_complete_discretized)) on the extended grid.
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
  int cx = (int)floor(px * dv.inv_h), cy = (int)floor(py * dv.inv_h), cz = (int)floor(pz * dv.inv_h);
  cx = min(max(cx, 0), dv.Mfree - 1);
  cy = min(max(cy, 0), dv.Mfree - 1);
  cz = min(max(cz, 0), dv.M - 1);
  // bins: (x band of kBin cells, z cell, y cell), y fastest -- a tile's candidates in one x band
  // and z cell are one contiguous run of the sorted order
  keys[i] = ((cx / kBin) * dv.M + cz) * dv.Mfree + cy;
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

// ------------------------------------------------------------------ stencil helpers
struct Stencil {
  int jx0, jy0, lz0;   // first node (free axes: grid index; z: unwrapped node)
};

__device__ __forceinline__ Stencil stencil_of(const KDev& dv, double px, double py, double pz) {
  Stencil s;
  int cx = (int)floor(px * dv.inv_h), cy = (int)floor(py * dv.inv_h);
  cx = min(max(cx, 0), dv.Mfree - 1);
  cy = min(max(cy, 0), dv.Mfree - 1);
  s.jx0 = cx + 1;
  s.jy0 = cy + 1;
  s.lz0 = (int)floor(pz * dv.inv_h - 0.5 * dv.P) + 1;
  return s;
}

// free-axis weight of node g (grid index) for a particle at coordinate p with stencil start j0
__device__ __forceinline__ double wfree(const KDev& dv, int g, int j0, double p) {
  if (g < j0 || g >= j0 + dv.P) return 0.0;
  const double d = ((double)g - 0.5 * dv.P) * dv.h - p;
  return exp(-dv.alpha * d * d);
}

// periodic-axis weight of grid node g in [0, M) for a particle at z with unwrapped start l0
__device__ __forceinline__ double wper(const KDev& dv, int g, int l0, double pz) {
  const int t = imod(g - l0, dv.M);
  if (t >= dv.P) return 0.0;
  const double d = (double)(l0 + t) * dv.h - pz;
  return exp(-dv.alpha * d * d);
}

// ------------------------------------------------------------------ gridding v1
// One CTA per kTX x kTY x kTZ tile of the extended grid (output-stationary, no atomics).
// Thread: one (x,y) column of the tile and 8 z points.  Particles of every bin whose
// stencils can reach the tile are staged in shared memory as tile-restricted weights.
constexpr int kBatch = 64;

__global__ void __launch_bounds__(128) k_spread_v1(KDev dv, const double4* __restrict__ P4,
                                                   const int* __restrict__ bin_start, double* __restrict__ grid) {
  __shared__ double swx[kBatch][kTX], swy[kBatch][kTY], swz[kBatch][kTZ];
  const int tz = blockIdx.x % dv.ntz, t2 = blockIdx.x / dv.ntz;
  const int ty = t2 % dv.nty, tx = t2 / dv.nty;
  const int X0 = tx * kTX, Y0 = ty * kTY, Z0 = tz * kTZ;
  const int tid = threadIdx.x;
  const int ix = tid & 7, iy = (tid >> 3) & 7, zh = tid >> 6;
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;

  // cells whose particles can touch the tile: cx in [X0-P, X0+kTX-2] etc. (stencil j0 = cx+1)
  const int bx0 = max(0, floordiv(X0 - dv.P, kBin)), bx1 = min(dv.nbx - 1, floordiv(X0 + kTX - 2, kBin));
  const int cy0 = max(0, Y0 - dv.P), cy1 = min(dv.Mfree - 1, Y0 + kTY - 2);
  int cz0 = Z0 - dv.P - 1, nz = kTZ + 2 * dv.P + 3;
  if (nz >= dv.M) { cz0 = 0; nz = dv.M; }

  for (int bx = bx0; bx <= bx1; ++bx)
    for (int zz = 0; zz < nz; ++zz) {
      if (cy1 < cy0) break;
      {
        const int row = (bx * dv.M + imod(cz0 + zz, dv.M)) * dv.Mfree;
        const int s = bin_start[row + cy0], e = bin_start[row + cy1 + 1];
        for (int base = s; base < e; base += kBatch) {
          const int cnt = min(kBatch, e - base);
          for (int task = tid; task < cnt * 4; task += blockDim.x) {
            const int p = task >> 2, d = task & 3;
            const double4 pp = P4[base + p];
            const Stencil st = stencil_of(dv, pp.x, pp.y, pp.z);
            if (d == 0) {
#pragma unroll
              for (int i = 0; i < kTX; ++i) swx[p][i] = wfree(dv, X0 + i, st.jx0, pp.x);
            } else if (d == 1) {
#pragma unroll
              for (int i = 0; i < kTY; ++i) swy[p][i] = wfree(dv, Y0 + i, st.jy0, pp.y);
            } else {
              const int k0 = (d - 2) * 8;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int g = Z0 + k0 + k;
                swz[p][k0 + k] = (g < dv.M) ? pp.w * wper(dv, g, st.lz0, pp.z) : 0.0;
              }
            }
          }
          __syncthreads();
          for (int p = 0; p < cnt; ++p) {
            const double c = swx[p][ix] * swy[p][iy];
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = fma(c, swz[p][zh * 8 + k], acc[k]);
          }
          __syncthreads();
        }
      }
    }
  const int gx = X0 + ix, gy = Y0 + iy;
  if (gx < dv.Mt && gy < dv.Mt) {
    double* col = grid + ((int64_t)gx * dv.Mt + gy) * dv.M;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int gz = Z0 + zh * 8 + k;
      if (gz < dv.M) col[gz] = acc[k];
    }
  }
}

void k_spread(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st) {
  (void)N;
  const KDev& dv = pl.dv;
  const unsigned nblk = (unsigned)(dv.ntx * dv.nty * dv.ntz);
  k_spread_v1<<<nblk, 128, 0, st>>>(dv, (const double4*)w.xs, w.bin_start, w.grid);
  SE1P_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ gather v1
// One warp per particle (sorted order): lanes split the P x P columns of the stencil and each
// dots a z-column with the periodic weights; fixed-order warp reduction.
__global__ void __launch_bounds__(256) k_gather_v1(KDev dv, const double4* __restrict__ P4, const int* __restrict__ perm,
                                                   const double* __restrict__ grid, int64_t N,
                                                   double* __restrict__ phi_out) {
  __shared__ double sw[8][3][64];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * 8 + wid;
  if (p >= N) return;
  const double4 pp = P4[p];
  const Stencil st = stencil_of(dv, pp.x, pp.y, pp.z);
  const int P = dv.P, M = dv.M, Mt = dv.Mt;
  for (int t = lane; t < P; t += 32) {
    const double dx = ((double)(st.jx0 + t) - 0.5 * P) * dv.h - pp.x;
    const double dy = ((double)(st.jy0 + t) - 0.5 * P) * dv.h - pp.y;
    const double dz = (double)(st.lz0 + t) * dv.h - pp.z;
    sw[wid][0][t] = exp(-dv.alpha * dx * dx);
    sw[wid][1][t] = exp(-dv.alpha * dy * dy);
    sw[wid][2][t] = exp(-dv.alpha * dz * dz);
  }
  __syncwarp();
  const int z0 = imod(st.lz0, M);
  double acc = 0.0;
  for (int ij = lane; ij < P * P; ij += 32) {
    const int i = ij / P, j = ij - i * P;
    const double* col = grid + ((int64_t)(st.jx0 + i) * Mt + (st.jy0 + j)) * M;
    double s = 0.0;
    int zi = z0;
    for (int k = 0; k < P; ++k) {
      s = fma(col[zi], sw[wid][2][k], s);
      if (++zi == M) zi = 0;
    }
    acc = fma(sw[wid][0][i] * sw[wid][1][j], s, acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) phi_out[perm[p]] = acc;
}

void k_gather(const KPlan& pl, KWork& w, int64_t N, double* phi_out, cudaStream_t st) {
  k_gather_v1<<<(unsigned)ceil_div(N, 8), 256, 0, st>>>(pl.dv, (const double4*)w.xs, w.perm, w.grid, N, phi_out);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
