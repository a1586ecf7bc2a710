// real.cu -- real-space sum phi^R (Eq. (3)) truncated at rc with linked cells
// and the self term (Eq. (6)).
//
// Cells: nc_d = max(1, floor(D L_d/rc)) per axis, so a cell is at least rc/D wide; free axes
// scan the cells within K_d = ceil(rc/cell_d) (no images), the periodic axis scans the unwrapped
// cells cz-K .. cz+K, K = ceil(rc/cell_z), each unwrapped cell u standing for cell (u mod nc_z)
// shifted by floor(u/nc_z) L3; a cell whose box lies farther than rc from the target is skipped.
// Every image within rc is visited exactly once, for any rc.
#include <vector>

#include "kspace.cuh"
#include "real.cuh"
#include "sort.cuh"

#ifndef SE1P_REAL_TABLE
#define SE1P_REAL_TABLE 1
#endif
// 1: warp per cell with hit masks (k_real_cells); 0: thread per target (k_real_sum).  Measured at
// C4/C5: 34.8/29.9 ms against 27.1/26.3 ms -- the box-to-box culling of a cell's neighbours scans
// ~1.5x the candidates of per-target culling and the warp issues more instructions per pair
// (7.1 against 5.5 per pair within rc; ncu: shared-load latency on the broadcast candidates and
// the lane-divergent table rows).  Estrin's scheme for the polynomial: +-2 %, not kept.
#ifndef SE1P_REAL_CELLS
#define SE1P_REAL_CELLS 0
#endif

// Cell width rc/D, D in 1..4 chosen for ~32 particles per cell (measured at C3/C4/C5: D = 3/4/2
// best, -45% / -57% / -33% against D = 1)
#ifndef SE1P_REAL_CELL_OCC
#define SE1P_REAL_CELL_OCC 32.0
#endif

namespace se1p {

__device__ __forceinline__ int rfloordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

__global__ void k_real_keys(RDev d, const double* __restrict__ x, int64_t N, int* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double pz = x[3 * i + 2];
  pz -= d.L[2] * floor(pz / d.L[2]);
  if (pz >= d.L[2]) pz -= d.L[2];
  int cx = min(max((int)floor(x[3 * i] / d.cs[0]), 0), d.nc[0] - 1);
  int cy = min(max((int)floor(x[3 * i + 1] / d.cs[1]), 0), d.nc[1] - 1);
  int cz = min(max((int)floor(pz / d.cs[2]), 0), d.nc[2] - 1);
  keys[i] = (cx * d.nc[1] + cy) * d.nc[2] + cz;
}

__global__ void k_real_permute(RDev d, const double* __restrict__ x, const double* __restrict__ q,
                               const int* __restrict__ perm, int64_t N, double4* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= N) return;
  const int64_t i = perm[s];
  double pz = x[3 * i + 2];
  pz -= d.L[2] * floor(pz / d.L[2]);
  if (pz >= d.L[2]) pz -= d.L[2];
  out[s] = make_double4(x[3 * i], x[3 * i + 1], pz, q[i]);
}

// One thread per target (sorted order, so neighbouring threads share cells).
// FIELD: also E^R = -grad_m phi^R = sum_n q_n (erfc(xi r)/r + 2 xi/sqrt(pi) e^{-xi^2 r^2}) r_vec/r^2,
// r_vec = x_m - x_n - alpha L3 e3 (Eq. (3) differentiated; the self term has no gradient).
template <bool FIELD>
__global__ void __launch_bounds__(128) k_real_sum(RDev d, const double4* __restrict__ P4, const int* __restrict__ perm,
                                                  const int* __restrict__ cell_start, int64_t N,
                                                  double* __restrict__ phi_out, double* __restrict__ field_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  const double4 pt = P4[t];
  const int cx = min(max((int)floor(pt.x / d.cs[0]), 0), d.nc[0] - 1);
  const int cy = min(max((int)floor(pt.y / d.cs[1]), 0), d.nc[1] - 1);
  const int cz = min(max((int)floor(pt.z / d.cs[2]), 0), d.nc[2] - 1);
  const double rc2 = d.rc * d.rc;
  double acc = 0.0, ex = 0.0, ey = 0.0, ez = 0.0;
  for (int ax = max(0, cx - d.Kx); ax <= min(d.nc[0] - 1, cx + d.Kx); ++ax) {
    // distance from the target to the cell's slab along x (0 inside)
    const double gx = fmax(fmax(ax * d.cs[0] - pt.x, pt.x - (ax + 1) * d.cs[0]), 0.0);
    for (int ay = max(0, cy - d.Ky); ay <= min(d.nc[1] - 1, cy + d.Ky); ++ay) {
      const double gy = fmax(fmax(ay * d.cs[1] - pt.y, pt.y - (ay + 1) * d.cs[1]), 0.0);
      if (gx * gx + gy * gy > rc2) continue;
      for (int u = cz - d.K; u <= cz + d.K; ++u) {
        const double gz = fmax(fmax(u * d.cs[2] - pt.z, pt.z - (u + 1) * d.cs[2]), 0.0);
        if (gx * gx + gy * gy + gz * gz > rc2) continue;   // no point of the cell within rc
        const int w = rfloordiv(u, d.nc[2]);
        const int az = u - w * d.nc[2];
        const double shift = w * d.L[2];
        const int c = (ax * d.nc[1] + ay) * d.nc[2] + az;
        const int s = cell_start[c], e = cell_start[c + 1];
        // candidates two at a time: both positions are loaded before either is used
        for (int j = s; j < e; j += 2) {
          const bool two = j + 1 < e;
          const double4 pa = P4[j];
          const double4 pb = two ? P4[j + 1] : pa;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            if (h2 == 1 && !two) break;
            const int jj = j + h2;
            const double4 ps = h2 ? pb : pa;
            if (w == 0 && jj == t) continue;   // the prime in Eq. (3): n = m only at p = 0
            const double dx = pt.x - ps.x, dy = pt.y - ps.y, dz = pt.z - (ps.z + shift);
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 <= rc2) {
#if SE1P_REAL_TABLE
              // erfc(xi r) from the local polynomial of r's interval (no erfc, exp or division)
              const double rinv = rsqrt(r2), r = r2 * rinv;
              const int it = min((int)(r * d.inv_dr), d.ntab - 1);
              const double u = r - ((double)it + 0.5) * d.dr;
              const double2* cf = reinterpret_cast<const double2*>(d.tab + it * (kTabDeg + 1));
              const double2 c67 = __ldg(cf + 3), c45 = __ldg(cf + 2), c23 = __ldg(cf + 1), c01 = __ldg(cf);
              double pv = fma(c67.y, u, c67.x);
              pv = fma(pv, u, c45.y);
              pv = fma(pv, u, c45.x);
              pv = fma(pv, u, c23.y);
              pv = fma(pv, u, c23.x);
              pv = fma(pv, u, c01.y);
              const double ec = fma(pv, u, c01.x) * rinv;
              acc = fma(ps.w, ec, acc);
              if (FIELD) {   // dv = d/dr erfc(xi r) = -(2 xi/sqrt(pi)) e^{-xi^2 r^2}
                double dv = 7.0 * c67.y;
                dv = fma(dv, u, 6.0 * c67.x);
                dv = fma(dv, u, 5.0 * c45.y);
                dv = fma(dv, u, 4.0 * c45.x);
                dv = fma(dv, u, 3.0 * c23.y);
                dv = fma(dv, u, 2.0 * c23.x);
                dv = fma(dv, u, c01.y);
                const double g = ps.w * (ec - dv) * (rinv * rinv);
                ex = fma(g, dx, ex);
                ey = fma(g, dy, ey);
                ez = fma(g, dz, ez);
              }
#else
              const double r = sqrt(r2);
              const double ec = erfc(d.xi * r) / r;
              acc = fma(ps.w, ec, acc);
              if (FIELD) {
                const double g = ps.w * (ec + 1.128379167095512573896158903121545172 * d.xi *   // 2/sqrt(pi)
                                                  exp(-d.xi * d.xi * r2)) / r2;
                ex = fma(g, dx, ex);
                ey = fma(g, dy, ey);
                ez = fma(g, dz, ez);
              }
#endif
            }
          }
        }
      }
    }
  }
  const int64_t u = perm[t];
  if (phi_out) phi_out[u] = acc - 2.0 * d.xi * pt.w * 0.564189583547756286948079451560772586;  // 1/sqrt(pi)
  if (FIELD) {
    field_out[3 * u] = ex;
    field_out[3 * u + 1] = ey;
    field_out[3 * u + 2] = ez;
  }
}

// Warp per target cell (up to 32 of its targets per pass, one per lane).  The warp walks the
// neighbour cells' particles in chunks of 32 staged in shared memory (coalesced loads, broadcast
// reads); each lane first tests the chunk's 32 candidates against its target with the cheap
// distance test alone (a uniform loop, a 32-bit hit mask), then evaluates erfc only over its own
// hits -- so the polynomial runs at the lanes' hit counts (~70 % of the warp busy) instead of
// under a branch taken by ~30 % of the lanes.  Cells are culled box to box: for a neighbour column
// (ax, ay) the z reach kz follows from the remaining distance; runs of z cells with one periodic
// image are contiguous in the sorted order and are walked as one range.  The erfc table sits in
// shared memory when it fits (STAB).
constexpr int kRealWarps = 8;
template <bool FIELD, bool STAB>
__global__ void __launch_bounds__(kRealWarps * 32) k_real_cells(RDev d, const double4* __restrict__ P4,
                                                                const int* __restrict__ perm,
                                                                const int* __restrict__ cell_start, int ncell,
                                                                double* __restrict__ phi_out,
                                                                double* __restrict__ field_out) {
  extern __shared__ double4 rsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double4* cand = rsm + warp * 32;
  const double2* tab;
  if (STAB) {
    double2* ts = reinterpret_cast<double2*>(rsm + kRealWarps * 32);
    const double2* tg = reinterpret_cast<const double2*>(d.tab);
    for (int k = threadIdx.x; k < d.ntab * (kTabDeg + 1) / 2; k += blockDim.x) ts[k] = __ldg(tg + k);
    __syncthreads();
    tab = ts;
  } else {
    tab = reinterpret_cast<const double2*>(d.tab);
  }
  const int c = blockIdx.x * kRealWarps + warp;
  if (c >= ncell) return;
  const int nc1 = d.nc[1], nc2 = d.nc[2];
  const int cz = c % nc2, cy = (c / nc2) % nc1, cx = c / (nc2 * nc1);
  const int ts0 = cell_start[c], te = cell_start[c + 1];
  const double rc2 = d.rc * d.rc;
  for (int t0 = ts0; t0 < te; t0 += 32) {
    const int t = t0 + lane;
    const bool active = t < te;
    const double4 pt = P4[active ? t : t0];
    double acc = 0.0, ex = 0.0, ey = 0.0, ez = 0.0;
    for (int ax = max(0, cx - d.Kx); ax <= min(d.nc[0] - 1, cx + d.Kx); ++ax) {
      const double gx = max(abs(ax - cx) - 1, 0) * d.cs[0];
      for (int ay = max(0, cy - d.Ky); ay <= min(nc1 - 1, cy + d.Ky); ++ay) {
        const double gy = max(abs(ay - cy) - 1, 0) * d.cs[1];
        const double rem = rc2 - gx * gx - gy * gy;
        if (rem < 0.0) continue;
        const int kz = min(d.K, 1 + (int)floor(sqrt(rem) / d.cs[2]));
        const int base = (ax * nc1 + ay) * nc2;
        for (int u = cz - kz; u <= cz + kz;) {
          const int wrap = rfloordiv(u, nc2);
          const int uend = min(cz + kz, (wrap + 1) * nc2 - 1);   // same image through uend
          const int s = cell_start[base + u - wrap * nc2], e = cell_start[base + uend - wrap * nc2 + 1];
          const double shift = wrap * d.L[2];
          for (int j0 = s; j0 < e; j0 += 32) {
            __syncwarp();
            if (j0 + lane < e) cand[lane] = P4[j0 + lane];
            __syncwarp();
            const int n = min(32, e - j0);
            unsigned mask = 0;
#pragma unroll 4
            for (int k = 0; k < n; ++k) {
              const double4 pc = cand[k];
              const double dx = pt.x - pc.x, dy = pt.y - pc.y, dz = pt.z - (pc.z + shift);
              const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
              if (r2 <= rc2) mask |= 1u << k;
            }
            if (wrap == 0 && t >= j0 && t < j0 + n) mask &= ~(1u << (t - j0));   // the prime: n = m at p = 0
            if (!active) mask = 0;
            // hits two at a time (independent chains); erfc by Estrin's scheme (depth 4, not 7)
            while (mask) {
              const int k1 = __ffs(mask) - 1;
              mask &= mask - 1;
              const int k2 = mask ? __ffs(mask) - 1 : -1;
              if (k2 >= 0) mask &= mask - 1;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int k = h ? k2 : k1;
                if (k < 0) break;
                const double4 pc = cand[k];
                const double dx = pt.x - pc.x, dy = pt.y - pc.y, dz = pt.z - (pc.z + shift);
                const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
                const double rinv = rsqrt(r2), r = r2 * rinv;
                const int it = min((int)(r * d.inv_dr), d.ntab - 1);
                const double uu = r - ((double)it + 0.5) * d.dr;
                const double2* cf = tab + it * ((kTabDeg + 1) / 2);
                const double2 c67 = cf[3], c45 = cf[2], c23 = cf[1], c01 = cf[0];
                const double u2 = uu * uu, u4 = u2 * u2;
                const double p01 = fma(c01.y, uu, c01.x), p23 = fma(c23.y, uu, c23.x);
                const double p45 = fma(c45.y, uu, c45.x), p67 = fma(c67.y, uu, c67.x);
                const double ec = fma(u4, fma(u2, p67, p45), fma(u2, p23, p01)) * rinv;
                acc = fma(pc.w, ec, acc);
                if (FIELD) {   // d/dr erfc(xi r) from the same polynomial
                  const double q12 = fma(2.0 * c23.x, uu, c01.y), q34 = fma(4.0 * c45.x, uu, 3.0 * c23.y);
                  const double q56 = fma(6.0 * c67.x, uu, 5.0 * c45.y);
                  const double dv = fma(u4, fma(u2, 7.0 * c67.y, q56), fma(u2, q34, q12));
                  const double g = pc.w * (ec - dv) * (rinv * rinv);
                  ex = fma(g, dx, ex);
                  ey = fma(g, dy, ey);
                  ez = fma(g, dz, ez);
                }
              }
            }
          }
          u = uend + 1;
        }
      }
    }
    if (active) {
      const int64_t uo = perm[t];
      if (phi_out) phi_out[uo] = acc - 2.0 * d.xi * pt.w * 0.564189583547756286948079451560772586;  // 1/sqrt(pi)
      if (FIELD) {
        field_out[3 * uo] = ex;
        field_out[3 * uo + 1] = ey;
        field_out[3 * uo + 2] = ez;
      }
    }
  }
}

template <bool FIELD>
static void launch_real_cells(const RDev& d, const double4* P4, const int* perm, const int* cell_start, int ncell,
                              double* phi_out, double* field_out, cudaStream_t st) {
  const size_t tab_bytes = (size_t)d.ntab * (kTabDeg + 1) * sizeof(double);
  const bool stab = tab_bytes <= 48 * 1024;
  const size_t smem = kRealWarps * 32 * sizeof(double4) + (stab ? tab_bytes : 0);
  const unsigned nb = (unsigned)ceil_div(ncell, kRealWarps);
  if (stab) {
    SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_real_cells<FIELD, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_real_cells<FIELD, true><<<nb, kRealWarps * 32, smem, st>>>(d, P4, perm, cell_start, ncell, phi_out, field_out);
  } else {
    k_real_cells<FIELD, false><<<nb, kRealWarps * 32, smem, st>>>(d, P4, perm, cell_start, ncell, phi_out, field_out);
  }
  SE1P_LAUNCH_CHECK();
}

RDev real_geometry(const double L[3], double xi, double rc, int64_t N) {
  RDev d;
  const double rho = (double)std::max<int64_t>(N, 1) / (L[0] * L[1] * L[2]);
  const double D = std::min(4.0, std::max(1.0, std::round(rc / std::cbrt(SE1P_REAL_CELL_OCC / rho))));
  for (int a = 0; a < 3; ++a) {
    d.L[a] = L[a];
    d.nc[a] = std::max(1, (int)std::floor(D * L[a] / rc));
    d.nc[a] = std::min(d.nc[a], 256);
    d.cs[a] = L[a] / d.nc[a];
  }
  d.K = (int)std::ceil(rc / d.cs[2]);
  d.Kx = (int)std::ceil(rc / d.cs[0]);
  d.Ky = (int)std::ceil(rc / d.cs[1]);
  d.xi = xi;
  d.rc = rc;
  return d;
}

// Taylor coefficients of erfc(xi r) about the interval midpoints r_i = (i + 1/2) dr:
// d^n/dx^n erfc(x) = (-1)^n (2/sqrt(pi)) H_{n-1}(x) e^{-x^2} (physicists' Hermite polynomials),
// evaluated in long double; term n carries xi^n/n!.  The interval count (real.cuh) keeps the
// degree-7 remainder below 1e-16 relative to erfc itself.
static std::vector<double> erfc_table(double xi, double rc, int ntab) {
  std::vector<double> t((size_t)ntab * (kTabDeg + 1));
  const long double dr = (long double)rc / ntab, two_over_sqrtpi = 1.128379167095512573896158903121545172L;
  for (int i = 0; i < ntab; ++i) {
    const long double x0 = (long double)xi * ((long double)i + 0.5L) * dr;
    const long double g = two_over_sqrtpi * expl(-x0 * x0);
    long double hm1 = 0.0L, h = 1.0L;   // H_{-1} (unused), H_0
    t[(size_t)i * (kTabDeg + 1)] = (double)erfcl(x0);
    long double xin = 1.0L, fact = 1.0L;
    for (int n = 1; n <= kTabDeg; ++n) {
      xin *= (long double)xi;
      fact *= (long double)n;
      // coefficient of u^n: (-1)^n (2/sqrt(pi)) H_{n-1}(x0) e^{-x0^2} xi^n / n!
      const long double c = ((n & 1) ? -1.0L : 1.0L) * g * h * xin / fact;
      t[(size_t)i * (kTabDeg + 1) + n] = (double)c;
      const long double hn = 2.0L * x0 * h - 2.0L * (long double)(n - 1) * hm1;   // H_n
      hm1 = h;
      h = hn;
    }
  }
  return t;
}

struct TabCache {
  double xi = 0, rc = 0;
  double* dev = nullptr;
  int64_t cap = 0;
};
static TabCache g_tab[64];

void real_release_tables(int dev) {
  TabCache& tc = g_tab[dev & 63];
  if (tc.dev) dev_free(tc.dev);
  tc = TabCache{};
}

void real_space(const RDev& d0, KWork& w, const double* x, const double* q, int64_t N, double* phi_out,
                cudaStream_t st, double* field_out) {
  RDev d = d0;
#if SE1P_REAL_TABLE
  {
    int dev = 0;
    SE1P_CUDA_TRY(cudaGetDevice(&dev));
    TabCache& tc = g_tab[dev & 63];
    const int ntab = real_table_intervals(d.xi, d.rc);
    if (!tc.dev || tc.xi != d.xi || tc.rc != d.rc) {
      const std::vector<double> t = erfc_table(d.xi, d.rc, ntab);
      if (tc.dev && tc.cap < (int64_t)t.size()) {
        dev_free(tc.dev);
        tc.dev = nullptr;
      }
      if (!tc.dev) {
        dev_alloc(tc.dev, t.size());
        tc.cap = (int64_t)t.size();
      }
      SE1P_CUDA_TRY(cudaMemcpyAsync(tc.dev, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice, st));
      SE1P_CUDA_TRY(cudaStreamSynchronize(st));
      tc.xi = d.xi;
      tc.rc = d.rc;
    }
    d.tab = tc.dev;
    d.ntab = ntab;
    d.dr = d.rc / ntab;
    d.inv_dr = ntab / d.rc;
  }
#endif
  const int ncell = d.nc[0] * d.nc[1] * d.nc[2];
  const unsigned nb = (unsigned)ceil_div(N, 256);
  k_real_keys<<<nb, 256, 0, st>>>(d, x, N, w.keys);
  SE1P_LAUNCH_CHECK();
  stable_bin_sort(w.keys, N, ncell, w.perm, w.bin_start, w.scratch, st);
  k_real_permute<<<nb, 256, 0, st>>>(d, x, q, w.perm, N, (double4*)w.xs);
  SE1P_LAUNCH_CHECK();
#if SE1P_REAL_CELLS && SE1P_REAL_TABLE
  if (field_out)
    launch_real_cells<true>(d, (const double4*)w.xs, w.perm, w.bin_start, ncell, phi_out, field_out, st);
  else
    launch_real_cells<false>(d, (const double4*)w.xs, w.perm, w.bin_start, ncell, phi_out, nullptr, st);
  return;
#endif
  const unsigned nt = (unsigned)ceil_div(N, 128);
  if (field_out)
    k_real_sum<true><<<nt, 128, 0, st>>>(d, (const double4*)w.xs, w.perm, w.bin_start, N, phi_out, field_out);
  else
    k_real_sum<false><<<nt, 128, 0, st>>>(d, (const double4*)w.xs, w.perm, w.bin_start, N, phi_out, nullptr);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
