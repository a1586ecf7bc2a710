// real.cu -- real-space sum phi^R (Eq. (3)) truncated at rc with cell lists
// and the self term (Eq. (6)).
//
// Product kernel: k_real_warp (warp per group of <= 32 targets of one (x, y) column, candidates
// from the columns within rc of the group's box, erfc from a 32-interval table in shared memory;
// see its header below and DESIGN.md section 4).  Kept as build options / fallback: k_real_sum
// (thread per target; also used when xi rc is beyond the shared table) and k_real_cells (warp per
// cell).  Their cells: nc_d = max(1, floor(D L_d/rc)) per axis, so a cell is at least rc/D wide;
// free axes scan the cells within K_d = ceil(rc/cell_d) (no images), the periodic axis scans the
// unwrapped cells cz-K .. cz+K, K = ceil(rc/cell_z), each unwrapped cell u standing for cell
// (u mod nc_z) shifted by floor(u/nc_z) L3; a cell whose box lies farther than rc from the target
// is skipped.  Every image within rc is visited exactly once, for any rc (all three kernels).
#include <array>
#include <cstdio>
#include <mutex>
#include <vector>

#include "kspace.cuh"
#include "real.cuh"
#include "sort.cuh"

#ifndef SE1P_REAL_TABLE
#define SE1P_REAL_TABLE 1
#endif
// 2: warp per 32 sorted targets, candidates culled against the warp's bounding box and the pairs
//    within rc evaluated densely after a warp-level compaction (k_real_warp);
// 1: warp per cell with hit masks (k_real_cells); 0: thread per target (k_real_sum).
// Measured at C4/C5 (round 2): kernel 0 27.1/26.3 ms, kernel 1 34.8/29.9 ms -- the box-to-box
// culling of a cell's neighbours scans ~1.5x the candidates of per-target culling and the warp
// issues more instructions per pair (7.1 against 5.5 per pair within rc; ncu: shared-load latency
// on the broadcast candidates and the lane-divergent table rows).  Estrin's scheme: +-2 %.
#ifndef SE1P_REAL_KERNEL
#define SE1P_REAL_KERNEL 2
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

// k_real_warp's keys: column (x cell, y cell), then a fine z bin (~2 particles per bin), so that
// 32 consecutive sorted targets are a compact box and any z interval of a column is one index range.
__global__ void k_real_keys_fine(RDev d, const double* __restrict__ x, int64_t N, int* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double pz = x[3 * i + 2];
  pz -= d.L[2] * floor(pz / d.L[2]);
  if (pz >= d.L[2]) pz -= d.L[2];
  const int cx = min(max((int)floor(x[3 * i] / d.cs[0]), 0), d.nc[0] - 1);
  const int cy = min(max((int)floor(x[3 * i + 1] / d.cs[1]), 0), d.nc[1] - 1);
  const int fz = min(max((int)floor(pz / d.hz), 0), d.nzf - 1);
  keys[i] = (cx * d.nc[1] + cy) * d.nzf + fz;
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
                                                  const int* __restrict__ cell_start, int64_t t_lo, int64_t t_hi,
                                                  double* __restrict__ phi_out, double* __restrict__ field_out) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= t_hi) return;
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


// ---------------------------------------------------------------- k_real_warp (SE1P_REAL_KERNEL 2)
// Warp per group of <= 32 targets of one column (one per lane; the column-then-fine-z order makes a
// group a compact box).  The warp walks the columns whose xy distance to its bounding box is <= rc;
// in each, the z interval within rc of the box is one index range per periodic image.  Candidates
// are loaded 32 at a time (coalesced), culled one per lane against the box, and the survivors
// staged in a 64-entry shared ring.  A *phase* (rw_phase) tests 32 staged candidates against every
// lane's target into hit masks, then walks the candidates any lane hits with every lane evaluating
// each and keeping its own term by a select.  erfc(xi r) from a small shared-memory table
// (rw_pair).  Each target sums its terms in candidate order: deterministic.  (Measured and not
// kept: the hit test in fp32 with a safe margin and an fp64 re-test at evaluation, +5 % at C5:
// the extra fp32 copy of the ring costs more than the cheaper test saves.)
#ifndef SE1P_REAL_RWW
#define SE1P_REAL_RWW 4
#endif
constexpr int kRWW = SE1P_REAL_RWW;        // warps per block (at most; fewer for small systems)
struct RWarpSm {
  double4 cand[64];                        // staged candidates: x, y, z + image shift, q (ring)
};

// 1/sqrt(r2) for normal r2 > 0: the hardware estimate and two Newton steps (relative error of
// the estimate < 2^-22, after two steps at the rounding level); no special-case paths.
__device__ __forceinline__ double rw_rsqrt(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  double e = fma(-r2 * y, y, 1.0);
  y = fma(0.5 * e, y, y);
  e = fma(-r2 * y, y, 1.0);
  return fma(0.5 * e, y, y);
}

// q_n erfc(xi r)/r (and, FIELD, g = q_n (erfc(xi r)/r - d/dr erfc(xi r))/r^2) of one pair, from
// k_real_warp's shared table: kRealK intervals of [0, rc], on each a polynomial of degree DEG in
// u = r - r_mid, coefficient-major [DEG + 1][kRealK].  A read of one coefficient by the 32 lanes
// costs two shared-memory wavefronts whatever the intervals (8-byte words, two half-warps), so
// the coefficient count is what the data pipe pays for; a 300-interval table in L1 cost ~12
// wavefronts per 16-byte load (measured: the L1 data pipe saturated at 97 %).
#ifndef SE1P_REAL_K
#define SE1P_REAL_K 32
#endif
constexpr int kRealK = SE1P_REAL_K;   // intervals of the shared table (16 / 64 / 128 measured slower)
template <bool FIELD, int DEG>
__device__ __forceinline__ double rw_pair(const RDev& d, const double* __restrict__ tab, double r2, double qj,
                                          double& g) {
  const double rinv = rw_rsqrt(r2);
  const double r = r2 * rinv;
  const int it = min((int)(r * d.tinvw), kRealK - 1);
  const double u = r - ((double)it + 0.5) * d.tw;
  const double* cf = tab + it;
  double pv = cf[DEG * kRealK];
  double dv = 0.0;
  if (FIELD) dv = (double)DEG * pv;
#pragma unroll
  for (int n = DEG - 1; n >= 0; --n) {
    const double c = cf[n * kRealK];
    pv = fma(pv, u, c);
    if (FIELD && n > 0) dv = fma(dv, u, (double)n * c);
  }
  const double ec = pv * rinv;
  if (FIELD) g = qj * (ec - dv) * (rinv * rinv);
  return qj * ec;
}

template <bool FIELD, int DEG>
__device__ __forceinline__ void rw_eval(const double4& pt, const double4& cc, bool hit, double rc2, const RDev& d,
                                        const double* tab, double& acc, double& ex, double& ey, double& ez) {
  const double dx = pt.x - cc.x, dy = pt.y - cc.y, dz = pt.z - cc.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double g = 0.0;
  const double v = rw_pair<FIELD, DEG>(d, tab, hit ? r2 : rc2, cc.w, g);
  acc += hit ? v : 0.0;
  if (FIELD) {
    const double gg = hit ? g : 0.0;
    ex = fma(gg, dx, ex);
    ey = fma(gg, dy, ey);
    ez = fma(gg, dz, ez);
  }
}

// One phase: n staged candidates from ring slot base (base + n <= 64) against the warp's targets,
// one target per lane, candidates broadcast from shared memory.  First every lane tests its target
// against the n candidates into a hit mask (independent, cheap); then the warp walks the
// candidates that any lane has within rc, four at a time (independent chains), every lane
// evaluating them and keeping its own terms by a select -- a lane-divergent "if within rc" would
// idle the lanes outside while the others evaluate.  Misses evaluate at r^2 = rc^2 (finite).  The
// prime in Eq. (3) (n = m in the unshifted image) is the pair at r^2 = 0 exactly: a target meets
// itself with identical coordinates, and a distinct particle at zero distance would make phi
// infinite (not a valid input).
#ifndef SE1P_REAL_WALK
#define SE1P_REAL_WALK 4   // candidates per round of the walk (2, 4 or 8)
#endif
#ifndef SE1P_REAL_WALK_F
#define SE1P_REAL_WALK_F SE1P_REAL_WALK   // the same for the field kernels
#endif
template <bool FIELD, int DEG, bool FULL>
__device__ __forceinline__ void rw_phase(const RWarpSm& s, int base, int n, const double4& pt, bool active,
                                         double rc2, const RDev& d, const double* tab, double& acc, double& ex,
                                         double& ey, double& ez) {
  constexpr unsigned kAll = 0xffffffffu;
  const double4* cb = s.cand + base;   // slots base .. base + 31 stay inside the ring
  unsigned m = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (FULL || k < n) {
      const double4 cc = cb[k];
      const double dx = pt.x - cc.x, dy = pt.y - cc.y, dz = pt.z - cc.z;
      const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
      if (r2 <= rc2 && r2 > 0.0) m |= 1u << k;
    }
  }
  if (!active) m = 0;
  unsigned am = __reduce_or_sync(kAll, m);
  constexpr int W = FIELD ? SE1P_REAL_WALK_F : SE1P_REAL_WALK;
  if (W >= 4) {
    while (am) {   // W candidates per round (independent chains)
      int kk[W >= 4 ? W : 4];
      bool ok[W >= 4 ? W : 4];
#pragma unroll
      for (int i = 0; i < W; ++i) {
        ok[i] = am != 0;
        kk[i] = ok[i] ? __ffs(am) - 1 : 0;
        am &= am - 1;
      }
#pragma unroll
      for (int i = 0; i < W; ++i)
        rw_eval<FIELD, DEG>(pt, cb[kk[i]], ok[i] && ((m >> kk[i]) & 1u), rc2, d, tab, acc, ex, ey, ez);
    }
  } else {
    while (am) {
      const int k1 = __ffs(am) - 1;
      am &= am - 1;
      const bool two = am != 0;
      const int k2 = two ? __ffs(am) - 1 : k1;
      am &= am - 1;
      const double4 c1 = cb[k1], c2 = cb[k2];
      rw_eval<FIELD, DEG>(pt, c1, (m >> k1) & 1u, rc2, d, tab, acc, ex, ey, ez);
      rw_eval<FIELD, DEG>(pt, c2, two && ((m >> k2) & 1u), rc2, d, tab, acc, ex, ey, ez);
    }
  }
}

// groups per column: ceil(n/32) (k_real_warp's target groups)
__global__ void k_real_group_counts(const int* __restrict__ bin_start, int ncol, int nzf, int* __restrict__ g) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncol) g[c] = (bin_start[(c + 1) * nzf] - bin_start[c * nzf] + 31) / 32;
}

#ifdef SE1P_REAL_COUNT   // experiment: chunks, survivors, full phases, pairs
__device__ unsigned long long g_rw_cnt[4];
__device__ double g_rw_ext[4];
#endif
template <bool FIELD, int DEG>
#ifndef SE1P_REAL_MINB
#define SE1P_REAL_MINB 4
#endif
__global__ void __launch_bounds__(kRWW * 32, SE1P_REAL_MINB) k_real_warp(RDev d, const double4* __restrict__ P4,
                                                         const int* __restrict__ perm,
                                                         const int* __restrict__ bin_start,
                                                         const int* __restrict__ gstart, int ncol, int part,
                                                         int nparts, double* __restrict__ phi_out,
                                                         double* __restrict__ field_out) {
  constexpr unsigned kAll = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char rw_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RWarpSm& s = reinterpret_cast<RWarpSm*>(rw_raw)[warp];
  const int nw = blockDim.x >> 5;
  double* tab = reinterpret_cast<double*>(rw_raw + nw * sizeof(RWarpSm));
  for (int i = threadIdx.x; i < (DEG + 1) * kRealK; i += blockDim.x) tab[i] = d.tab2[i];
  __syncthreads();
  // target group gw: column col's sorted run cut into G = ceil(n/32) near-equal pieces (groups
  // never straddle two columns, so the box stays compact); col by a 32-ary search of gstart
  // part `part` of `nparts` (ranks sharing the sum): groups [G part / nparts, G (part+1) / nparts)
  const int gtot = gstart[ncol];
  const int g_hi = (int)(((int64_t)gtot * (part + 1)) / nparts);
  const int gw = (int)(((int64_t)gtot * part) / nparts) + blockIdx.x * nw + warp;
  if (gw >= g_hi) return;
  int clo = 0, chi = ncol;   // gstart[clo] <= gw < gstart[chi]
  while (chi - clo > 1) {
    const int step = (chi - clo + 31) / 32;
    const int ci = clo + lane * step;
    const unsigned le = __ballot_sync(kAll, ci < chi && gstart[ci] <= gw);
    clo += (31 - __clz(le)) * step;
    chi = min(chi, clo + step);
  }
  const int cbeg = bin_start[clo * d.nzf], nsrc = bin_start[(clo + 1) * d.nzf] - cbeg;
  const int G = (nsrc + 31) / 32, kg = gw - gstart[clo];
  const int t0 = cbeg + (int)(((int64_t)kg * nsrc) / G), t1 = cbeg + (int)(((int64_t)(kg + 1) * nsrc) / G);
  const int tl = t0 + lane;
  const bool active = tl < t1;
  const double4 pt = P4[active ? tl : t0];
  double lo0 = pt.x, lo1 = pt.y, lo2 = pt.z, hi0 = pt.x, hi1 = pt.y, hi2 = pt.z;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo0 = fmin(lo0, __shfl_xor_sync(kAll, lo0, o));
    lo1 = fmin(lo1, __shfl_xor_sync(kAll, lo1, o));
    lo2 = fmin(lo2, __shfl_xor_sync(kAll, lo2, o));
    hi0 = fmax(hi0, __shfl_xor_sync(kAll, hi0, o));
    hi1 = fmax(hi1, __shfl_xor_sync(kAll, hi1, o));
    hi2 = fmax(hi2, __shfl_xor_sync(kAll, hi2, o));
  }
  const double rc2 = d.rc * d.rc;
  const double rc2c = rc2 * (1.0 + 1e-12);   // culling bound: never drops a pair within rc
  const int nc1 = d.nc[1], nzf = d.nzf;
  double acc = 0.0, ex = 0.0, ey = 0.0, ez = 0.0;
  int base = 0, ns = 0;                       // staged ring: first slot and count (warp-uniform)
  const int ax0 = max(0, (int)floor((lo0 - d.rc) / d.cs[0])), ax1 = min(d.nc[0] - 1, (int)floor((hi0 + d.rc) / d.cs[0]));
  const int ay0 = max(0, (int)floor((lo1 - d.rc) / d.cs[1])), ay1 = min(nc1 - 1, (int)floor((hi1 + d.rc) / d.cs[1]));
  for (int ax = ax0; ax <= ax1; ++ax) {
    const double gx = fmax(fmax(ax * d.cs[0] - hi0, lo0 - (ax + 1) * d.cs[0]), 0.0);
    for (int ay = ay0; ay <= ay1; ++ay) {
      const double gy = fmax(fmax(ay * d.cs[1] - hi1, lo1 - (ay + 1) * d.cs[1]), 0.0);
      const double rem = rc2c - gx * gx - gy * gy;
      if (rem < 0.0) continue;
      const double rz = sqrt(rem);
      // fine bins of the z interval [lo2 - rz, hi2 + rz], one bin of margin each side (rounding)
      const int fl = (int)floor((lo2 - rz) / d.hz) - 1, fh = (int)floor((hi2 + rz) / d.hz) + 1;
      const int colbase = (ax * nc1 + ay) * nzf;
      const int w1 = rfloordiv(fh, nzf);
      for (int w = rfloordiv(fl, nzf); w <= w1; ++w) {
        const int fa = max(fl - w * nzf, 0), fb = min(fh - w * nzf, nzf - 1);
        const int js = bin_start[colbase + fa], je = bin_start[colbase + fb + 1];
        const double shift = w * d.L[2];
        for (int j0 = js; j0 < je; j0 += 32) {
          const int j = j0 + lane;
          const bool ok = j < je;
          double4 cc = ok ? P4[j] : make_double4(0.0, 0.0, 0.0, 0.0);
          cc.z += shift;
          const double g0 = fmax(fmax(lo0 - cc.x, cc.x - hi0), 0.0);
          const double g1 = fmax(fmax(lo1 - cc.y, cc.y - hi1), 0.0);
          const double g2 = fmax(fmax(lo2 - cc.z, cc.z - hi2), 0.0);
          const bool keep = ok && fma(g0, g0, fma(g1, g1, g2 * g2)) <= rc2c;
          const unsigned m = __ballot_sync(kAll, keep);
          if (keep) {
            const int pos = (base + ns + __popc(m & ((1u << lane) - 1u))) & 63;
            s.cand[pos] = cc;
          }
          ns += __popc(m);
#ifdef SE1P_REAL_COUNT
          const unsigned mok = __ballot_sync(kAll, ok);
          if (lane == 0) { atomicAdd(&g_rw_cnt[0], 1ull); atomicAdd(&g_rw_cnt[1], (unsigned long long)__popc(m));
                           atomicAdd(&g_rw_ext[3], (double)__popc(mok)); }
#endif
          __syncwarp();
          if (ns >= 32) {
            rw_phase<FIELD, DEG, true>(s, base, 32, pt, active, rc2, d, tab, acc, ex, ey, ez);
            base = (base + 32) & 63;
            ns -= 32;
#ifdef SE1P_REAL_COUNT
            if (lane == 0) atomicAdd(&g_rw_cnt[2], 1ull);
#endif
          }
        }
      }
    }
  }
#ifdef SE1P_REAL_COUNT
  if (lane == 0) {
    atomicAdd(&g_rw_cnt[3], 1ull);
    atomicAdd(&g_rw_ext[0], hi0 - lo0);
    atomicAdd(&g_rw_ext[1], hi1 - lo1);
    atomicAdd(&g_rw_ext[2], hi2 - lo2);
  }
#endif
  if (ns > 0) rw_phase<FIELD, DEG, false>(s, base, ns, pt, active, rc2, d, tab, acc, ex, ey, ez);
  if (active) {
    const int64_t uo = perm[tl];
    if (phi_out) phi_out[uo] = acc - 2.0 * d.xi * pt.w * 0.564189583547756286948079451560772586;  // 1/sqrt(pi)
    if (FIELD) {
      field_out[3 * uo] = ex;
      field_out[3 * uo + 1] = ey;
      field_out[3 * uo + 2] = ez;
    }
  }
}

template <bool FIELD, int DEG>
static void launch_real_warp_deg(const RDev& d, const double4* P4, const int* perm, const int* bin_start,
                                 const int* gstart, int64_t N, int part, int nparts, double* phi_out,
                                 double* field_out, cudaStream_t st) {
  // warps per block: 8, halved while that leaves fewer than two blocks per SM (small systems)
  const int ncol = d.nc[0] * d.nc[1];
  const int64_t groups = ceil_div(ceil_div(N, 32) + ncol, nparts) + 1;   // >= this part's groups
  int nw = kRWW;
  while (nw > 1 && ceil_div(groups, nw) < 2 * 148) nw /= 2;
  const size_t smem = nw * sizeof(RWarpSm) + (size_t)(DEG + 1) * kRealK * sizeof(double);
  SE1P_CUDA_TRY(cudaFuncSetAttribute((const void*)k_real_warp<FIELD, DEG>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned nb = (unsigned)ceil_div(groups, nw);
#ifdef SE1P_REAL_COUNT
  unsigned long long z[4] = {0, 0, 0, 0};
  SE1P_CUDA_TRY(cudaMemcpyToSymbol(g_rw_cnt, z, sizeof(z)));
  double ze[4] = {0, 0, 0, 0};
  SE1P_CUDA_TRY(cudaMemcpyToSymbol(g_rw_ext, ze, sizeof(ze)));
#endif
  k_real_warp<FIELD, DEG><<<nb, nw * 32, smem, st>>>(d, P4, perm, bin_start, gstart, ncol, part, nparts, phi_out,
                                                       field_out);
  SE1P_LAUNCH_CHECK();
#ifdef SE1P_REAL_COUNT
  SE1P_CUDA_TRY(cudaMemcpyFromSymbol(z, g_rw_cnt, sizeof(z)));
  SE1P_CUDA_TRY(cudaMemcpyFromSymbol(ze, g_rw_ext, sizeof(ze)));
  fprintf(stderr, "bbox mean %g %g %g loaded %g\n", ze[0] / z[3], ze[1] / z[3], ze[2] / z[3], ze[3] / z[3]);
  fprintf(stderr, "k_real_warp N=%lld nzf=%d degree %d: chunks %llu survivors %llu full phases %llu warps %llu\n",
          (long long)N, d.nzf, DEG, z[0], z[1], z[2], z[3]);
#endif
}

// the compiled table degrees (a fitted degree is padded up to the next)
constexpr int kRealDeg[] = {7, 8, 9, 10, 11, 13, 15, 19, 23, 31};
template <bool FIELD>
static void launch_real_warp(const RDev& d, const double4* P4, const int* perm, const int* bin_start,
                             const int* gstart, int64_t N, int part, int nparts, double* phi_out, double* field_out,
                             cudaStream_t st) {
#define SE1P_RW_CASE(D)                                                                                    \
  case D:                                                                                                  \
    launch_real_warp_deg<FIELD, D>(d, P4, perm, bin_start, gstart, N, part, nparts, phi_out, field_out, st); \
    break;
  switch (d.tdeg) {
    SE1P_RW_CASE(7) SE1P_RW_CASE(8) SE1P_RW_CASE(9) SE1P_RW_CASE(10) SE1P_RW_CASE(11)
    SE1P_RW_CASE(13) SE1P_RW_CASE(15) SE1P_RW_CASE(19) SE1P_RW_CASE(23) SE1P_RW_CASE(31)
    default: throw Error{6, "real space: no kernel for this table degree"};
  }
#undef SE1P_RW_CASE
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
  // ~2 particles per fine z bin, at most 2^22 bins in all
  const int64_t ncol = (int64_t)d.nc[0] * d.nc[1];
  const int64_t nz = std::max<int64_t>(1, (N + 2 * ncol - 1) / (2 * ncol));
  d.nzf = (int)std::min<int64_t>(nz, std::max<int64_t>(1, ((int64_t)1 << 22) / ncol));
  d.hz = L[2] / d.nzf;
#if SE1P_REAL_KERNEL == 2 && SE1P_REAL_TABLE
  d.tdeg = real_table_deg(xi, rc);   // 0: xi rc beyond the shared table, thread-per-target kernel
#endif
  return d;
}

int64_t real_scratch_ints(const RDev& d, int64_t N) {
  const int64_t ncol = (int64_t)d.nc[0] * d.nc[1];
  return std::max<int64_t>(sort_scratch_ints(N, real_nbins(d)), 2 * ncol + 1 + scan_scratch_ints(ncol));
}

int real_nbins(const RDev& d) {
  return d.tdeg > 0 ? d.nc[0] * d.nc[1] * d.nzf : d.nc[0] * d.nc[1] * d.nc[2];
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

// k_real_warp's few-interval table: kRealK = 32 intervals of [0, rc]; on each, the polynomial in
// u = r - r_mid interpolating erfc(xi r) at the interval's Chebyshev points (erfcl, long double),
// converted to monomial coefficients.  The degree is the smallest for which every interval stays
// within 2e-16 of erfc in absolute terms (checked on 65 points per interval in long double): half
// an ulp of erfc(0) = 1, so a pair's error is at most that of the rounding of the nearest pairs'
// terms, which dominate the sum -- degree 8 at xi rc = 3 (C5), 9 at 4.6 - 4.9 (C1 - C4, C5 at
// rc = 0.164).  (2e-16 *relative* to erfc, the 300-interval table's target, takes 9 and 12 - 13:
// the tail intervals, where erfc is small, decide it; Taylor polynomials about the midpoints take
// ~3 degrees more again.)  The degree is padded up to a compiled one (kRealDeg).  Beyond degree
// 31 real_space falls back to the thread-per-target kernel and its long Taylor table.
static bool cheb_interval(double xi, long double rmid, long double hw, int n, long double* mono) {
  long double f[32], a[32], T[32][32] = {}, tm[32] = {};
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k = 0; k <= n; ++k) f[k] = erfcl((long double)xi * (rmid + hw * cosl(pi * (k + 0.5L) / (n + 1))));
  for (int j = 0; j <= n; ++j) {
    long double sum = 0.0L;
    for (int k = 0; k <= n; ++k) sum += f[k] * cosl(pi * j * (k + 0.5L) / (n + 1));
    a[j] = sum * 2.0L / (n + 1);
  }
  a[0] *= 0.5L;
  T[0][0] = 1.0L;   // monomial coefficients of T_j(t)
  if (n >= 1) T[1][1] = 1.0L;
  for (int j = 2; j <= n; ++j)
    for (int m = 0; m <= j; ++m) T[j][m] = (m > 0 ? 2.0L * T[j - 1][m - 1] : 0.0L) - T[j - 2][m];
  for (int j = 0; j <= n; ++j)
    for (int m = 0; m <= j; ++m) tm[m] += a[j] * T[j][m];
  long double sc = 1.0L;   // t = u / hw
  for (int m = 0; m <= n; ++m) {
    mono[m] = tm[m] / sc;
    sc *= hw;
  }
  for (int k = 0; k <= 64; ++k) {   // relative error on a fine grid
    const long double u = hw * (-1.0L + 2.0L * k / 64.0L);
    long double pv = mono[n];
    for (int m = n - 1; m >= 0; --m) pv = pv * u + mono[m];
    const long double e = erfcl((long double)xi * (rmid + u));
    if (fabsl(pv - e) > 2e-16L) return false;
  }
  return true;
}

// degree and monomial coefficients [K][32] (0 past the degree); degree 0: not representable
static std::vector<long double> erfc_cheb_k(double xi, double rc, int& deg) {
  const int K = kRealK;
  const long double w = (long double)rc / K, hw = 0.5L * w;
  std::vector<long double> c((size_t)K * 32, 0.0L);
  for (deg = 3; deg <= 31; ++deg) {
    bool ok = true;
    for (int i = 0; i < K && ok; ++i) ok = cheb_interval(xi, ((long double)i + 0.5L) * w, hw, deg, &c[(size_t)i * 32]);
    if (ok) return c;
    std::fill(c.begin(), c.end(), 0.0L);
  }
  deg = 0;
  return c;
}

int real_table_deg(double xi, double rc) {   // memoised: the fit costs milliseconds of host time
  static std::mutex mu;
  static std::vector<std::array<double, 3>> memo;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& m : memo)
      if (m[0] == xi && m[1] == rc) return (int)m[2];
  }
  int deg = 0, td = 0;
  erfc_cheb_k(xi, rc, deg);
  if (deg > 0)
    for (int v : kRealDeg)
      if (v >= deg) {
        td = v;
        break;
      }
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() > 64) memo.clear();
  memo.push_back({xi, rc, (double)td});
  return td;
}

static std::vector<double> erfc_small_table(double xi, double rc, int tdeg) {
  int deg = 0;
  const std::vector<long double> c = erfc_cheb_k(xi, rc, deg);
  const int K = kRealK;
  std::vector<double> t((size_t)(tdeg + 1) * K, 0.0);   // coefficient-major [tdeg + 1][K]
  for (int n = 0; n <= tdeg; ++n)
    for (int i = 0; i < K; ++i) t[(size_t)n * K + i] = n <= deg ? (double)c[(size_t)i * 32 + n] : 0.0;
  return t;
}

std::vector<double> real_table_host(double xi, double rc, int& degree, int& intervals) {
  degree = real_table_deg(xi, rc);
  intervals = kRealK;
  return degree > 0 ? erfc_small_table(xi, rc, degree) : std::vector<double>();
}

struct TabCache {
  double xi = 0, rc = 0;
  double* dev = nullptr;
  int64_t cap = 0;
};
static TabCache g_tab[64];
struct SmallTabCache {
  double xi = 0, rc = 0;
  double* dev = nullptr;
  int64_t cap = 0;
};
static SmallTabCache g_tab2[64];

void real_release_tables(int dev) {
  TabCache& tc = g_tab[dev & 63];
  if (tc.dev) dev_free(tc.dev);
  tc = TabCache{};
  SmallTabCache& t2 = g_tab2[dev & 63];
  if (t2.dev) dev_free(t2.dev);
  t2 = SmallTabCache{};
}

void real_space(const RDev& d0, KWork& w, const double* x, const double* q, int64_t N, double* phi_out,
                cudaStream_t st, double* field_out, int part, int nparts) {
  RDev d = d0;
#if SE1P_REAL_TABLE
  if (d.tdeg == 0) {
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
  if (d.tdeg > 0) {   // k_real_warp's shared table
    int dev = 0;
    SE1P_CUDA_TRY(cudaGetDevice(&dev));
    SmallTabCache& tc = g_tab2[dev & 63];
    if (!tc.dev || tc.xi != d.xi || tc.rc != d.rc) {
      const std::vector<double> t = erfc_small_table(d.xi, d.rc, d.tdeg);
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
    d.tab2 = tc.dev;
    d.tw = d.rc / kRealK;
    d.tinvw = kRealK / d.rc;
  }
  const int nbins = real_nbins(d);
  const unsigned nb = (unsigned)ceil_div(N, 256);
  if (d.tdeg > 0)
    k_real_keys_fine<<<nb, 256, 0, st>>>(d, x, N, w.keys);
  else
    k_real_keys<<<nb, 256, 0, st>>>(d, x, N, w.keys);
  SE1P_LAUNCH_CHECK();
  stable_bin_sort(w.keys, N, nbins, w.perm, w.bin_start, w.scratch, st);
  k_real_permute<<<nb, 256, 0, st>>>(d, x, q, w.perm, N, (double4*)w.xs);
  SE1P_LAUNCH_CHECK();
  if (d.tdeg > 0) {
    const int ncol = d.nc[0] * d.nc[1];
    int* gcnt = w.scratch;   // the sort's scratch is free again (real_scratch_ints sizes it)
    int* gstart = gcnt + ncol;
    k_real_group_counts<<<(unsigned)ceil_div(ncol, 256), 256, 0, st>>>(w.bin_start, ncol, d.nzf, gcnt);
    SE1P_LAUNCH_CHECK();
    exclusive_scan_ints(gcnt, ncol, gstart, gstart + ncol + 1, st);
    if (field_out)
      launch_real_warp<true>(d, (const double4*)w.xs, w.perm, w.bin_start, gstart, N, part, nparts, phi_out,
                             field_out, st);
    else
      launch_real_warp<false>(d, (const double4*)w.xs, w.perm, w.bin_start, gstart, N, part, nparts, phi_out,
                              nullptr, st);
    return;
  }
#if SE1P_REAL_KERNEL == 1 && SE1P_REAL_TABLE
  if (nparts > 1) throw Error{1, "real space: parts need the warp or thread-per-target kernel"};
  if (field_out)
    launch_real_cells<true>(d, (const double4*)w.xs, w.perm, w.bin_start, nbins, phi_out, field_out, st);
  else
    launch_real_cells<false>(d, (const double4*)w.xs, w.perm, w.bin_start, nbins, phi_out, nullptr, st);
  return;
#endif
  const int64_t t_lo = N * part / nparts, t_hi = N * (part + 1) / nparts;   // this part's sorted targets
  const unsigned nt = (unsigned)std::max<int64_t>(1, ceil_div(t_hi - t_lo, 128));
  if (field_out)
    k_real_sum<true><<<nt, 128, 0, st>>>(d, (const double4*)w.xs, w.perm, w.bin_start, t_lo, t_hi, phi_out, field_out);
  else
    k_real_sum<false><<<nt, 128, 0, st>>>(d, (const double4*)w.xs, w.perm, w.bin_start, t_lo, t_hi, phi_out, nullptr);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
