// real.cuh -- real-space geometry (see real.cu).
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

#include "kspace.cuh"

namespace se1p {

struct RDev {
  double L[3];
  double cs[3];   // cell sizes
  int nc[3];      // cells per axis
  int K;          // periodic-axis cell reach
  int Kx, Ky;     // free-axis cell reach (cells are >= rc/D wide)
  double xi, rc;
  // k_real_warp's sort bins: columns (x cell, y cell) of nzf fine z bins hz = L3/nzf wide
  int nzf = 1;
  double hz = 0.0;
  // erfc(xi r) on [0, rc] as ntab local Taylor polynomials of degree kTabDeg in r - r_mid
  const double* tab = nullptr;
  int ntab = 0;
  double inv_dr = 0.0, dr = 0.0;
  // k_real_warp's table: kRealK intervals of [0, rc] (width tw), polynomials of degree tdeg in
  // r - r_mid, coefficient-major [tdeg + 1][kRealK] (real.cu)
  const double* tab2 = nullptr;
  int tdeg = 0;
  double tw = 0.0, tinvw = 0.0;
};
// degree 7 (8 coefficients, four 16-byte loads per pair); the interval count grows with
// X = xi rc so that the remainder (2 X dx)^8/8! (dx the interval half-width in xi r) stays
// below 1e-16 relative: ntab = X^2 / 0.03 (C5: 300 intervals, 19 KB)
constexpr int kTabDeg = 7;
inline int real_table_intervals(double xi, double rc) {
  const double X = xi * rc;
  return std::min(8192, std::max(64, (int)std::ceil(X * X / 0.03)));
}

RDev real_geometry(const double L[3], double xi, double rc, int64_t N);
int real_nbins(const RDev& d);   // bins of the real-space sort (workspace sizing)
int64_t real_scratch_ints(const RDev& d, int64_t N);
int real_table_deg(double xi, double rc);
// the shared table k_real_warp uses (coefficient-major [degree + 1][intervals]; empty if degree 0)
std::vector<double> real_table_host(double xi, double rc, int& degree, int& intervals);   // k_real_warp's table degree, 0 if unsupported   // ints of KWork::scratch the real-space sum needs
// part/nparts: only the targets of part `part` (the warp kernel's target groups, or sorted targets
// for the fallback kernel, split in nparts near-equal ranges) are written
void real_space(const RDev& d, KWork& w, const double* x, const double* q, int64_t N, double* phi_out,
                cudaStream_t st, double* field_out = nullptr, int part = 0, int nparts = 1);
void real_release_tables(int dev);   // the cached erfc table of device dev

}  // namespace se1p
