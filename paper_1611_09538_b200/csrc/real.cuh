// real.cuh -- real-space geometry (see real.cu).
#pragma once
#include <algorithm>
#include <cmath>

#include "kspace.cuh"

namespace se1p {

struct RDev {
  double L[3];
  double cs[3];   // cell sizes
  int nc[3];      // cells per axis
  int K;          // periodic-axis cell reach
  int Kx, Ky;     // free-axis cell reach (cells are >= rc/D wide)
  double xi, rc;
  // erfc(xi r) on [0, rc] as kTabN local Taylor polynomials of degree kTabDeg in r - r_mid
  const double* tab = nullptr;
  double inv_dr = 0.0, dr = 0.0;
};
constexpr int kTabN = 256, kTabDeg = 10;

RDev real_geometry(const double L[3], double xi, double rc, int64_t N);
void real_space(const RDev& d, KWork& w, const double* x, const double* q, int64_t N, double* phi_out,
                cudaStream_t st, double* field_out = nullptr);
void real_release_tables(int dev);   // the cached erfc table of device dev

}  // namespace se1p
