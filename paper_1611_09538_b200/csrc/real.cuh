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
};

RDev real_geometry(const double L[3], double xi, double rc, int64_t N);
void real_space(const RDev& d, KWork& w, const double* x, const double* q, int64_t N, double* phi_out,
                cudaStream_t st, double* field_out = nullptr);

}  // namespace se1p
