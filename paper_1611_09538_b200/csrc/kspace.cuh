// kspace.cuh -- plan and workspace of the SE1P k-space path (Alg. 1).
#pragma once
#include <vector>

#include "../../include/se1p.h"
#include "fft.cuh"

namespace se1p {

// plan-time scratch of the kernel-spectrum builder (build_kernel_spectrum, modes.cu)
struct KernScratch {
  double* tmp;   // [Mt][S/2+1]
  double2* A;    // [LK][LK]
  double2* B;    // [LK][LK]
};


// Particle bins: x bands of kBin cells; inside a band by periodic stencil start, then y cell.
constexpr int kBin = 4;

// Layout of a k3-plane buffer: rows x in [xlo[0], xlo[nslab]) split into
// nslab consecutive x slabs; slab r holds, for each of the nloc plane slots i, its rows
// xlo[r] .. xlo[r+1]-1.  Element (i, x, y) lives at slab_row(L, i, x, Mt) + y:
//   ((nloc (xlo[r] - xlo[0]) + i (xlo[r+1] - xlo[r]) + x - xlo[r]) Mt + y).
// Single GPU: nslab = 1, xlo = {0, Mt}, nloc = M/2+1 -> the plain [plane][x][y] array.
constexpr int kMaxSlabs = 16;
struct SlabLayout {
  int nslab;
  int nloc;
  int xlo[kMaxSlabs + 1];
};
__host__ __device__ inline int64_t slab_row(const SlabLayout& L, int i, int x, int Mt) {
  int r = 0;
  while (r + 1 < L.nslab && x >= L.xlo[r + 1]) ++r;
  const int W = L.xlo[r + 1] - L.xlo[r];
  return ((int64_t)L.nloc * (L.xlo[r] - L.xlo[0]) + (int64_t)i * W + (x - L.xlo[r])) * Mt;
}
inline SlabLayout single_layout(int Mt, int nloc) {
  SlabLayout L{};
  L.nslab = 1;
  L.nloc = nloc;
  L.xlo[0] = 0;
  L.xlo[1] = Mt;
  return L;
}

struct KParams {       // everything a k-space plan is keyed on
  double L[3];
  double xi;
  int M, P;
  double eta;          // resolved (> 0)
  int n_l;             // resolved (>= 0)
  int S0, SI, SJ;      // resolved padded extents
  int periodic = 0;    // 1: SE3P transform plan (grid Mfree x Mfree x M, every plane a J plane, SJ = Mfree)
  std::vector<int> SIn;   // multi-tier upsampling: extent of mode n = 1..n_l (empty: SI for all)
  int device = -1;        // the plan cache keys plans per device (kplan_get)
  bool operator==(const KParams& o) const {
    return device == o.device && L[0] == o.L[0] && L[1] == o.L[1] && L[2] == o.L[2] && xi == o.xi && M == o.M && P == o.P &&
           eta == o.eta && n_l == o.n_l && S0 == o.S0 && SI == o.SI && SJ == o.SJ && periodic == o.periodic &&
           SIn == o.SIn;
  }
};

// Device view of the plan, passed by value to kernels.
struct KDev {
  int M, P, Mfree, Mt;          // grid: Mt x Mt (free, extended) x M (periodic)
  double h, inv_h, alpha;       // alpha = 2 xi^2 / eta (window exponent)
  double L3;
  int nbx;                      // bins: x bands of kBin cells
  int nsxy, nsz, nslot;         // gather partial slots per particle
  int* err;                     // device error word of the tile kernels (bounds checks)
  int64_t N;
};

struct KPlan {
  KParams prm;
  KDev dv;
  int LK = 0;                   // FFT extent of the kernel (upsampled) planes
  int n_planes = 0;             // M/2 + 1
  int n_kernel = 0;             // planes 0..n_kernel-1 use the plan-time kernel (k3 = 0 and I)
  FftDesc fz, fJ, fK;           // FFT lengths M, SJ, LK
  double2* d_tw = nullptr;      // all twiddle tables
  int twz = 0, twJ = 0, twK = 0;
  double* d_khat = nullptr;     // [n_kernel][LK][LK] real kernel spectra (constants folded)
  double* d_exJ = nullptr;      // [SJ] e^{-(1-eta) kappa_a^2/(4 xi^2)}, kappa_a = 2 pi a'/(SJ h)
  double* d_k2J = nullptr;      // [SJ] kappa_a^2
  double* d_pl = nullptr;       // [n_planes][2]: e^{-(1-eta) k3^2/(4xi^2)} * C_J, k3^2
  double* d_f1 = nullptr;       // [P] e^{-alpha h^2 t^2}, the particle-independent FGG factor
  int64_t t_off_total = 0;      // workspace T size (complex) for the 2D passes
  std::vector<int64_t> t_off;   // per plane offset into T
  double const_gather = 0;      // 4 pi h^3 (2 xi^2/(pi eta))^3 (reading R-1)
  double plan_ms = 0;
};

struct KWork {                  // per-N workspace (grown on demand)
  int64_t cap_xs = 0, cap_perm = 0, cap_keys = 0, cap_bs = 0;
  double* xs = nullptr;         // sorted particles: x, y, z (folded), q  (double4 per particle)
  int* s4 = nullptr;            // sorted stencil starts: jx0, jy0, lz0, lz0 mod M (int4)
  int64_t cap_s4 = 0;
  double* rec = nullptr;        // sorted particle records (tiles.cuh, k_records)
  int64_t cap_rec = 0;
  int* perm = nullptr;          // sorted position -> original index
  int* keys = nullptr;
  int* bin_start = nullptr;
  int* scratch = nullptr;       // sort scratch (sort_scratch_ints)
  int64_t scratch_cap = 0;
  double* grid = nullptr;       // real grid Mt x Mt x M (H, then H~)
  double* grid3 = nullptr;      // SE3P: the folded periodic grid Mfree x Mfree x M
  int64_t grid3_cap = 0;
  double2* planes = nullptr;    // Hk: n_planes x Mt x Mt
  double2* T = nullptr;         // 2D pass workspace
  int64_t grid_cap = 0, planes_cap = 0, T_cap = 0;
  double* gpart = nullptr;      // gather partials [slot][value][N]
  int64_t gpart_cap = 0;
  double* over = nullptr;       // gridding overhang [chunk][Mt][Mt][P-1] (sweep.cu)
  int64_t over_cap = 0;
  int* items = nullptr;         // sweep work items + work counter
  int64_t items_cap = 0;
  double* red = nullptr;        // reductions (neutrality check)
  int* flag = nullptr;
  double* host_x = nullptr;     // staging for host_io
  cudaStream_t side = nullptr;  // second stream of the mode stage (kernel planes beside J planes)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t side2 = nullptr; // third stream (second half of the J planes)
  cudaEvent_t ev_join2 = nullptr;
};

KPlan* kplan_get(const KParams& p, cudaStream_t st);   // cached
void kplan_release_all(int device);   // the plans of one device
uint64_t kplan_generation();   // changes whenever a plan is built or freed
void plan_from_tol(const double L[3], double Q, double xi, double tol, se1p_tol_plan* out);   // planner.cu
double lambert_w0(double x);

// Stages (launch on st).
void k_bin_particles(const KPlan& pl, KWork& w, const double* x, const double* q, int64_t N, cudaStream_t st);
// distributed path (particles.cu): compact the particles meeting slab rows [row_lo, row_hi)
void k_slab_select(const KPlan& pl, const double* x, const double* q, int64_t N, int row_lo, int row_hi, int* flags,
                   int* pos, int* scan_scratch, double* xc, double* qc, int* idmap, cudaStream_t st);
void k_scatter_partial_stage(const double* phic, const int* idmap, int64_t n, double* phi, cudaStream_t st);
void k_records_stage(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, bool field = false);   // sweep.cu
// z-aligned DMMA column sweeps over x tiles [tx_lo, tx_hi) (tx_hi < 0: all), tiles of 16 grid rows
void k_spread_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo = 0, int tx_hi = -1);
// field: also E = -grad phi (3 doubles per particle, user order) -- the gradient of the gather
void k_gather_tiles(const KPlan& pl, KWork& w, int64_t N, cudaStream_t st, int tx_lo = 0, int tx_hi = -1,
                    bool field = false);
void k_gather_finish_stage(const KPlan& pl, KWork& w, int64_t N, double* phi_out, cudaStream_t st, int tx_lo = 0,
                           int tx_hi = -1, double* field = nullptr);
int64_t gather_slots(const KDev& dv);
void slot_geometry(KDev& dv);
int64_t sweep_overhang_doubles(const KDev& dv);
int64_t sweep_items_max(const KDev& dv);
void k_zfft_forward(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, const int* slot_of,
                    cudaStream_t st);
void k_mode_stage(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, const int* glK, const int* liK,
                  int nK, const int* glJ, const int* liJ, int nJ, cudaStream_t st);
void k_zfft_inverse(const KPlan& pl, KWork& w, const double2* planes, const SlabLayout& L, const int* slot_of,
                    cudaStream_t st);
// SE3P (se3p.cu): fold the extended grid of the 1P tile plan onto the periodic grid and back
void k_fold_3p(const KPlan& ext, const double* grid_ext, double* grid_per, cudaStream_t st);
void k_unfold_3p(const KPlan& ext, const double* grid_per, double* grid_ext, cudaStream_t st);

}  // namespace se1p
