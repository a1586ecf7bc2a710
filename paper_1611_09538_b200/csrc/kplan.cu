// kplan.cu -- k-space plan: Alg. 1 step 1, FFT descriptors, scaling tables and
// the plan-time kernel spectra of the upsampled planes.
#include <chrono>
#include <cmath>
#include <memory>
#include <vector>

#include "kspace.cuh"

namespace se1p {

void build_kernel_spectrum(const KPlan& pl, int S, const double* d_sig, double* khat_out, double scale,
                           cudaStream_t st);

// 1 - J0(x) without cancellation for small x (series), glibc j0 otherwise.
static double one_minus_j0(double x) {
  if (x < 1.0) {
    const double q = 0.25 * x * x;
    double term = 1.0, s = 0.0;
    for (int k = 1; k < 40; ++k) {
      term *= -q / ((double)k * k);
      s -= term;
      if (std::fabs(term) < 1e-18 * std::fabs(s)) break;
    }
    return s;
  }
  return 1.0 - ::j0(x);
}

// Scaling function of Eq. (scale_1p)/(G_kappa_k) at kappa^2, k3^2:
//   e^{-(1-eta)(kappa^2+k3^2)/4xi^2} Ghat(kappa, k3).
static double scaling(double kap2, double k3sq, double eta, double xi, double R) {
  const double damp = std::exp(-(1.0 - eta) * (kap2 + k3sq) / (4.0 * xi * xi));
  if (k3sq > 0.0) return damp / (kap2 + k3sq);
  if (kap2 == 0.0) return damp * R * R / 4.0 * (1.0 - 2.0 * std::log(R));     // Eq. (g_zeromod0)
  const double kap = std::sqrt(kap2);
  return damp * (one_minus_j0(R * kap) / kap2 - R * std::log(R) * ::j1(R * kap) / kap);  // Eq. (g_zeromod)
}

static std::vector<std::unique_ptr<KPlan>> g_plans;
static uint64_t g_plan_generation = 1;   // bumped whenever a plan is built or freed (graphs bake its pointers)

uint64_t kplan_generation() { return g_plan_generation; }

static KPlan* build(const KParams& p, cudaStream_t st) {
  auto t0 = std::chrono::steady_clock::now();
  auto pl = std::make_unique<KPlan>();
  pl->prm = p;
  KDev& dv = pl->dv;
  dv.M = p.M;
  dv.P = p.P;
  dv.h = p.L[2] / p.M;
  dv.inv_h = 1.0 / dv.h;
  dv.Mfree = (int)std::lround(p.L[0] / dv.h);
  dv.Mt = p.periodic ? dv.Mfree : dv.Mfree + p.P;   // SE3P transform plan: no free-axis extension
  dv.alpha = 2.0 * p.xi * p.xi / p.eta;
  dv.L3 = p.L[2];
  dv.nbx = (int)ceil_div(dv.Mfree, kBin);
  const int Mt = dv.Mt;
  pl->n_planes = p.M / 2 + 1;
  pl->n_kernel = std::max(0, std::min(p.n_l + 1, pl->n_planes));
  pl->LK = p.periodic ? p.SJ : next_friendly(2 * Mt - 1);

  std::vector<double2> tw;
  // (z-FFT: radix <= 5, its kernels run at 4 blocks per SM; the 2D passes: radix 8/9 at 3)
  if (!fft_make(p.M, pl->fz, tw, false) || !fft_make(p.SJ, pl->fJ, tw, true) || !fft_make(pl->LK, pl->fK, tw, true))
    throw Error{4, "FFT extent has a prime factor > 61"};
  // descriptor offsets (twoff/rootoff) index the combined table directly
  pl->twz = pl->twJ = pl->twK = 0;
  dev_alloc(pl->d_tw, tw.size());
  SE1P_CUDA_TRY(cudaMemcpy(pl->d_tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));

  const double h = dv.h, xi = p.xi, eta = p.eta, L3 = p.L[2];
  // gather constant (reading R-1): phi = 4 pi h^3 (2xi^2/(pi eta))^3 sum H'~ W, H' without prefactor
  const double pref = std::pow(2.0 * xi * xi / (kPi * eta), 1.5);
  pl->const_gather = 4.0 * kPi * h * h * h * pref * pref;
  const double R = std::sqrt(2.0) * Mt * h;  // reading R-6: sqrt(L~1^2 + L~2^2), square cross-section

  // J-plane tables
  {
    const int SJ = p.SJ;
    std::vector<double> ex(SJ), k2(SJ);
    for (int a = 0; a < SJ; ++a) {
      const int ap = (2 * a < SJ) ? a : a - SJ;
      const double kap = 2.0 * kPi * ap / (SJ * h);
      k2[a] = kap * kap;
      ex[a] = std::exp(-(1.0 - eta) * kap * kap / (4.0 * xi * xi));
    }
    std::vector<double2> plv(pl->n_planes);
    for (int n = 0; n < pl->n_planes; ++n) {
      const double k3 = 2.0 * kPi * n / L3;
      plv[n] = make_double2(pl->const_gather / ((double)p.M * (double)SJ * (double)SJ) *
                                std::exp(-(1.0 - eta) * k3 * k3 / (4.0 * xi * xi)),
                            k3 * k3);
    }
    dev_alloc(pl->d_exJ, SJ);
    dev_alloc(pl->d_k2J, SJ);
    dev_alloc(pl->d_pl, 2 * (size_t)pl->n_planes);   // (e^{...} C_J, k3^2) pairs
    SE1P_CUDA_TRY(cudaMemcpy(pl->d_exJ, ex.data(), sizeof(double) * SJ, cudaMemcpyHostToDevice));
    SE1P_CUDA_TRY(cudaMemcpy(pl->d_k2J, k2.data(), sizeof(double) * SJ, cudaMemcpyHostToDevice));
    SE1P_CUDA_TRY(cudaMemcpy(pl->d_pl, plv.data(), sizeof(double2) * pl->n_planes, cudaMemcpyHostToDevice));
  }

  // Fast Gaussian Gridding table f1[t] = e^{-alpha h^2 t^2}
  {
    std::vector<double> f1(p.P);
    for (int t = 0; t < p.P; ++t) f1[t] = std::exp(-dv.alpha * h * h * (double)t * (double)t);
    dev_alloc(pl->d_f1, p.P);
    SE1P_CUDA_TRY(cudaMemcpy(pl->d_f1, f1.data(), sizeof(double) * p.P, cudaMemcpyHostToDevice));
  }

  // kernel planes: k3 = 0 (extent S0) and 0 < k3 <= 2 pi n_l/L3 (extent SI)
  {
    const int LK = pl->LK;
    dev_alloc(pl->d_khat, (size_t)pl->n_kernel * LK * LK);
    const double scale = pl->const_gather / ((double)p.M * (double)LK * (double)LK);
    for (int n = 0; n < pl->n_kernel; ++n) {
      const int S = (n == 0) ? p.S0 : ((size_t)(n - 1) < p.SIn.size() ? p.SIn[n - 1] : p.SI);
      const int H = S / 2 + 1;
      const double k3 = 2.0 * kPi * n / L3;
      const double dk = 2.0 * kPi / (S * h);
      std::vector<double> sig((size_t)H * H);
      for (int m1 = 0; m1 < H; ++m1)
        for (int m2 = 0; m2 <= m1; ++m2) {
          const double kap2 = dk * dk * ((double)m1 * m1 + (double)m2 * m2);
          const double v = scaling(kap2, k3 * k3, eta, xi, R);
          sig[(size_t)m1 * H + m2] = v;
          sig[(size_t)m2 * H + m1] = v;
        }
      double* d_sig = nullptr;
      dev_alloc(d_sig, sig.size());
      SE1P_CUDA_TRY(cudaMemcpy(d_sig, sig.data(), sizeof(double) * sig.size(), cudaMemcpyHostToDevice));
      build_kernel_spectrum(*pl, S, d_sig, pl->d_khat + (size_t)n * LK * LK, scale, st);
      dev_free(d_sig);
    }
  }
  pl->t_off_total = (int64_t)pl->n_kernel * Mt * pl->LK + (int64_t)(pl->n_planes - pl->n_kernel) * Mt * p.SJ;
  pl->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  KPlan* raw = pl.get();
  g_plans.push_back(std::move(pl));
  return raw;
}

KPlan* kplan_get(const KParams& p0, cudaStream_t st) {
  KParams p = p0;
  SE1P_CUDA_TRY(cudaGetDevice(&p.device));   // tables live on one device: plans are per device
  for (auto& q : g_plans)
    if (q->prm == p) return q.get();
  ++g_plan_generation;
  if (g_plans.size() >= 16) {
    KPlan* old = g_plans.front().get();
    dev_free(old->d_tw);
    dev_free(old->d_khat);
    dev_free(old->d_exJ);
    dev_free(old->d_k2J);
    dev_free(old->d_pl);
    dev_free(old->d_f1);
    g_plans.erase(g_plans.begin());
  }
  return build(p, st);
}

void kplan_release_all(int device) {
  ++g_plan_generation;
  for (auto it = g_plans.begin(); it != g_plans.end();) {
    KPlan* q = it->get();
    if (q->prm.device != device) {
      ++it;
      continue;
    }
    dev_free(q->d_tw);
    dev_free(q->d_khat);
    dev_free(q->d_exJ);
    dev_free(q->d_k2J);
    dev_free(q->d_pl);
    dev_free(q->d_f1);
    it = g_plans.erase(it);
  }
}

}  // namespace se1p
