// kplan.cu -- k-space plan: Alg. 1 step 1, FFT descriptors, scaling tables and
// the plan-time kernel spectra of the upsampled planes.
#include <chrono>
#include <cstdio>
#include <thread>
#include <cmath>
#include <memory>
#include <vector>

#include "kspace.cuh"

namespace se1p {

void build_kernel_spectrum(const KPlan& pl, int S, const double* d_sig, double* khat_out, double scale,
                           const KernScratch& ks, cudaStream_t st);

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

#ifndef SE1P_PLAN_TRACE
#define SE1P_PLAN_TRACE 0
#endif
static KPlan* build(const KParams& p, cudaStream_t st) {
  auto t0 = std::chrono::steady_clock::now();
  auto tr = [&](const char* what) {
    if (SE1P_PLAN_TRACE)
      fprintf(stderr, "plan %s %.1f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
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

  tr("twiddles");
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

  tr("tables");
  // kernel planes: k3 = 0 (extent S0) and 0 < k3 <= 2 pi n_l/L3 (extent SI)
  {
    const int LK = pl->LK;
    dev_alloc(pl->d_khat, (size_t)pl->n_kernel * LK * LK);
    const double scale = pl->const_gather / ((double)p.M * (double)LK * (double)LK);
    auto extent = [&](int n) { return (n == 0) ? p.S0 : ((size_t)(n - 1) < p.SIn.size() ? p.SIn[n - 1] : p.SI); };
    int Hmax = 1;
    for (int n = 0; n < pl->n_kernel; ++n) Hmax = std::max(Hmax, extent(n) / 2 + 1);
    // scratch allocated once; the host builds plane n + 1's table while the device transforms
    // plane n (stream order keeps the single table buffer safe)
    KernScratch ks{};
    double* d_sig = nullptr;
    if (pl->n_kernel > 0) {
      dev_alloc(d_sig, (size_t)Hmax * Hmax);
      dev_alloc(ks.tmp, (size_t)Mt * Hmax);
      dev_alloc(ks.A, (size_t)LK * LK);
      dev_alloc(ks.B, (size_t)LK * LK);
    }
    const int nth = std::max(1, std::min(16, (int)std::thread::hardware_concurrency()));
    std::vector<double> sig;
    for (int n = 0; n < pl->n_kernel; ++n) {
      const int S = extent(n);
      const int H = S / 2 + 1;
      const double k3 = 2.0 * kPi * n / L3;
      const double dk = 2.0 * kPi / (S * h);
      sig.assign((size_t)H * H, 0.0);
      // the (S/2+1)^2 table on the host's cores (rows interleaved over threads)
      std::vector<std::thread> pool;
      for (int th = 0; th < nth; ++th)
        pool.emplace_back([&, th]() {
          for (int m1 = th; m1 < H; m1 += nth)
            for (int m2 = 0; m2 <= m1; ++m2) {
              const double kap2 = dk * dk * ((double)m1 * m1 + (double)m2 * m2);
              const double v = scaling(kap2, k3 * k3, eta, xi, R);
              sig[(size_t)m1 * H + m2] = v;
              sig[(size_t)m2 * H + m1] = v;
            }
        });
      for (auto& t : pool) t.join();
      tr("sig");
      SE1P_CUDA_TRY(cudaMemcpyAsync(d_sig, sig.data(), sizeof(double) * sig.size(), cudaMemcpyHostToDevice, st));
      build_kernel_spectrum(*pl, S, d_sig, pl->d_khat + (size_t)n * LK * LK, scale, ks, st);
      tr("spectrum");
    }
    if (pl->n_kernel > 0) {
      SE1P_CUDA_TRY(cudaStreamSynchronize(st));
      dev_free(d_sig);
      dev_free(ks.tmp);
      dev_free(ks.A);
      dev_free(ks.B);
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
