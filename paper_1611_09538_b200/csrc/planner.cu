// planner.cu -- parameters from an error tolerance, host code only.
//
// The paper's recipe (Sec. "Parameter selection") step by step:
//   rc    Eq. (rc)   P:138  rc = [3 W(4/3 C^{2/3})]^{1/2} / (2 xi),  C = Q / (2 V xi E^2)
//   kinf  Eq. (kinf) P:139  kinf = sqrt(3) L3 xi/(2 pi) [W(D/(xi E^2)^{2/3})]^{1/2},
//                           D = 4/(3 L3^2) (Q/pi)^{2/3}
//   M     = 2 kinf, rounded up to an even FFT-friendly count >= P with integer L1/h,
//         L2/h and eta <= 0.8
//   P     smallest even integer with A e^{-c^2 pi P/2} <= E, A = sqrt(Q xi L3)/L3 (Eq.
//         (approximation_error_oneterm); "set to even integers" P:690)
//   eta   Eq. (comp_eta), c = 0.95
//   s_l   e^{-2 pi s_l} < E (Eq. (choose_sl)) and the image-distance form of the same
//         estimate for non-cubic boxes (reading R-18), extent ceil(s_l M~)
//   n_l   M ~ 10 n_l (Eq. (choose_nl)): ceil(M/10)
//   s0    the minimal 1 + sqrt(2) of P:522 ("s0 ~ 2.4"), extent ceil(s0 M~)
//   Ntilde  >= M~, widened by the aliasing rule of reading R-8 (FFT-friendly).
// Budget (reading R-18): real space tol/2, k-space truncation and aliasing tol/10, window tol/100.
// Reading R-18: for a non-cubic box the estimates' L^3 is the volume L1 L2 L3 and
// their L the periodic length L3 (the k3 spacing 2 pi/L3 is what kinf counts).
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/se1p.h"
#include "fft.cuh"
#include "kspace.cuh"

namespace se1p {

// Principal branch W0(x), x >= 0: Halley iteration on w e^w = x from a log-based start.
double lambert_w0(double x) {
  if (x == 0.0) return 0.0;
  double w = x < 1.0 ? x * (1.0 - x) : std::log(x) - std::log(std::log(x) + 1.0);
  for (int it = 0; it < 100; ++it) {
    const double ew = std::exp(w);
    const double f = w * ew - x;
    const double wp1 = w + 1.0;
    const double dw = f / (ew * wp1 - (w + 2.0) * f / (2.0 * wp1));
    w -= dw;
    if (std::fabs(dw) <= 1e-16 * (1.0 + std::fabs(w))) break;
  }
  return w;
}

static bool friendly(int n) {
  std::vector<int> r;
  return fft_factor(n, r);
}

void plan_from_tol(const double L[3], double Q, double xi, double E, se1p_tol_plan* o) {
  if (!L || !o) throw Error{1, "null pointer"};
  if (!(L[0] > 0) || !(L[1] > 0) || !(L[2] > 0) || !(Q > 0) || !(xi > 0) || !(E > 0) || !(E < 1))
    throw Error{1, "L, Q, xi must be > 0 and 0 < tol < 1"};
  const double V = L[0] * L[1] * L[2], L3 = L[2], c = 0.95, Lsq = std::max(L[0], L[1]);
  *o = se1p_tol_plan{};
  o->xi = xi;
  o->tol = E;
  o->Q = Q;
  // error budget (reading R-18): the estimates are "~" for one error source each; the real-space
  // one is sharp (Fig. kolafa_perram) and gets half; the k-space truncation and aliasing sources
  // get a tenth each and the window (P) a hundredth -- measured on the Alg. 1 oracle, the literal
  // inversion misses the tolerance by up to 300x and this budget meets it (tests/test_planner.py).
  const double ER = 0.5 * E, EF = 0.1 * E, EP = 0.01 * E, eta_max = 0.8;
  const double C = Q / (2.0 * V * xi * ER * ER);
  o->rc = std::sqrt(3.0 * lambert_w0(4.0 / 3.0 * std::pow(C, 2.0 / 3.0))) / (2.0 * xi);
  const double D = 4.0 / (3.0 * L3 * L3) * std::pow(Q / kPi, 2.0 / 3.0);
  o->kinf = std::sqrt(3.0) * L3 * xi / (2.0 * kPi) * std::sqrt(lambert_w0(D / std::pow(xi * EF * EF, 2.0 / 3.0)));
  const double A = std::sqrt(Q * xi * L3) / L3;
  int P = 2;
  while (A * std::exp(-c * c * kPi * P / 2.0) > EP && P < 64) P += 2;
  // M: the smallest admissible even count >= 2 kinf at which eta <= 0.8 (eta < 1 so the scaling
  // e^{-(1-eta) k^2/4 xi^2} damps; the error grows as eta -> 1 at fixed P: reading R-18)
  int M = 2 * (int)std::ceil(o->kinf - 1e-12);
  for (;; M += 2) {
    if (M > 8192) throw Error{4, "no admissible M <= 8192 (L1/h and L2/h integers, eta < 1)"};
    const double m1 = Lsq * M / L3;   // the square domain the solve runs on (api.cu resolve)
    if (std::fabs(m1 - std::lround(m1)) > 1e-9 * m1) continue;
    if (!friendly(M) || M < P) continue;   // P <= M (Thm 1)
    const double hm = L3 / M;
    if (P * xi * xi * hm * hm / (c * c * kPi) <= eta_max) break;
  }
  o->M = M;
  o->h = L3 / M;
  o->Mfree = (int)std::lround(Lsq / o->h);
  o->P = P;
  o->Mt = o->Mfree + P;
  o->eta = P * xi * xi * o->h * o->h / (c * c * kPi);
  o->n_local = std::min(M / 2, std::max(1, (int)std::ceil(M / 10.0 - 1e-12)));
  // Upsampled and J planes: after the padded transform of length S h, mode k3 sees the periodic
  // images of the free-space solution at distance S h - L_free, which contribute ~ sqrt(Q)
  // e^{-|k3| (S h - L_free)} (the paper's e^{-2 pi |k3|/h_k} of Eq. (proof_I2d), with
  // h_k = 2 pi/(S h) and the charges' extent taken off; reading R-8 / R-18).  The slowest mode
  // of each set binds: k3 = 2 pi/L3 for the I planes, 2 pi (n_l+1)/L3 for the J planes.
  const double budget = std::max(0.0, std::log(std::sqrt(Q) / EF));
  const double dI = budget * L3 / (2.0 * kPi), dJ = dI / (o->n_local + 1);
  o->s_l = std::max({1.0, std::log(1.0 / EF) / (2.0 * kPi), (Lsq + dI) / (o->Mt * o->h)});   // (choose_sl) P:697
  o->SI = (int)std::ceil(o->s_l * o->Mt - 1e-9);
  o->s0 = 1.0 + std::sqrt(2.0);
  o->S0 = (int)std::ceil(o->s0 * o->Mt - 1e-9);
  o->Ntilde = next_friendly(std::max(o->Mt, (int)std::ceil((Lsq + dJ) / o->h - 1e-9)));
  o->est_real = std::sqrt(Q * o->rc / (2.0 * V)) / (xi * o->rc * xi * o->rc) * std::exp(-xi * xi * o->rc * o->rc);
  const double ki = M / 2.0;   // the grid resolves |k3| <= 2 pi (M/2)/L3
  o->est_fourier = xi / (kPi * kPi) * std::pow(ki, -1.5) * std::sqrt(Q) * std::exp(-std::pow(kPi * ki / (xi * L3), 2));
  o->est_approx = A * std::exp(-c * c * kPi * P / 2.0);
}

}  // namespace se1p
