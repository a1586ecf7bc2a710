/* ewald3p.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * The triply periodic Ewald sum, the baseline of SURVEY 8(f) NEXT-4 (the paper's Ex. 5, P:953-1006,
 * compares SE1P with SE3P of its reference [Lindbo2011]).  Plain definitions, fp64 with Neumaier
 * sums, O(m N) per term:
 *   phi(x_m) = phi^R + phi^F + phi^self, tin-foil boundary, neutral systems:
 *   phi^R    = sum_{p in Z^3} sum_n' q_n erfc(xi |x_m - x_n + p L|) / |x_m - x_n + p L|
 *   phi^F    = (4 pi / V) sum_{k != 0} e^{-k^2/4xi^2} / k^2 sum_n q_n cos(k . (x_m - x_n)),
 *              k = 2 pi (j1/L1, j2/L2, j3/L3)
 *   phi^self = -2 xi q_m / sqrt(pi)                         (as Eq. (6))
 * The same split as Eq. (2) with all three directions periodic. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define O3_PI 3.141592653589793238462643383279502884

typedef struct {
  double s, c;
} nsum3;
static inline void n3_add(nsum3* a, double v) {
  double t = a->s + v;
  if (fabs(a->s) >= fabs(v))
    a->c += (a->s - t) + v;
  else
    a->c += (v - t) + a->s;
  a->s = t;
}
static inline double n3_get(const nsum3* a) { return a->s + a->c; }

/* phi^R truncated at |r| <= rc, images p with |p_d| <= ceil(rc/L_d) + 1. */
void orc3_phi_real(const double* x, const double* q, int64_t N, const double* L, double xi, double rc,
                   const int64_t* targets, int64_t m, double* out) {
  int64_t A[3];
  for (int d = 0; d < 3; ++d) A[d] = (int64_t)ceil(rc / L[d]) + 1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum3 s = {0.0, 0.0};
    for (int64_t a = -A[0]; a <= A[0]; ++a)
      for (int64_t b = -A[1]; b <= A[1]; ++b)
        for (int64_t c = -A[2]; c <= A[2]; ++c)
          for (int64_t n = 0; n < N; ++n) {
            if (a == 0 && b == 0 && c == 0 && n == t) continue;
            const double dx = x[3 * t] - x[3 * n] + a * L[0];
            const double dy = x[3 * t + 1] - x[3 * n + 1] + b * L[1];
            const double dz = x[3 * t + 2] - x[3 * n + 2] + c * L[2];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            if (d <= rc) n3_add(&s, q[n] * erfc(xi * d) / d);
          }
    out[it] = n3_get(&s);
  }
}

/* phi^F over |j_d| <= K (all k != 0 in the box), structure factors computed once per k. */
void orc3_phi_kspace(const double* x, const double* q, int64_t N, const double* L, double xi, int K,
                     const int64_t* targets, int64_t m, double* out) {
  const int64_t nk = (int64_t)(2 * K + 1) * (2 * K + 1) * (2 * K + 1);
  double* Sc = (double*)calloc((size_t)nk, sizeof(double));
  double* Ss = (double*)calloc((size_t)nk, sizeof(double));
  double* wk = (double*)calloc((size_t)nk, sizeof(double));
  const double V = L[0] * L[1] * L[2];
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t id = 0; id < nk; ++id) {
    const int j1 = (int)(id / ((2 * K + 1) * (2 * K + 1))) - K;
    const int j2 = (int)((id / (2 * K + 1)) % (2 * K + 1)) - K;
    const int j3 = (int)(id % (2 * K + 1)) - K;
    if (j1 == 0 && j2 == 0 && j3 == 0) continue;
    const double k1 = 2.0 * O3_PI * j1 / L[0], k2 = 2.0 * O3_PI * j2 / L[1], k3 = 2.0 * O3_PI * j3 / L[2];
    const double kk = k1 * k1 + k2 * k2 + k3 * k3;
    wk[id] = 4.0 * O3_PI / V * exp(-kk / (4.0 * xi * xi)) / kk;
    nsum3 c = {0.0, 0.0}, s = {0.0, 0.0};
    for (int64_t n = 0; n < N; ++n) {
      const double ph = k1 * x[3 * n] + k2 * x[3 * n + 1] + k3 * x[3 * n + 2];
      n3_add(&c, q[n] * cos(ph));
      n3_add(&s, q[n] * sin(ph));
    }
    Sc[id] = n3_get(&c);
    Ss[id] = n3_get(&s);
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum3 s = {0.0, 0.0};
    for (int64_t id = 0; id < nk; ++id) {
      if (wk[id] == 0.0) continue;
      const int j1 = (int)(id / ((2 * K + 1) * (2 * K + 1))) - K;
      const int j2 = (int)((id / (2 * K + 1)) % (2 * K + 1)) - K;
      const int j3 = (int)(id % (2 * K + 1)) - K;
      const double ph = 2.0 * O3_PI * (j1 * x[3 * t] / L[0] + j2 * x[3 * t + 1] / L[1] + j3 * x[3 * t + 2] / L[2]);
      /* Re[e^{i k x_m} conj(S(k))], S(k) = sum_n q_n e^{i k x_n} */
      n3_add(&s, wk[id] * (cos(ph) * Sc[id] + sin(ph) * Ss[id]));
    }
    out[it] = n3_get(&s);
  }
  free(Sc);
  free(Ss);
  free(wk);
}

/* Converged parameters at the oracle's own xi: erfc(6.6) ~ 1e-20 in real space, and
   e^{-k^2/4xi^2} < 1e-20 at the shortest truncated wave vector in k space. */
double orc3_rc_converged(double xi) { return 6.6 / xi; }
int orc3_kmax_converged(double xi, const double* L) {
  double Lmax = L[0];
  if (L[1] > Lmax) Lmax = L[1];
  if (L[2] > Lmax) Lmax = L[2];
  return (int)ceil(2.0 * xi * 6.8 * Lmax / (2.0 * O3_PI)) + 1;
}

/* Total potential (tin-foil), converged, at xi_o (<= 0 -> 3.2 / min L). */
void orc3_phi_exact(const double* x, const double* q, int64_t N, const double* L, double xi_o,
                    const int64_t* targets, int64_t m, double* out) {
  double Lmin = L[0];
  if (L[1] < Lmin) Lmin = L[1];
  if (L[2] < Lmin) Lmin = L[2];
  if (!(xi_o > 0)) xi_o = 3.2 / Lmin;
  double* r = (double*)malloc(sizeof(double) * 2 * (size_t)m);
  orc3_phi_real(x, q, N, L, xi_o, orc3_rc_converged(xi_o), targets, m, r);
  orc3_phi_kspace(x, q, N, L, xi_o, orc3_kmax_converged(xi_o, L), targets, m, r + m);
  for (int64_t i = 0; i < m; ++i) {
    nsum3 s = {0.0, 0.0};
    n3_add(&s, r[i]);
    n3_add(&s, r[m + i]);
    n3_add(&s, -2.0 * xi_o * q[targets[i]] / sqrt(O3_PI));
    out[i] = n3_get(&s);
  }
  free(r);
}
