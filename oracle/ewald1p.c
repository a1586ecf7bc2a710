/*
 * oracle/ewald1p.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU evaluation of the singly periodic Ewald sum (Ewald1P) of
 * Saffar Shamshirgar & Tornberg, "The Spectral Ewald method for singly periodic
 * domains" (arXiv:1611.09538).  Citations "P:n" are lines of PAPER.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code with the CUDA path
 * (paper_1611_09538_b200/) and the CUDA path never calls it.
 *
 * What is computed (Eq. (2) `eq:full_potential`):
 *   phi(x_m) = phi^R + phi^{F,k3!=0} + phi^{F,k3=0} + phi^self
 *   phi^R         Eq. (3)  P:86   sum_alpha' sum_n q_n erfc(xi d)/d,  d=|x_m-x_n+alpha L3 e3|
 *   phi^{F,k3!=0} Eq. (4b) P:88   (1/L3) sum_{k3!=0} sum_n q_n e^{i k3 dz} K0(k3^2/4xi^2, rho^2 xi^2)
 *   phi^{F,k3=0}  Eq. (5)  P:89   -(1/L3) sum_{n!=m} q_n {gamma + log(xi^2 rho^2) + E1(xi^2 rho^2)}
 *   phi^self      Eq. (6)  P:90   -2 xi q_m / sqrt(pi)
 * plus the definition itself, Eq. (1) with P_1, as a brute-force image sum.
 *
 * Special functions follow Appendix A:
 *   K0(a,b) incomplete Bessel: Gauss-Legendre on [0,v] u [v,1]
 *   E1(x): continued fraction for x >= 1, series for x < 1
 *   gamma + log x + E1(x) via the series without cancellation for x < 1
 *   k0(x) (complete modified Bessel function of the second kind, "besselk"):
 *         trapezoidal rule on K0(x) = int_0^inf exp(-x cosh t) dt (textbook integral form;
 *         the paper delegates k0 to a library, reading R-11).
 * All sums over sources use Neumaier compensated summation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_GAMMA 0.577215664901532860606512090082402431
#define ORC_PI 3.14159265358979323846264338327950288

/* ---------------------------------------------------------------- summation */
typedef struct { double s, c; } nsum;
static inline void nsum_add(nsum* a, double v) {
  double t = a->s + v;
  if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
  else a->c += (v - t) + a->s;
  a->s = t;
}
static inline double nsum_get(const nsum* a) { return a->s + a->c; }

/* Work split for the source sums: target it, sources [n0, n1) of block bk.  Large systems use a
   fixed number of source blocks (independent of the thread count) with one compensated partial
   each, combined in block order -- deterministic, and every core busy for any number of targets;
   small systems (N < 65536, every test size) use one block, i.e. the plain per-target sum. */
static int64_t orc_src_blocks(int64_t N) { return N < 65536 ? 1 : 64; }
static double orc_combine(const nsum* part, int64_t nb) {
  if (nb == 1) return nsum_get(&part[0]);
  nsum t = {0.0, 0.0};
  for (int64_t b = 0; b < nb; ++b) {
    nsum_add(&t, part[b].s);
    nsum_add(&t, part[b].c);
  }
  return nsum_get(&t);
}
#ifdef _OPENMP
#include <omp.h>
int orc_threads(void) { return omp_get_max_threads(); }
#else
int orc_threads(void) { return 1; }
#endif

/* ---------------------------------------------------------------- E1, g */
/* App. A uses the series for 0<x<1 and the continued fraction for "x >~ 1".  The
   series loses ~e^x/E1(x) * eps to cancellation above ~1.5, so the switch is at x = 1.5
   (reading R-12). */
#define ORC_E1_SWITCH 1.5
/* E1(x) = int_1^inf e^{-xt}/t dt.  x < 1.5: series; otherwise the continued
   fraction with n = 1. */
double orc_e1(double x) {
  if (!(x > 0.0)) return NAN;
  if (x < ORC_E1_SWITCH) {
    /* E1(x) = -gamma - log x - sum_{m>=1} (-1)^m x^m / (m! m) */
    double term = 1.0, s = 0.0;
    for (int m = 1; m < 400; ++m) {
      term *= -x / m;            /* (-x)^m / m! */
      double t = term / m;
      s += t;
      if (fabs(t) < 1e-19 * fabs(s)) break;
    }
    return -ORC_GAMMA - log(x) - s;
  }
  if (x > 745.0) return 0.0;
  /* e^{-x} ( 1/(x+1-) 1^2/(x+3-) 2^2/(x+5-) ... ), evaluated from the tail (depth 120 converges
     to < 3e-16 relative for x >= 1.5; backward evaluation avoids the Lentz rounding drift). */
  double f = 0.0;
  for (int i = 120; i >= 1; --i) f = -((double)i * (double)i) / (x + 2.0 * i + 1.0 + f);
  return exp(-x) / (x + 1.0 + f);
}

/* g(u) = gamma + log u + E1(u), with g(0) = 0.  For u < 1 the series
   g(u) = -sum_{m>=1} (-u)^m/(m m!) (rearranged P:1108) has no cancellation. */
double orc_g(double u) {
  if (u <= 0.0) return 0.0;
  if (u < ORC_E1_SWITCH) {
    double term = 1.0, s = 0.0;
    for (int m = 1; m < 400; ++m) {
      term *= -u / m;
      double t = term / m;
      s += t;
      if (fabs(t) < 1e-19 * fabs(s)) break;
    }
    return -s;
  }
  return ORC_GAMMA + log(u) + orc_e1(u);
}

/* ---------------------------------------------------------------- k0 */
/* K_0(x) = int_0^inf exp(-x cosh t) dt.  The integrand is even and entire in t, so the
   trapezoidal rule with step dt converges geometrically; dt = 1/32 is far past 1e-16. */
double orc_k0(double x) {
  if (!(x > 0.0)) return NAN;
  /* K_0(x) = e^{-x} int_0^inf exp(-2x sinh^2(t/2)) dt: the factor e^{-x} is pulled out so the
     exponent stays small near the peak (relative accuracy does not degrade like x eps). */
  const double dt = fmin(1.0 / 32.0, 0.25 / sqrt(x));
  nsum s = {0.5, 0.0};
  for (int k = 1; k < 1000000; ++k) {
    double sh = sinh(0.5 * k * dt);
    double v = exp(-2.0 * x * sh * sh);
    nsum_add(&s, v);
    if (v < 1e-22 * nsum_get(&s)) break;
  }
  return exp(-x) * dt * nsum_get(&s);
}

/* ---------------------------------------------------------------- Gauss-Legendre */
#define ORC_GL_N 32
static double gl_x[ORC_GL_N], gl_w[ORC_GL_N];
static int gl_ready = 0;

/* Nodes/weights on [-1,1]: Newton iteration on P_n via the three-term recurrence. */
static void gl_init(void) {
  const int n = ORC_GL_N;
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = cos(ORC_PI * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (fabs(z - z1) < 1e-16) break;
    }
    gl_x[i] = -z;
    gl_x[n - 1 - i] = z;
    gl_w[i] = gl_w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
  gl_ready = 1;
}

void orc_gauss_legendre(int which, double* x_out, double* w_out) {
  (void)which;
  if (!gl_ready) gl_init();
  memcpy(x_out, gl_x, sizeof gl_x);
  memcpy(w_out, gl_w, sizeof gl_w);
}

/* int_lo^hi e^{-a/t - b t} dt/t by ORC_GL_N-point Gauss-Legendre. */
static double k0_piece(double a, double b, double lo, double hi) {
  if (hi <= lo) return 0.0;
  double half = 0.5 * (hi - lo), mid = 0.5 * (hi + lo);
  nsum s = {0.0, 0.0};
  for (int i = 0; i < ORC_GL_N; ++i) {
    double t = mid + half * gl_x[i];
    nsum_add(&s, gl_w[i] * exp(-a / t - b * t) / t);
  }
  return half * nsum_get(&s);
}

/* Incomplete Bessel K0(a,b) = int_1^inf e^{-at-b/t} dt/t = int_0^1 e^{-a/t-bt} dt/t.
   App. A: for a > b integrate over [0,v] u [v,1] with v = min(sqrt(b),1);
   for a < b use K0(a,b) = 2 k0(2 sqrt(ab)) - K0(b,a), integrating K0(b,a) over [0,v] u [v,1]
   with v = min(b sqrt(b/a), 1).  Each piece is further halved geometrically towards t=0
   (reading R-10) so the e^{-a/t} boundary layer is resolved for any a. */
static double k0_split(double a, double b, double v) {
  /* [v,1] plus [0,v] subdivided as [v/2^(k+1), v/2^k]; the integrand peaks at
     t* = (sqrt(1+4ab)-1)/(2b) (-> a as b -> 0) and the pieces below t* decay like e^{-a/t},
     so the subdivision stops once it is below t* and a piece no longer registers. */
  double s = 0.0;
  /* [v,1] as [v 2^k, v 2^(k+1)] so every piece has endpoint ratio <= 2 (the integrand has
     an essential singularity at t=0 which limits Gauss-Legendre on a long [v,1]) */
  for (double lo = v; lo < 1.0;) {
    double hi = fmin(2.0 * lo, 1.0);
    s += k0_piece(a, b, lo, hi);
    lo = hi;
  }
  const double tstar = (b > 0.0) ? 2.0 * a / (sqrt(1.0 + 4.0 * a * b) + 1.0) : a;
  double hi = v;
  for (int k = 0; k < 2000 && hi > 1e-300; ++k) {
    double lo = 0.5 * hi;
    double piece = k0_piece(a, b, lo, hi);
    s += piece;
    if (hi < tstar && piece <= 1e-21 * fabs(s)) break;
    if (a / hi > 800.0) break;       /* e^{-a/t} < e^{-800} below this point */
    hi = lo;
  }
  return s;
}

double orc_K0inc(double a, double b) {
  if (!gl_ready) gl_init();
  if (!(a > 0.0) || b < 0.0) return NAN;
  if (b == 0.0) return orc_e1(a);               /* K0(a,0) = E1(a) */
  if (a >= b) {
    double v = fmin(sqrt(b), 1.0);
    return k0_split(a, b, v);
  }
  double v = fmin(b * sqrt(b / a), 1.0);
  return 2.0 * orc_k0(2.0 * sqrt(a * b)) - k0_split(b, a, v);
}

/* dK0(a,b)/db = -int_0^1 e^{-a/s - b s} ds (differentiating P:95 under the integral after
   s = 1/t).  The integrand is analytic on (0,1] with a boundary layer e^{-a/s} at 0 and its
   peak at s* = sqrt(a/b); [0,1] is cut into pieces with endpoint ratio <= 2 around s*, each by
   ORC_GL_N-point Gauss-Legendre (the construction of DESIGN.md reading R-10). */
static double kd_piece(double a, double b, double lo, double hi) {
  if (hi <= lo) return 0.0;
  double half = 0.5 * (hi - lo), mid = 0.5 * (hi + lo);
  nsum s = {0.0, 0.0};
  for (int i = 0; i < ORC_GL_N; ++i) {
    double t = mid + half * gl_x[i];
    nsum_add(&s, gl_w[i] * exp(-a / t - b * t));
  }
  return half * nsum_get(&s);
}

double orc_dK0db(double a, double b) {
  if (!gl_ready) gl_init();
  if (!(a > 0.0) || b < 0.0) return NAN;
  const double sstar = (b > 0.0) ? fmin(sqrt(a / b), 1.0) : 1.0;
  double s = 0.0;
  for (double lo = sstar; lo < 1.0;) {   /* [s*, 1] in doubling pieces */
    double hi = fmin(2.0 * lo, 1.0);
    s += kd_piece(a, b, lo, hi);
    lo = hi;
  }
  double hi = sstar;                     /* [0, s*] in halving pieces */
  for (int k = 0; k < 2000 && hi > 1e-300; ++k) {
    double lo = 0.5 * hi;
    double piece = kd_piece(a, b, lo, hi);
    s += piece;
    if (piece <= 1e-21 * fabs(s) || a / hi > 800.0) break;
    hi = lo;
  }
  return -s;
}

/* ---------------------------------------------------------------- the sums */
/* P_1 images: p = (0, 0, alpha L3).  Targets are indices into the same particle set
   (target points = charge locations, Alg. 1 step 6 P:270). */

/* phi^R at (xi, rc): Eq. (3), truncated at d <= rc.  All images alpha with
   |alpha| <= ceil(rc/L3)+1 are scanned, which contains every image within rc. */
void orc_phi_real(const double* x, const double* q, int64_t N, const double* L, double xi,
                  double rc, const int64_t* targets, int64_t m, double* out) {
  const double L3 = L[2];
  const int64_t A = (int64_t)ceil(rc / L3) + 1, NB = orc_src_blocks(N);
  nsum* part = (nsum*)malloc(sizeof(nsum) * (size_t)(m * NB));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < m * NB; ++k) {
    const int64_t it = k / NB, bk = k % NB, n0 = N * bk / NB, n1 = N * (bk + 1) / NB;
    const int64_t t = targets[it];
    nsum s = {0.0, 0.0};
    for (int64_t alpha = -A; alpha <= A; ++alpha) {
      for (int64_t n = n0; n < n1; ++n) {
        if (alpha == 0 && n == t) continue;          /* the prime in Eq. (3) */
        double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
        double dz = x[3 * t + 2] - x[3 * n + 2] + alpha * L3;
        double d = sqrt(dx * dx + dy * dy + dz * dz);
        if (d <= rc) nsum_add(&s, q[n] * erfc(xi * d) / d);
      }
    }
    part[k] = s;
  }
  for (int64_t it = 0; it < m; ++it) out[it] = orc_combine(part + it * NB, NB);
  free(part);
}

/* phi^{F,k3!=0}: Eq. (4b) P:88 with the +k3 and -k3 terms folded into 2cos(k3 dz).
   k3 = 2 pi j / L3, j = 1..J.  n = m is included (rho = 0 -> K0(a,0) = E1(a)). */
void orc_phi_k3nz(const double* x, const double* q, int64_t N, const double* L, double xi,
                  int J, const int64_t* targets, int64_t m, double* out) {
  if (!gl_ready) gl_init();
  const double L3 = L[2];
  const int64_t NB = orc_src_blocks(N);
  nsum* part = (nsum*)malloc(sizeof(nsum) * (size_t)(m * NB));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < m * NB; ++k) {
    const int64_t it = k / NB, bk = k % NB, n0 = N * bk / NB, n1 = N * (bk + 1) / NB;
    const int64_t t = targets[it];
    nsum s = {0.0, 0.0};
    for (int j = 1; j <= J; ++j) {
      const double k3 = 2.0 * ORC_PI * j / L3;
      const double a = k3 * k3 / (4.0 * xi * xi);
      for (int64_t n = n0; n < n1; ++n) {
        double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
        double dz = x[3 * t + 2] - x[3 * n + 2];
        double rho2 = dx * dx + dy * dy;
        nsum_add(&s, q[n] * 2.0 * cos(k3 * dz) * orc_K0inc(a, rho2 * xi * xi));
      }
    }
    part[k] = s;
  }
  for (int64_t it = 0; it < m; ++it) out[it] = orc_combine(part + it * NB, NB) / L3;
  free(part);
}

/* phi^{F,k3=0}: Eq. (5); the n = m term is excluded. */
void orc_phi_k30(const double* x, const double* q, int64_t N, const double* L, double xi,
                 const int64_t* targets, int64_t m, double* out) {
  const double L3 = L[2];
  const int64_t NB = orc_src_blocks(N);
  nsum* part = (nsum*)malloc(sizeof(nsum) * (size_t)(m * NB));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < m * NB; ++k) {
    const int64_t it = k / NB, bk = k % NB, n0 = N * bk / NB, n1 = N * (bk + 1) / NB;
    const int64_t t = targets[it];
    nsum s = {0.0, 0.0};
    for (int64_t n = n0; n < n1; ++n) {
      if (n == t) continue;
      double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
      nsum_add(&s, q[n] * orc_g(xi * xi * (dx * dx + dy * dy)));
    }
    part[k] = s;
  }
  for (int64_t it = 0; it < m; ++it) out[it] = -orc_combine(part + it * NB, NB) / L3;
  free(part);
}

/* phi^self: Eq. (6) P:90. */
void orc_phi_self(const double* q, double xi, const int64_t* targets, int64_t m, double* out) {
  for (int64_t it = 0; it < m; ++it) out[it] = -2.0 * xi * q[targets[it]] / sqrt(ORC_PI);
}

/* Number of k3 modes so that every omitted term is below E1(a_J) <= e^{-a}/a < 1e-21:
   a_J = (pi J/(xi L3))^2 >= 48. */
int orc_modes_needed(double xi, double L3) {
  return (int)ceil(sqrt(48.0) * xi * L3 / ORC_PI);
}

/* Converged cutoff for phi^R: erfc(xi rc)/rc with xi rc = 6.6 gives erfc < 1e-20. */
double orc_rc_converged(double xi) { return 6.6 / xi; }

/* Full potential phi = Eq. (2), evaluated at the oracle's own Ewald parameter xi_o with
   both sums converged (the total does not depend on xi).  xi_o <= 0 picks
   xi_o = 0.7/L3 (reading R-9: fewest K0 modes for few images).  comps (optional, 4*m) receives
   the four terms per target: R, k3!=0, k3=0, self. */
void orc_phi_exact(const double* x, const double* q, int64_t N, const double* L, double xi_o,
                   const int64_t* targets, int64_t m, double* out, double* comps) {
  if (xi_o <= 0.0) xi_o = 0.7 / L[2];
  double* r = (double*)malloc(sizeof(double) * 4 * (size_t)m);
  orc_phi_real(x, q, N, L, xi_o, orc_rc_converged(xi_o), targets, m, r);
  orc_phi_k3nz(x, q, N, L, xi_o, orc_modes_needed(xi_o, L[2]), targets, m, r + m);
  orc_phi_k30(x, q, N, L, xi_o, targets, m, r + 2 * m);
  orc_phi_self(q, xi_o, targets, m, r + 3 * m);
  for (int64_t i = 0; i < m; ++i) {
    nsum s = {0.0, 0.0};
    for (int c = 0; c < 4; ++c) nsum_add(&s, r[c * m + i]);
    out[i] = nsum_get(&s);
    if (comps)
      for (int c = 0; c < 4; ++c) comps[4 * i + c] = r[c * m + i];
  }
  free(r);
}

/* The definition, Eq. (1) with P_1: symmetric truncation |alpha| <= A.
   Under neutrality the truncation error is O(A^-2); callers extrapolate in A. */
void orc_phi_brute(const double* x, const double* q, int64_t N, const double* L, int64_t A,
                   const int64_t* targets, int64_t m, double* out) {
  const double L3 = L[2];
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum s = {0.0, 0.0};
    for (int64_t n = 0; n < N; ++n) {
      double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
      double dz0 = x[3 * t + 2] - x[3 * n + 2];
      double rho2 = dx * dx + dy * dy;
      nsum sn = {0.0, 0.0};
      /* sum pairs alpha, -alpha from the outside in, so small terms are added first */
      for (int64_t alpha = A; alpha >= 1; --alpha) {
        double zp = dz0 + alpha * L3, zm = dz0 - alpha * L3;
        nsum_add(&sn, 1.0 / sqrt(rho2 + zp * zp) + 1.0 / sqrt(rho2 + zm * zm));
      }
      if (n != t) nsum_add(&sn, 1.0 / sqrt(rho2 + dz0 * dz0));
      nsum_add(&s, q[n] * nsum_get(&sn));
    }
    out[it] = nsum_get(&s);
  }
}


/* ---------------------------------------------------------------- fields (forces) */
/* Electric field E = -grad phi at the target, the target's own charge excluded exactly as in
   the potential (the force on particle m is q_m E(x_m), P:535-551 -- written here as the
   gradients of Eqs. (3)-(5), not copied).  out[3*it + c], c = x, y, z. */

/* E^R: -grad of q_n erfc(xi d)/d = q_n (erfc(xi d)/d + 2 xi/sqrt(pi) e^{-xi^2 d^2}) r/d^2, d <= rc. */
void orc_field_real(const double* x, const double* q, int64_t N, const double* L, double xi,
                    double rc, const int64_t* targets, int64_t m, double* out) {
  const double L3 = L[2];
  const int64_t A = (int64_t)ceil(rc / L3) + 1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum s[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int64_t alpha = -A; alpha <= A; ++alpha) {
      for (int64_t n = 0; n < N; ++n) {
        if (alpha == 0 && n == t) continue;
        double r[3] = {x[3 * t] - x[3 * n], x[3 * t + 1] - x[3 * n + 1], x[3 * t + 2] - x[3 * n + 2] + alpha * L3};
        double d2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2], d = sqrt(d2);
        if (d > rc) continue;
        double f = q[n] * (erfc(xi * d) / d + 2.0 * xi / sqrt(ORC_PI) * exp(-xi * xi * d2)) / d2;
        for (int c = 0; c < 3; ++c) nsum_add(&s[c], f * r[c]);
      }
    }
    for (int c = 0; c < 3; ++c) out[3 * it + c] = nsum_get(&s[c]);
  }
}

/* E^{F,k3!=0} from Eq. (4b): phi = (2/L3) sum_j sum_n q_n cos(k dz) K0(a_j, xi^2 rho^2):
   E_z = (2/L3) sum q_n k sin(k dz) K0,  E_r = -(2/L3) sum q_n cos(k dz) dK0/db 2 xi^2 (r_m - r_n). */
void orc_field_k3nz(const double* x, const double* q, int64_t N, const double* L, double xi,
                    int J, const int64_t* targets, int64_t m, double* out) {
  if (!gl_ready) gl_init();
  const double L3 = L[2];
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum s[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int j = 1; j <= J; ++j) {
      const double k3 = 2.0 * ORC_PI * j / L3;
      const double a = k3 * k3 / (4.0 * xi * xi);
      for (int64_t n = 0; n < N; ++n) {
        double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
        double dz = x[3 * t + 2] - x[3 * n + 2];
        double b = xi * xi * (dx * dx + dy * dy);
        nsum_add(&s[2], q[n] * 2.0 * k3 * sin(k3 * dz) * orc_K0inc(a, b));
        if (b > 0.0) {
          double g = -q[n] * 2.0 * cos(k3 * dz) * orc_dK0db(a, b) * 2.0 * xi * xi;
          nsum_add(&s[0], g * dx);
          nsum_add(&s[1], g * dy);
        }
      }
    }
    for (int c = 0; c < 3; ++c) out[3 * it + c] = nsum_get(&s[c]) / L3;
  }
}

/* E^{F,k3=0} from Eq. (5): phi = -(1/L3) sum_{n!=m} q_n g(xi^2 rho^2), g'(u) = (1 - e^{-u})/u:
   E_r = (1/L3) sum q_n g'(u) 2 xi^2 (r_m - r_n), E_z = 0. */
void orc_field_k30(const double* x, const double* q, int64_t N, const double* L, double xi,
                   const int64_t* targets, int64_t m, double* out) {
  const double L3 = L[2];
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum s[2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int64_t n = 0; n < N; ++n) {
      if (n == t) continue;
      double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
      double u = xi * xi * (dx * dx + dy * dy);
      double gp = (u < 1e-8) ? 1.0 - 0.5 * u : -expm1(-u) / u;
      double f = q[n] * gp * 2.0 * xi * xi;
      nsum_add(&s[0], f * dx);
      nsum_add(&s[1], f * dy);
    }
    out[3 * it] = nsum_get(&s[0]) / L3;
    out[3 * it + 1] = nsum_get(&s[1]) / L3;
    out[3 * it + 2] = 0.0;
  }
}

/* Full field at the oracle's xi_o, converged (independent of xi_o like the potential).
   comps (optional, 9*m): R, k3!=0, k3=0 (3 components each). */
void orc_field_exact(const double* x, const double* q, int64_t N, const double* L, double xi_o,
                     const int64_t* targets, int64_t m, double* out, double* comps) {
  if (xi_o <= 0.0) xi_o = 0.7 / L[2];
  double* r = (double*)malloc(sizeof(double) * 9 * (size_t)m);
  orc_field_real(x, q, N, L, xi_o, orc_rc_converged(xi_o), targets, m, r);
  orc_field_k3nz(x, q, N, L, xi_o, orc_modes_needed(xi_o, L[2]), targets, m, r + 3 * m);
  orc_field_k30(x, q, N, L, xi_o, targets, m, r + 6 * m);
  for (int64_t i = 0; i < m; ++i)
    for (int c = 0; c < 3; ++c) {
      nsum s = {0.0, 0.0};
      for (int k = 0; k < 3; ++k) nsum_add(&s, r[k * 3 * m + 3 * i + c]);
      out[3 * i + c] = nsum_get(&s);
      if (comps)
        for (int k = 0; k < 3; ++k) comps[9 * i + 3 * k + c] = r[k * 3 * m + 3 * i + c];
    }
  free(r);
}

/* The definition: E = sum_alpha sum'_n q_n r / |r|^3, r = x_m - x_n - alpha L3 e3, |alpha| <= A
   (symmetric; callers extrapolate in A). */
void orc_field_brute(const double* x, const double* q, int64_t N, const double* L, int64_t A,
                     const int64_t* targets, int64_t m, double* out) {
  const double L3 = L[2];
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t it = 0; it < m; ++it) {
    const int64_t t = targets[it];
    nsum s[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int64_t n = 0; n < N; ++n) {
      double dx = x[3 * t] - x[3 * n], dy = x[3 * t + 1] - x[3 * n + 1];
      double dz0 = x[3 * t + 2] - x[3 * n + 2];
      double rho2 = dx * dx + dy * dy;
      nsum sn[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int64_t alpha = A; alpha >= -A; --alpha) {
        if (alpha == 0 && n == t) continue;
        double dz = dz0 + alpha * L3;
        double d2 = rho2 + dz * dz, inv3 = 1.0 / (d2 * sqrt(d2));
        nsum_add(&sn[0], dx * inv3);
        nsum_add(&sn[1], dy * inv3);
        nsum_add(&sn[2], dz * inv3);
      }
      for (int c = 0; c < 3; ++c) nsum_add(&s[c], q[n] * nsum_get(&sn[c]));
    }
    for (int c = 0; c < 3; ++c) out[3 * it + c] = nsum_get(&s[c]);
  }
}
