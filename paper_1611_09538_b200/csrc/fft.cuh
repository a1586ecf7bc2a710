// fft.cuh -- shared-memory mixed-radix Stockham FFT used by every transform of the SE1P
// path (the z-FFT of AFT step 1 and the per-k3 2D transforms of Alg. 2/3).
//
// One FFT length n = r_0 r_1 ... r_{S-1}; stage s (radix r, Ns = r_0...r_{s-1}) reads
// v_t = in[j + t n/r], multiplies by w^{t (j mod Ns)} with w = e^{-+2 pi i/(Ns r)}, does an
// r-point DFT and writes out[(j/Ns) Ns r + (j mod Ns) + q Ns] (Stockham autosort, natural
// order in and out).  Radices 8, 9, 4, 2, 3, 5 have dedicated butterflies; any other prime
// factor up to 61 uses an O(r^2) butterfly with a root table.  Twiddles are tabulated on
// the host in long double and rounded once.
#pragma once
#include <vector>

#include "common.cuh"

namespace se1p {

constexpr int kMaxStages = 16;
constexpr int kMaxGenericRadix = 61;

struct FftDesc {
  int n = 0;
  int nst = 0;
  int rad[kMaxStages];
  int twoff[kMaxStages];   // stage twiddles: tw[twoff + k (r-1) + t - 1] = e^{-2 pi i t k/(Ns r)}
  int rootoff[kMaxStages]; // generic radix roots: tw[rootoff + k] = e^{-2 pi i k / r}
  int total = 0;           // table length (complex entries)
};

// ------------------------------------------------------------------ butterflies
// DIR = -1: forward (e^{-i...}), DIR = +1: inverse (unnormalised).
template <int DIR>
__device__ __forceinline__ double2 mul_i_dir(double2 a) {  // a * (DIR * i)
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <int DIR>
__device__ __forceinline__ void bfly2(double2* v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <int DIR>
__device__ __forceinline__ void bfly4(double2* v) {
  double2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
  double2 c = cadd(v[1], v[3]), d = mul_i_dir<DIR>(csub(v[1], v[3]));
  v[0] = cadd(a, c);
  v[2] = csub(a, c);
  v[1] = cadd(b, d);
  v[3] = csub(b, d);
}

template <int DIR>
__device__ __forceinline__ void bfly3(double2* v) {
  const double s3 = 0.866025403784438646763723170752936183;  // sqrt(3)/2
  double2 s = cadd(v[1], v[2]);
  double2 t = make_double2(v[0].x - 0.5 * s.x, v[0].y - 0.5 * s.y);
  double2 d = mul_i_dir<DIR>(csub(v[1], v[2]));
  d.x *= s3;
  d.y *= s3;
  v[0] = cadd(v[0], s);
  v[1] = cadd(t, d);
  v[2] = csub(t, d);
}

template <int DIR>
__device__ __forceinline__ void bfly5(double2* v) {
  // X_q = sum_t v_t w^{qt}, w = e^{DIR 2 pi i/5}
  const double c1 = 0.309016994374947424102293417182819059;   // cos(2pi/5)
  const double c2 = -0.809016994374947424102293417182819059;  // cos(4pi/5)
  const double s1 = 0.951056516295153572116439333379382143;   // sin(2pi/5)
  const double s2 = 0.587785252292473129168705954639072769;   // sin(4pi/5)
  double2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
  double2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
  double2 r1 = make_double2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
  double2 r2 = make_double2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
  double2 i1 = make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
  double2 i2 = make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
  i1 = mul_i_dir<DIR>(i1);
  i2 = mul_i_dir<DIR>(i2);
  v[0] = make_double2(v[0].x + a1.x + a2.x, v[0].y + a1.y + a2.y);
  v[1] = cadd(r1, i1);
  v[4] = csub(r1, i1);
  v[2] = cadd(r2, i2);
  v[3] = csub(r2, i2);
}

// 8-point DFT as two 4-point DFTs (even / odd inputs) and a radix-2 combine with w8^q
template <int DIR>
__device__ __forceinline__ void bfly8(double2* v) {
  const double r = 0.707106781186547524400844362104849039;   // 1/sqrt(2)
  double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  bfly4<DIR>(e);
  bfly4<DIR>(o);
  // w8^1 = (r, DIR r), w8^2 = DIR i, w8^3 = (-r, DIR r)
  const double2 o1 = make_double2(r * (o[1].x - DIR * o[1].y), r * (o[1].y + DIR * o[1].x));
  const double2 o2 = mul_i_dir<DIR>(o[2]);
  const double2 o3 = make_double2(-r * (o[3].x + DIR * o[3].y), r * (DIR * o[3].x - o[3].y));
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

// 9-point DFT as 3 x 3: DFT3 over t1 of v[3 t1 + t2], twiddle w9^(t2 q1), DFT3 over t2 -> q1 + 3 q2
template <int DIR>
__device__ __forceinline__ void bfly9(double2* v) {
  const double c1 = 0.766044443118978035202392650555416673;   // cos(2pi/9)
  const double s1 = 0.642787609686539326322643409907263432;   // sin(2pi/9)
  const double c2 = 0.173648177666930348851716626769314796;   // cos(4pi/9)
  const double s2 = 0.984807753012208059366743024589523014;   // sin(4pi/9)
  const double c4 = -0.939692620785908384054109277324731470;  // cos(8pi/9)
  const double s4 = 0.342020143325668733044099614682259581;   // sin(8pi/9)
  double2 y[3][3];
#pragma unroll
  for (int t2 = 0; t2 < 3; ++t2) {
    double2 a[3] = {v[t2], v[3 + t2], v[6 + t2]};
    bfly3<DIR>(a);
    y[t2][0] = a[0];
    y[t2][1] = a[1];
    y[t2][2] = a[2];
  }
  // w9^k = (cos, DIR sin)
  y[1][1] = cmul(y[1][1], make_double2(c1, DIR * s1));
  y[1][2] = cmul(y[1][2], make_double2(c2, DIR * s2));
  y[2][1] = cmul(y[2][1], make_double2(c2, DIR * s2));
  y[2][2] = cmul(y[2][2], make_double2(c4, DIR * s4));
#pragma unroll
  for (int q1 = 0; q1 < 3; ++q1) {
    double2 a[3] = {y[0][q1], y[1][q1], y[2][q1]};
    bfly3<DIR>(a);
    v[q1] = a[0];
    v[q1 + 3] = a[1];
    v[q1 + 6] = a[2];
  }
}

// ------------------------------------------------------------------ one stage
// Butterfly j (0 <= j < n/R) of row `row`: inputs j + t n/R, twiddle index k = j mod Ns, outputs
// (j / Ns) Ns R + k + q Ns.  Threads own a fixed j across rows (when n/R <= nthr) so the index
// arithmetic and the twiddle loads happen once per stage, not once per butterfly.
template <int R, int DIR>
__device__ __forceinline__ void bfly_fixed(double2* v) {
  if (R == 2) bfly2<DIR>(v);
  if (R == 3) bfly3<DIR>(v);
  if (R == 4) bfly4<DIR>(v);
  if (R == 5) bfly5<DIR>(v);
  if (R == 8) bfly8<DIR>(v);
  if (R == 9) bfly9<DIR>(v);
}

template <int R, int DIR>
__device__ __forceinline__ void stage_fixed(const double2* __restrict__ in, double2* __restrict__ out,
                                            int n, int Ns, const double2* __restrict__ tw, int nrows,
                                            int rowstride, int tid, int nthr) {
  const int nb = n / R;
  int j, row0, rstep, jstep;
  if (nb <= nthr) {
    rstep = nthr / nb;
    if (tid >= rstep * nb) return;
    j = tid % nb;
    row0 = tid / nb;
    jstep = nb;   // one j per thread
  } else {
    rstep = 1;
    j = tid;
    row0 = 0;
    jstep = nthr;
  }
  for (; j < nb; j += jstep) {
    const int k = j % Ns;
    double2 w[R];
#pragma unroll
    for (int t = 1; t < R; ++t) w[t] = (k > 0) ? tw[k * (R - 1) + t - 1] : make_double2(1.0, 0.0);
    const int obase = (j / Ns) * Ns * R + k;
    for (int row = row0; row < nrows; row += rstep) {
      const double2* src = in + row * rowstride + j;
      double2 v[R];
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = src[t * nb];
      if (k > 0) {
#pragma unroll
        for (int t = 1; t < R; ++t) v[t] = DIR < 0 ? cmul(v[t], w[t]) : cmulc(v[t], w[t]);
      }
      bfly_fixed<R, DIR>(v);
      double2* dst = out + row * rowstride + obase;
#pragma unroll
      for (int q = 0; q < R; ++q) dst[q * Ns] = v[q];
    }
  }
}

template <int DIR>
__device__ void stage_generic(const double2* __restrict__ in, double2* __restrict__ out, int n, int R,
                              int Ns, const double2* __restrict__ tw, const double2* __restrict__ roots,
                              int nrows, int rowstride, int tid, int nthr) {
  const int nb = n / R;
  int j, row0, rstep, jstep;
  if (nb <= nthr) {
    rstep = nthr / nb;
    if (tid >= rstep * nb) return;
    j = tid % nb;
    row0 = tid / nb;
    jstep = nb;
  } else {
    rstep = 1;
    j = tid;
    row0 = 0;
    jstep = nthr;
  }
  for (; j < nb; j += jstep) {
    const int k = j % Ns;
    const int obase = (j / Ns) * Ns * R + k;
    for (int row = row0; row < nrows; row += rstep) {
      const double2* src = in + row * rowstride + j;
      double2 v[kMaxGenericRadix];
      for (int t = 0; t < R; ++t) {
        double2 x = src[t * nb];
        if (k > 0 && t > 0) {
          double2 w = tw[k * (R - 1) + t - 1];
          x = DIR < 0 ? cmul(x, w) : cmulc(x, w);
        }
        v[t] = x;
      }
      double2* dst = out + row * rowstride + obase;
      for (int q = 0; q < R; ++q) {
        double2 acc = v[0];
        int e = 0;
        for (int t = 1; t < R; ++t) {
          e += q;
          if (e >= R) e -= R;
          double2 w = roots[e];
          acc = cadd(acc, DIR < 0 ? cmul(v[t], w) : cmulc(v[t], w));
        }
        dst[q * Ns] = acc;
      }
    }
  }
}

// Batched FFT of `nrows` rows (row r at buf[r*rowstride], length d.n) held in shared memory.
// Uses `buf` and `tmp` as ping-pong buffers; returns the buffer holding the result.
// Must be called by all `nthr` threads of the block (contains __syncthreads).
template <int DIR>
__device__ double2* fft_rows(double2* buf, double2* tmp, const FftDesc& d, const double2* __restrict__ tw,
                             int nrows, int rowstride, int tid, int nthr) {
  double2* in = buf;
  double2* out = tmp;
  int Ns = 1;
  for (int s = 0; s < d.nst; ++s) {
    const int R = d.rad[s];
    const double2* tws = tw + d.twoff[s];
    switch (R) {
      case 2: stage_fixed<2, DIR>(in, out, d.n, Ns, tws, nrows, rowstride, tid, nthr); break;
      case 3: stage_fixed<3, DIR>(in, out, d.n, Ns, tws, nrows, rowstride, tid, nthr); break;
      case 4: stage_fixed<4, DIR>(in, out, d.n, Ns, tws, nrows, rowstride, tid, nthr); break;
      case 5: stage_fixed<5, DIR>(in, out, d.n, Ns, tws, nrows, rowstride, tid, nthr); break;
      case 8: stage_fixed<8, DIR>(in, out, d.n, Ns, tws, nrows, rowstride, tid, nthr); break;
      case 9: stage_fixed<9, DIR>(in, out, d.n, Ns, tws, nrows, rowstride, tid, nthr); break;
      default:
        stage_generic<DIR>(in, out, d.n, R, Ns, tws, tw + d.rootoff[s], nrows, rowstride, tid, nthr);
    }
    __syncthreads();
    double2* t = in;
    in = out;
    out = t;
    Ns *= R;
  }
  return in;
}

// ------------------------------------------------------------------ compile-time plans
// The same Stockham stages with the length, the rows per block and every stage's radix and
// stride known at compile time (index splits by constants, no radix switch, no per-stage
// branches): used where a plan's extents match one of the instantiated shapes (modes.cu).
template <int R, int DIR, int N, int NS, int NROWS>
__device__ __forceinline__ void stage_ct(const double2* __restrict__ in, double2* __restrict__ out,
                                         const double2* __restrict__ tw, int rowstride, int tid, int nthr) {
  constexpr int NB = N / R;
  for (int t = tid; t < NB * NROWS; t += nthr) {
    const int row = t / NB, j = t - row * NB;
    const int k = j % NS;
    const double2* src = in + row * rowstride + j;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = src[q * NB];
    if (NS > 1 && k > 0) {
#pragma unroll
      for (int q = 1; q < R; ++q) {
        const double2 w = tw[k * (R - 1) + q - 1];
        v[q] = DIR < 0 ? cmul(v[q], w) : cmulc(v[q], w);
      }
    }
    bfly_fixed<R, DIR>(v);
    double2* dst = out + row * rowstride + (j / NS) * NS * R + k;
#pragma unroll
    for (int q = 0; q < R; ++q) dst[q * NS] = v[q];
  }
}

template <int DIR, int N, int NROWS, int NS, int R, int... Rest>
__device__ __forceinline__ double2* fft_ct(double2* in, double2* out, const FftDesc& d, const double2* __restrict__ tw,
                                           int s, int rowstride, int tid, int nthr) {
  stage_ct<R, DIR, N, NS, NROWS>(in, out, tw + d.twoff[s], rowstride, tid, nthr);
  __syncthreads();
  if constexpr (sizeof...(Rest) == 0) {
    return out;
  } else {
    return fft_ct<DIR, N, NROWS, NS * R, Rest...>(out, in, d, tw, s + 1, rowstride, tid, nthr);
  }
}

// plan shapes with compile-time kernels (0: the generic fft_rows)
constexpr int kPlanGeneric = 0, kPlan320 = 1, kPlan576 = 2, kPlan256 = 3;
inline int fft_plan_shape(const FftDesc& d) {
  if (d.n == 256 && d.nst == 4 && d.rad[0] == 4 && d.rad[1] == 4 && d.rad[2] == 4 && d.rad[3] == 4) return kPlan256;
  if (d.n == 320 && d.nst == 3 && d.rad[0] == 5 && d.rad[1] == 8 && d.rad[2] == 8) return kPlan320;
  if (d.n == 576 && d.nst == 3 && d.rad[0] == 9 && d.rad[1] == 8 && d.rad[2] == 8) return kPlan576;
  return kPlanGeneric;
}

// rows of a block through the compile-time plan SHAPE (NROWS rows) or the generic one
template <int DIR, int SHAPE, int NROWS>
__device__ __forceinline__ double2* fft_rows_sh(double2* buf, double2* tmp, const FftDesc& d,
                                                const double2* __restrict__ tw, int nrows, int rowstride, int tid,
                                                int nthr) {
  if constexpr (SHAPE == kPlan320) {
    return fft_ct<DIR, 320, NROWS, 1, 5, 8, 8>(buf, tmp, d, tw, 0, rowstride, tid, nthr);
  } else if constexpr (SHAPE == kPlan576) {
    return fft_ct<DIR, 576, NROWS, 1, 9, 8, 8>(buf, tmp, d, tw, 0, rowstride, tid, nthr);
  } else if constexpr (SHAPE == kPlan256) {
    return fft_ct<DIR, 256, NROWS, 1, 4, 4, 4, 4>(buf, tmp, d, tw, 0, rowstride, tid, nthr);
  } else {
    return fft_rows<DIR>(buf, tmp, d, tw, nrows, rowstride, tid, nthr);
  }
}

// ------------------------------------------------------------------ host side
// Factorise n into stage radices: odd ones first (9 if r8, 3, 5), then 8 (if r8), 4, 2, then any
// other prime.  Returns false if a prime factor exceeds kMaxGenericRadix or there are too many
// stages.
bool fft_factor(int n, std::vector<int>& rad, bool r8 = false);
// Build the descriptor and append its twiddle/root table to `table` (host), setting offsets.
// r8: radix-8/9 stages (fewer shared-memory passes, more registers per butterfly).
bool fft_make(int n, FftDesc& d, std::vector<double2>& table, bool r8);
// "FFT-friendly": only factors 2, 3, 5.
bool fft_friendly(int n);
int next_friendly(int n);

}  // namespace se1p
