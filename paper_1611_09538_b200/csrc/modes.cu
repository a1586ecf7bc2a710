// modes.cu -- the adaptive FFT of Alg. 2, the scaling of Alg. 1 step 4 and the inverse
// adaptive FFT of Alg. 3, for the k3 >= 0 half of the modes.
//
// Layout:
//   grid   [Mt][Mt][M]     real, z fastest           (H after gridding, H~ before gather)
//   planes [M/2+1][Mt][Mt] complex, one plane per k3 (only the M~ x M~ content is stored;
//                                                     padding to S is virtual)
//   T      per plane [Mt][W] complex, W = LK (kernel planes) or SJ (J planes)
//
// Passes:  zfwd -> rowfwd -> colpass(FFT, multiply, IFFT) -> rowinv -> zinv.
// J planes (s = 1): W = SJ and the multiplier is Eq. (scale_1p) sampled at kappa = 2 pi a'/(SJ h).
// Kernel planes (k3 = 0 and the I modes): W = LK >= 2 M~ - 1 and the multiplier is the
// plan-time spectrum of the exact aperiodic kernel equivalent to the paper's padded
// transform of extent S.  All normalisations (1/M, 1/W^2) and the
// gather constant are folded into the multipliers.
#include <algorithm>
#include <type_traits>

#include "kspace.cuh"

namespace se1p {

static int zcols(int M) { return M >= 256 ? 16 : (M >= 64 ? 32 : 64); }   // columns (2 per FFT)
// shared-memory budget of a row-pass block and columns per column-pass block (build knobs, see
// tools/exp_variant.sh)
#ifndef SE1P_ROW_SMEM
#define SE1P_ROW_SMEM 49152   // measured: 96 KB -> 48 KB is -7% (C5) / -8% (C4) on the mode stage
#endif
#ifndef SE1P_COLS_SMALL
#define SE1P_COLS_SMALL 8
#endif
#ifndef SE1P_COLS_LARGE
#define SE1P_COLS_LARGE 4
#endif
#ifndef SE1P_MODES_TWO_STREAMS
#define SE1P_MODES_TWO_STREAMS 2   // 1: kernel planes beside J planes; 2: and the J planes in two halves
#endif
#ifndef SE1P_FFT_CT   // compile-time FFT plans for the shapes fft_plan_shape knows (0: generic only)
#define SE1P_FFT_CT 1
#endif
#ifndef SE1P_MODES_JSPLIT
#define SE1P_MODES_JSPLIT 2
#endif
#ifndef SE1P_FFT_THREADS
#define SE1P_FFT_THREADS 256
#endif
// persistent column passes: columns per item (3 slots per CTA)
#ifndef SE1P_PCOLS_SMALL
#define SE1P_PCOLS_SMALL 4
#endif
#ifndef SE1P_PCOLS_LARGE
#define SE1P_PCOLS_LARGE 2
#endif
static int rows_for(int W) { int r = SE1P_ROW_SMEM / (2 * W * 16); return r < 1 ? 1 : (r > 16 ? 16 : r); }
static int cols_for(int W) { return W > 400 ? SE1P_COLS_LARGE : SE1P_COLS_SMALL; }
constexpr int kFftThreads = SE1P_FFT_THREADS;   // threads per block of the FFT passes
constexpr int kColMaxThreads = 384;             // column pass: block size chosen per plan (col_threads)
// blocks per SM the register allocation targets: z passes (radix <= 5) and 2D passes (radix 8/9)
#ifndef SE1P_FFT_MINB_Z
#define SE1P_FFT_MINB_Z 4
#endif
#ifndef SE1P_FFT_MINB_2D
#define SE1P_FFT_MINB_2D 3
#endif
#define SE1P_FFT_LBZ __launch_bounds__(SE1P_FFT_THREADS, SE1P_FFT_MINB_Z)
#define SE1P_FFT_LB __launch_bounds__(SE1P_FFT_THREADS, SE1P_FFT_MINB_2D)

// Global -> shared copies with U independent loads in flight per thread (a plain strided loop
// waits out one load latency per element): st(i, ld(i)) for i in [0, n).
template <int U, class T, class LD, class ST>
__device__ __forceinline__ void copy_batched(int n, int tid, int nthr, LD ld, ST st) {
  for (int b = tid; b < n; b += U * nthr) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + u * nthr;
      if (i < n) v[u] = ld(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + u * nthr;
      if (i < n) st(i, v[u]);
    }
  }
}
#ifndef SE1P_LDU
#define SE1P_LDU 8
#endif
constexpr int kLdU = SE1P_LDU;

// ------------------------------------------------------------------ z-FFT (AFT step 1)
// Rows x = L.xlo[0] .. L.xlo[L.nslab]-1 of the grid; plane n goes to slot slot_of[n] (identity if
// null) of the plane buffer in layout L (kspace.cuh, slab_row).
// Two real z columns per complex FFT (columns 2r and 2r+1 of the block as z_r = col_2r + i col_2r+1):
// their spectra separate as A[n] = (Z[n] + conj Z[M-n])/2, B[n] = (Z[n] - conj Z[M-n])/(2i).
// CB (columns per block) is a template constant and M's log2 (or -1) is passed, so the index
// splits below are shifts, not integer divisions by runtime values.
template <int CB, int SHAPE = kPlanGeneric>
__global__ void SE1P_FFT_LBZ k_zfwd(int Mt, int M, int mshift, int nplanes, FftDesc fz, const double2* __restrict__ tw,
                       const double* __restrict__ grid, double2* __restrict__ planes, SlabLayout L,
                       const int* __restrict__ slot_of) {
  extern __shared__ double2 sm[];
  const int S = M + 1;   // padded row stride: the transposed accesses below stay conflict-free
  constexpr int CH = CB / 2;
  double2* buf = sm;
  double2* tmp = sm + CH * S;
  const int x = L.xlo[0] + blockIdx.y, y0 = blockIdx.x * CB;
  const double* src = grid + ((int64_t)x * Mt + y0) * M;
  double* bd = reinterpret_cast<double*>(buf);
  const int ncol = min(CB, Mt - y0);
  copy_batched<kLdU, double>(
      CB * M, threadIdx.x, blockDim.x,
      [&](int idx) {
        const int c = mshift >= 0 ? idx >> mshift : idx / M;
        return c < ncol ? __ldg(src + idx) : 0.0;
      },
      [&](int idx, double v) {
        const int c = mshift >= 0 ? idx >> mshift : idx / M, k = idx - c * M;
        bd[2 * ((c >> 1) * S + k) + (c & 1)] = v;
      });
  __syncthreads();
  double2* out = fft_rows_sh<-1, SHAPE, CH>(buf, tmp, fz, tw, CH, S, threadIdx.x, blockDim.x);
  for (int idx = threadIdx.x; idx < nplanes * CB; idx += blockDim.x) {
    const int n = idx / CB, c = idx - n * CB;
    if (y0 + c < Mt) {
      const double2 Z = out[(c >> 1) * S + n], Zm = out[(c >> 1) * S + (n ? M - n : 0)];
      const double2 v = (c & 1) ? make_double2(0.5 * (Z.y + Zm.y), 0.5 * (Zm.x - Z.x))    // (Z - conj Zm)/(2i)
                                : make_double2(0.5 * (Z.x + Zm.x), 0.5 * (Z.y - Zm.y));   // (Z + conj Zm)/2
      planes[slab_row(L, slot_of ? slot_of[n] : n, x, Mt) + y0 + c] = v;
    }
  }
}

// Inverse: the Hermitian spectra a, b of columns 2r, 2r+1 combine into W[n] = a[n] + i b[n],
// W[M-n] = conj a[n] + i conj b[n]; the complex inverse FFT gives col_2r + i col_2r+1.
template <int CB, int SHAPE = kPlanGeneric>
__global__ void SE1P_FFT_LBZ k_zinv(int Mt, int M, int mshift, int nplanes, FftDesc fz, const double2* __restrict__ tw,
                       const double2* __restrict__ planes, double* __restrict__ grid, SlabLayout L,
                       const int* __restrict__ slot_of) {
  extern __shared__ double2 sm[];
  const int S = M + 1;   // padded row stride (conflict-free transposed accesses)
  constexpr int CH = CB / 2;
  double2* buf = sm;
  double2* tmp = sm + CH * S;
  const int x = L.xlo[0] + blockIdx.y, y0 = blockIdx.x * CB;
  copy_batched<4, double4>(
      nplanes * CH, threadIdx.x, blockDim.x,
      [&](int idx) {
        const int n = idx / CH, r = idx - n * CH;
        const int64_t row = slab_row(L, slot_of ? slot_of[n] : n, x, Mt) + y0 + 2 * r;
        const double2 a = (y0 + 2 * r < Mt) ? planes[row] : make_double2(0.0, 0.0);
        const double2 b = (y0 + 2 * r + 1 < Mt) ? planes[row + 1] : make_double2(0.0, 0.0);
        return make_double4(a.x, a.y, b.x, b.y);
      },
      [&](int idx, double4 ab) {
        const int n = idx / CH, r = idx - n * CH;
        buf[r * S + n] = make_double2(ab.x - ab.w, ab.y + ab.z);
        if (n > 0 && 2 * n < M) buf[r * S + (M - n)] = make_double2(ab.x + ab.w, ab.z - ab.y);   // Hermitian half
      });
  __syncthreads();
  double2* out = fft_rows_sh<1, SHAPE, CH>(buf, tmp, fz, tw, CH, S, threadIdx.x, blockDim.x);
  double* dst = grid + ((int64_t)x * Mt + y0) * M;
  for (int idx = threadIdx.x; idx < CB * M; idx += blockDim.x) {
    const int c = mshift >= 0 ? idx >> mshift : idx / M, k = idx - c * M;
    if (y0 + c < Mt) {
      const double2 v = out[(c >> 1) * S + k];
      dst[idx] = (c & 1) ? v.y : v.x;
    }
  }
}

// ------------------------------------------------------------------ 2D passes
// Launched plane blockIdx.y is global plane gl[by] (nfirst + by if null) held in slot li[by]
// (= its global index if null) of the plane buffer in layout L.
struct PlaneSel {
  const int* gl;
  const int* li;
  int nfirst;
  __device__ __forceinline__ int global(int by) const { return gl ? gl[by] : nfirst + by; }
  __device__ __forceinline__ int slot(int by) const { return li ? li[by] : global(by); }
};

__global__ void SE1P_FFT_LB k_rowfwd(int Mt, int W, int64_t base, int RB, FftDesc f, const double2* __restrict__ tw,
                         const double2* __restrict__ planes, double2* __restrict__ T, SlabLayout L, PlaneSel S) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* tmp = sm + RB * W;
  const int i = S.slot(blockIdx.y), x0 = blockIdx.x * RB;
  const int nr = min(RB, Mt - x0);
  copy_batched<kLdU, double2>(
      RB * W, threadIdx.x, blockDim.x,
      [&](int idx) {
        const int r = idx / W, y = idx - r * W;
        return (r < nr && y < Mt) ? planes[slab_row(L, i, x0 + r, Mt) + y] : make_double2(0.0, 0.0);
      },
      [&](int idx, double2 v) { buf[idx] = v; });
  __syncthreads();
  double2* out = fft_rows<-1>(buf, tmp, f, tw, RB, W, threadIdx.x, blockDim.x);
  double2* dst = T + base + (int64_t)blockIdx.y * Mt * W + (int64_t)x0 * W;
  for (int idx = threadIdx.x; idx < nr * W; idx += blockDim.x) dst[idx] = out[idx];
}

__global__ void SE1P_FFT_LB k_rowinv(int Mt, int W, int64_t base, int RB, FftDesc f, const double2* __restrict__ tw,
                         const double2* __restrict__ T, double2* __restrict__ planes, SlabLayout L, PlaneSel S) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* tmp = sm + RB * W;
  const int i = S.slot(blockIdx.y), x0 = blockIdx.x * RB;
  const int nr = min(RB, Mt - x0);
  const double2* src = T + base + (int64_t)blockIdx.y * Mt * W + (int64_t)x0 * W;
  copy_batched<kLdU, double2>(
      RB * W, threadIdx.x, blockDim.x, [&](int idx) { return idx < nr * W ? src[idx] : make_double2(0.0, 0.0); },
      [&](int idx, double2 v) { buf[idx] = v; });
  __syncthreads();
  double2* out = fft_rows<1>(buf, tmp, f, tw, RB, W, threadIdx.x, blockDim.x);
  for (int r = 0; r < nr; ++r) {
    double2* dst = planes + slab_row(L, i, x0 + r, Mt);
    for (int y = threadIdx.x; y < Mt; y += blockDim.x) dst[y] = out[r * W + y];
  }
}

// 1/d for d > 0 (normal): the hardware approximation refined by two Newton steps (relative error
// ~2^-23 -> 2^-46 -> below 1 ulp), a fraction of the cost of an IEEE division
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// Column pass: FFT along x, multiply, inverse FFT along x, keep rows < Mt.
// kernel_class: multiplier = khat[n][a][y] (n < n_kernel); else the J-plane scaling of plane n.
template <int CB, int SHAPE>
__global__ void __launch_bounds__(kColMaxThreads, 2) k_colpass(int Mt, int W, int64_t base, FftDesc f, const double2* __restrict__ tw,
                          double2* __restrict__ T, int kernel_class, const double* __restrict__ khat,
                          const double* __restrict__ exJ, const double* __restrict__ k2J,
                          const double2* __restrict__ pl, PlaneSel S) {
  extern __shared__ double2 sm[];
  const int SW = W + 1;   // padded row stride: the transposed accesses stay conflict-free
  double2* buf = sm;
  double2* tmp = sm + CB * SW;
  double* mul = reinterpret_cast<double*>(sm + 2 * CB * SW);   // kernel class: khat columns [CB][W]
  const int n = S.global(blockIdx.y), y0 = blockIdx.x * CB;
  const int nc = min(CB, W - y0);
  double2* Tp = T + base + (int64_t)blockIdx.y * Mt * W;
  copy_batched<kLdU, double2>(
      CB * W, threadIdx.x, blockDim.x,
      [&](int idx) {
        const int a = idx / CB, c = idx - a * CB;
        return (a < Mt && c < nc) ? Tp[(int64_t)a * W + y0 + c] : make_double2(0.0, 0.0);
      },
      [&](int idx, double2 v) {
        const int a = idx / CB, c = idx - a * CB;
        buf[c * SW + a] = v;
      });
  if (kernel_class)   // khat[n][a][y0 + c], issued before the FFT so its latency overlaps it
    copy_batched<kLdU, double>(
        CB * W, threadIdx.x, blockDim.x,
        [&](int idx) {
          const int a = idx / CB, c = idx - a * CB;
          return __ldg(khat + ((int64_t)n * W + a) * W + min(y0 + c, W - 1));
        },
        [&](int idx, double v) {
          const int a = idx / CB, c = idx - a * CB;
          mul[c * W + a] = v;
        });
  __syncthreads();
#ifndef SE1P_COLPASS_EXP   // experiment builds: 1 no FFTs, 2 no multiply, 3 neither
#define SE1P_COLPASS_EXP 0
#endif
  double2* out = (SE1P_COLPASS_EXP & 1) ? buf : fft_rows_sh<-1, SHAPE, CB>(buf, tmp, f, tw, CB, SW, threadIdx.x, blockDim.x);
  double2* oth = (out == buf) ? tmp : buf;
  const double2 pn = pl[n];
  // flat loop over the CB x W entries with the (c, a) split carried incrementally (no division)
  int c = threadIdx.x / W, a = threadIdx.x - c * W;
  const int dc = blockDim.x / W, da = blockDim.x - dc * W;
  for (; c < CB && !(SE1P_COLPASS_EXP & 2);) {
    const int y = min(y0 + c, W - 1);
    double m;
    if (kernel_class) {
      m = mul[c * W + a];
    } else {
      const double den = k2J[a] + k2J[y] + pn.y;   // 0 only at k = 0 of an SE3P plan: mode dropped
      m = den > 0.0 ? pn.x * exJ[a] * exJ[y] * rcp_nr(den) : 0.0;
    }
    double2 v = out[c * SW + a];
    out[c * SW + a] = make_double2(v.x * m, v.y * m);
    c += dc;
    a += da;
    if (a >= W) {
      a -= W;
      ++c;
    }
  }
  __syncthreads();
  double2* res = (SE1P_COLPASS_EXP & 1) ? out : fft_rows_sh<1, SHAPE, CB>(out, oth, f, tw, CB, SW, threadIdx.x, blockDim.x);
  for (int idx = threadIdx.x; idx < Mt * CB; idx += blockDim.x) {
    const int a = idx / CB, c = idx - a * CB;
    if (c < nc) Tp[(int64_t)a * W + y0 + c] = res[c * SW + a];
  }
}

static void set_smem(const void* fn, size_t bytes) {
  SE1P_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

static int log2_or_neg(int n) {
  int s = 0;
  while ((1 << s) < n) ++s;
  return (1 << s) == n ? s : -1;
}

// ------------------------------------------------------------------ persistent passes
// The FFT passes above load a block's data, transform it and store it in sequence, so every
// block waits out a full global-memory latency with nothing else to do (a variant with the
// transforms removed keeps 2/3 of the mode stage's time).  The persistent form runs
// ~blocks-per-SM x 148 CTAs that walk the pass's items, and prefetches item i + grid into a third
// shared buffer with cp.async (SASS LDGSTS; zero-fill for padding) while item i is transformed in
// the other two.  Each pass supplies load (async copies into a slot), compute (returns the
// buffer holding the result; may use both buffers) and store.
// SE1P_PERSIST bits: 1 z-FFT, 2 inverse z-FFT, 4 row passes, 8 column passes.  Measured at C5:
// rows 87 -> 78 us and inverse z 167 -> 158 us persistent (per launch, generic plans); the column
// passes lose (their slot budget halves the columns per item: 133 -> 170 us); the z-FFT is even
// with the generic plan and gains with the compile-time one (stage 0.163 -> 0.149 ms).
#ifndef SE1P_PERSIST
#define SE1P_PERSIST 7
#endif
__device__ __forceinline__ unsigned sm_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sm_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sm_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <class PassT, int MINB>
__global__ void __launch_bounds__(SE1P_FFT_THREADS, MINB) k_persist(const PassT P) {
  extern __shared__ double2 sm[];
  double2* B[3] = {sm, sm + P.slot, sm + 2 * P.slot};
  int d = 0, p = 1;
  const int x = 2;
  int it = blockIdx.x;
  if (it < P.n_items) P.load(it, B[d]);
  cp_async_commit();
  for (; it < P.n_items; it += gridDim.x) {
    const int nx = it + gridDim.x;
    if (nx < P.n_items) P.load(nx, B[p]);
    cp_async_commit();
    cp_async_wait1();   // every group but the newest: item it has landed (this thread's copies)
    __syncthreads();    // (and every thread's)
    const double2* res = P.compute(it, B[d], B[x]);
    P.store(it, res);
    __syncthreads();    // result read out before its buffers take the next prefetch
    const int t = d;
    d = p;
    p = t;
  }
}

// rows of a plane: item = (plane by, row group); planes -> FFT along y -> T
template <int SHAPE, int NR>   // compile-time plan and rows per item (generic: RB at run time)
struct RowFwdPass {
  int n_items, slot, nxb, Mt, W, RB;
  int64_t base;
  FftDesc f;
  const double2* tw;
  const double2* planes;
  double2* T;
  SlabLayout L;
  PlaneSel S;
  __device__ void load(int it, double2* dst) const {
    const int by = it / nxb, x0 = (it - by * nxb) * RB, i = S.slot(by), nr = min(RB, Mt - x0);
    for (int r = 0; r < RB; ++r) {
      const double2* src = planes + (r < nr ? slab_row(L, i, x0 + r, Mt) : 0);
      for (int y = threadIdx.x; y < W; y += blockDim.x) {
        const bool v = r < nr && y < Mt;
        cp_async16(dst + r * W + y, v ? src + y : planes, v);
      }
    }
  }
  __device__ const double2* compute(int, double2* b, double2* t) const {
    return fft_rows_sh<-1, SHAPE, NR>(b, t, f, tw, RB, W, threadIdx.x, blockDim.x);
  }
  __device__ void store(int it, const double2* res) const {
    const int by = it / nxb, x0 = (it - by * nxb) * RB, nr = min(RB, Mt - x0);
    double2* dst = T + base + (int64_t)by * Mt * W + (int64_t)x0 * W;
    for (int idx = threadIdx.x; idx < nr * W; idx += blockDim.x) dst[idx] = res[idx];
  }
};

// inverse rows: T -> inverse FFT along y -> planes (y < Mt)
template <int SHAPE, int NR>
struct RowInvPass {
  int n_items, slot, nxb, Mt, W, RB;
  int64_t base;
  FftDesc f;
  const double2* tw;
  const double2* T;
  double2* planes;
  SlabLayout L;
  PlaneSel S;
  __device__ void load(int it, double2* dst) const {
    const int by = it / nxb, x0 = (it - by * nxb) * RB, nr = min(RB, Mt - x0);
    const double2* src = T + base + (int64_t)by * Mt * W + (int64_t)x0 * W;
    for (int idx = threadIdx.x; idx < RB * W; idx += blockDim.x) {
      const bool v = idx < nr * W;
      cp_async16(dst + idx, v ? src + idx : T, v);
    }
  }
  __device__ const double2* compute(int, double2* b, double2* t) const {
    return fft_rows_sh<1, SHAPE, NR>(b, t, f, tw, RB, W, threadIdx.x, blockDim.x);
  }
  __device__ void store(int it, const double2* res) const {
    const int by = it / nxb, x0 = (it - by * nxb) * RB, i = S.slot(by), nr = min(RB, Mt - x0);
    for (int r = 0; r < nr; ++r) {
      double2* dst = planes + slab_row(L, i, x0 + r, Mt);
      for (int y = threadIdx.x; y < Mt; y += blockDim.x) dst[y] = res[r * W + y];
    }
  }
};

// columns: item = (plane by, column block of CB); FFT along x, multiply, inverse FFT; the kernel
// class's multiplier columns khat[n][a][y] ride in the slot behind the data
template <int CB>
struct ColPass {
  int n_items, slot, ncb, Mt, W, kernel_class;
  int64_t base;
  FftDesc f;
  const double2* tw;
  double2* T;
  const double* khat;
  const double* exJ;
  const double* k2J;
  const double2* pl;
  PlaneSel S;
  __device__ void load(int it, double2* dst) const {
    const int by = it / ncb, y0 = (it - by * ncb) * CB, nc = min(CB, W - y0), SW = W + 1, n = S.global(by);
    const double2* Tp = T + base + (int64_t)by * Mt * W;
    for (int idx = threadIdx.x; idx < CB * W; idx += blockDim.x) {
      const int a = idx / CB, c = idx - a * CB;
      const bool v = a < Mt && c < nc;
      cp_async16(dst + c * SW + a, v ? Tp + (int64_t)a * W + y0 + c : Tp, v);
    }
    if (kernel_class) {
      double* mul = reinterpret_cast<double*>(dst + CB * SW);
      for (int idx = threadIdx.x; idx < CB * W; idx += blockDim.x) {
        const int a = idx / CB, c = idx - a * CB;
        cp_async8(mul + c * W + a, khat + ((int64_t)n * W + a) * W + min(y0 + c, W - 1), true);
      }
    }
  }
  __device__ const double2* compute(int it, double2* b, double2* t) const {
    const int by = it / ncb, y0 = (it - by * ncb) * CB, SW = W + 1, n = S.global(by);
    const double* mul = reinterpret_cast<const double*>(b + CB * SW);
    double2* out = fft_rows<-1>(b, t, f, tw, CB, SW, threadIdx.x, blockDim.x);
    double2* oth = (out == b) ? t : b;
    const double2 pn = pl[n];
    for (int idx = threadIdx.x; idx < CB * W; idx += blockDim.x) {
      const int c = idx / W, a = idx - c * W;
      double m;
      if (kernel_class) {
        m = mul[c * W + a];
      } else {
        const int y = min(y0 + c, W - 1);
        const double den = k2J[a] + k2J[y] + pn.y;   // 0 only at k = 0 of an SE3P plan: mode dropped
        m = den > 0.0 ? pn.x * exJ[a] * exJ[y] * rcp_nr(den) : 0.0;
      }
      const double2 v = out[c * SW + a];
      out[c * SW + a] = make_double2(v.x * m, v.y * m);
    }
    __syncthreads();
    return fft_rows<1>(out, oth, f, tw, CB, SW, threadIdx.x, blockDim.x);
  }
  __device__ void store(int it, const double2* res) const {
    const int by = it / ncb, y0 = (it - by * ncb) * CB, nc = min(CB, W - y0), SW = W + 1;
    double2* Tp = T + base + (int64_t)by * Mt * W;
    for (int idx = threadIdx.x; idx < Mt * CB; idx += blockDim.x) {
      const int a = idx / CB, c = idx - a * CB;
      if (c < nc) Tp[(int64_t)a * W + y0 + c] = res[c * SW + a];
    }
  }
};

// z-FFT: item = (grid row x, column block of CB); two real columns per complex FFT (see k_zfwd)
template <int CB, int SHAPE = kPlanGeneric>
struct ZfwdPass {
  int n_items, slot, ncb, Mt, M, mshift, nplanes;
  FftDesc f;
  const double2* tw;
  const double* grid;
  double2* planes;
  SlabLayout L;
  const int* slot_of;
  __device__ void load(int it, double2* dst) const {
    const int xr = it / ncb, x = L.xlo[0] + xr, y0 = (it - xr * ncb) * CB, ncol = min(CB, Mt - y0), S = M + 1;
    const double* src = grid + ((int64_t)x * Mt + y0) * M;
    double* bd = reinterpret_cast<double*>(dst);
    for (int idx = threadIdx.x; idx < CB * M; idx += blockDim.x) {
      const int c = mshift >= 0 ? idx >> mshift : idx / M, k = idx - c * M;
      const bool v = c < ncol;
      cp_async8(bd + 2 * ((c >> 1) * S + k) + (c & 1), v ? src + idx : grid, v);
    }
  }
  __device__ const double2* compute(int, double2* b, double2* t) const {
    return fft_rows_sh<-1, SHAPE, CB / 2>(b, t, f, tw, CB / 2, M + 1, threadIdx.x, blockDim.x);
  }
  __device__ void store(int it, const double2* out) const {
    const int xr = it / ncb, x = L.xlo[0] + xr, y0 = (it - xr * ncb) * CB, S = M + 1;
    for (int idx = threadIdx.x; idx < nplanes * CB; idx += blockDim.x) {
      const int n = idx / CB, c = idx - n * CB;
      if (y0 + c < Mt) {
        const double2 Z = out[(c >> 1) * S + n], Zm = out[(c >> 1) * S + (n ? M - n : 0)];
        const double2 v = (c & 1) ? make_double2(0.5 * (Z.y + Zm.y), 0.5 * (Zm.x - Z.x))    // (Z - conj Zm)/(2i)
                                  : make_double2(0.5 * (Z.x + Zm.x), 0.5 * (Z.y - Zm.y));   // (Z + conj Zm)/2
        planes[slab_row(L, slot_of ? slot_of[n] : n, x, Mt) + y0 + c] = v;
      }
    }
  }
};

// inverse z-FFT: the slot first holds the raw (a, b) spectrum pairs, combined into the FFT input
// in the other buffer (see k_zinv)
template <int CB, int SHAPE = kPlanGeneric>
struct ZinvPass {
  int n_items, slot, ncb, Mt, M, mshift, nplanes;
  FftDesc f;
  const double2* tw;
  const double2* planes;
  double* grid;
  SlabLayout L;
  const int* slot_of;
  __device__ void load(int it, double2* dst) const {
    constexpr int CH = CB / 2;
    const int xr = it / ncb, x = L.xlo[0] + xr, y0 = (it - xr * ncb) * CB;
    for (int idx = threadIdx.x; idx < nplanes * CH; idx += blockDim.x) {
      const int n = idx / CH, r = idx - n * CH;
      const int64_t row = slab_row(L, slot_of ? slot_of[n] : n, x, Mt) + y0 + 2 * r;
      const bool va = y0 + 2 * r < Mt, vb = y0 + 2 * r + 1 < Mt;
      cp_async16(dst + 2 * idx, va ? planes + row : planes, va);
      cp_async16(dst + 2 * idx + 1, vb ? planes + row + 1 : planes, vb);
    }
  }
  __device__ const double2* compute(int, double2* b, double2* t) const {
    constexpr int CH = CB / 2;
    const int S = M + 1;
    for (int idx = threadIdx.x; idx < nplanes * CH; idx += blockDim.x) {
      const int n = idx / CH, r = idx - n * CH;
      const double2 a = b[2 * idx], bb = b[2 * idx + 1];
      t[r * S + n] = make_double2(a.x - bb.y, a.y + bb.x);
      if (n > 0 && 2 * n < M) t[r * S + (M - n)] = make_double2(a.x + bb.y, bb.x - a.y);   // Hermitian half
    }
    __syncthreads();
    return fft_rows_sh<1, SHAPE, CH>(t, b, f, tw, CH, S, threadIdx.x, blockDim.x);
  }
  __device__ void store(int it, const double2* out) const {
    const int xr = it / ncb, x = L.xlo[0] + xr, y0 = (it - xr * ncb) * CB, S = M + 1;
    double* dstg = grid + ((int64_t)x * Mt + y0) * M;
    for (int idx = threadIdx.x; idx < CB * M; idx += blockDim.x) {
      const int c = mshift >= 0 ? idx >> mshift : idx / M, k = idx - c * M;
      if (y0 + c < Mt) {
        const double2 v = out[(c >> 1) * S + k];
        dstg[idx] = (c & 1) ? v.y : v.x;
      }
    }
  }
};

// grid for a persistent pass: resident CTAs (occupancy query) x SMs, at most one per item
template <class PassT, int MINB>
static void persist_launch(const PassT& P, cudaStream_t st) {
  if (P.n_items <= 0) return;
  const size_t smem = 3 * (size_t)P.slot * sizeof(double2);
  const void* fn = (const void*)k_persist<PassT, MINB>;
  set_smem(fn, smem);
  int dev = 0, nsm = 0, per = 0;
  SE1P_CUDA_TRY(cudaGetDevice(&dev));
  SE1P_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  SE1P_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, SE1P_FFT_THREADS, smem));
  const int grid = std::max(1, std::min(P.n_items, std::max(per, 1) * nsm));
  k_persist<PassT, MINB><<<grid, SE1P_FFT_THREADS, smem, st>>>(P);
  SE1P_LAUNCH_CHECK();
}

template <int CB, int SHAPE>
static void zfwd_launch_sh(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, const int* slot_of,
                           int rows, cudaStream_t st) {
  const int M = pl.dv.M, Mt = pl.dv.Mt;
#if SE1P_PERSIST & 1
  {
    ZfwdPass<CB, SHAPE> P{};
    P.ncb = (int)ceil_div(Mt, CB);
    P.n_items = P.ncb * rows;
    P.slot = (CB / 2) * (M + 1);
    P.Mt = Mt;
    P.M = M;
    P.mshift = log2_or_neg(M);
    P.nplanes = pl.n_planes;
    P.f = pl.fz;
    P.tw = pl.d_tw + pl.twz;
    P.grid = w.grid;
    P.planes = planes;
    P.L = L;
    P.slot_of = slot_of;
    persist_launch<ZfwdPass<CB, SHAPE>, SE1P_FFT_MINB_Z>(P, st);
    return;
  }
#endif
  const size_t smem = 2 * (size_t)(CB / 2) * (M + 1) * sizeof(double2);
  set_smem((const void*)k_zfwd<CB, SHAPE>, smem);
  dim3 grid((unsigned)ceil_div(Mt, CB), (unsigned)rows);
  k_zfwd<CB, SHAPE><<<grid, kFftThreads, smem, st>>>(Mt, M, log2_or_neg(M), pl.n_planes, pl.fz, pl.d_tw + pl.twz, w.grid,
                                              planes, L, slot_of);
  SE1P_LAUNCH_CHECK();
}

template <int CB, int SHAPE>
static void zinv_launch_sh(const KPlan& pl, KWork& w, const double2* planes, const SlabLayout& L, const int* slot_of,
                           int rows, cudaStream_t st) {
  const int M = pl.dv.M, Mt = pl.dv.Mt;
#if SE1P_PERSIST & 2
  {
    ZinvPass<CB, SHAPE> P{};
    P.ncb = (int)ceil_div(Mt, CB);
    P.n_items = P.ncb * rows;
    P.slot = std::max((CB / 2) * (M + 1), 2 * pl.n_planes * (CB / 2));
    P.Mt = Mt;
    P.M = M;
    P.mshift = log2_or_neg(M);
    P.nplanes = pl.n_planes;
    P.f = pl.fz;
    P.tw = pl.d_tw + pl.twz;
    P.planes = planes;
    P.grid = w.grid;
    P.L = L;
    P.slot_of = slot_of;
    persist_launch<ZinvPass<CB, SHAPE>, SE1P_FFT_MINB_Z>(P, st);
    return;
  }
#endif
  const size_t smem = 2 * (size_t)(CB / 2) * (M + 1) * sizeof(double2);
  set_smem((const void*)k_zinv<CB, SHAPE>, smem);
  dim3 grid((unsigned)ceil_div(Mt, CB), (unsigned)rows);
  k_zinv<CB, SHAPE><<<grid, kFftThreads, smem, st>>>(Mt, M, log2_or_neg(M), pl.n_planes, pl.fz, pl.d_tw + pl.twz, planes,
                                              w.grid, L, slot_of);
  SE1P_LAUNCH_CHECK();
}

// the z-FFT with the compile-time 256-point plan where it applies (16 columns: 8 rows)
template <int CB>
static void zfwd_launch(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, const int* slot_of,
                        int rows, cudaStream_t st) {
  // (measured at C5: the compile-time plan in the one-shot forward kernel 0.163 -> 0.179 ms, in the
  // persistent one 0.149 ms)
  if (SE1P_FFT_CT && (SE1P_PERSIST & 1) && CB == 16 && fft_plan_shape(pl.fz) == kPlan256)
    zfwd_launch_sh<CB, kPlan256>(pl, w, planes, L, slot_of, rows, st);
  else
    zfwd_launch_sh<CB, kPlanGeneric>(pl, w, planes, L, slot_of, rows, st);
}
template <int CB>
static void zinv_launch(const KPlan& pl, KWork& w, const double2* planes, const SlabLayout& L, const int* slot_of,
                        int rows, cudaStream_t st) {
  if (SE1P_FFT_CT && CB == 16 && fft_plan_shape(pl.fz) == kPlan256)
    zinv_launch_sh<CB, kPlan256>(pl, w, planes, L, slot_of, rows, st);
  else
    zinv_launch_sh<CB, kPlanGeneric>(pl, w, planes, L, slot_of, rows, st);
}

void k_zfft_forward(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, const int* slot_of,
                    cudaStream_t st) {
  const int rows = L.xlo[L.nslab] - L.xlo[0];
  if (rows <= 0) return;
  switch (zcols(pl.dv.M)) {
    case 4: zfwd_launch<4>(pl, w, planes, L, slot_of, rows, st); break;
    case 8: zfwd_launch<8>(pl, w, planes, L, slot_of, rows, st); break;
    case 16: zfwd_launch<16>(pl, w, planes, L, slot_of, rows, st); break;
    case 32: zfwd_launch<32>(pl, w, planes, L, slot_of, rows, st); break;
    default: zfwd_launch<64>(pl, w, planes, L, slot_of, rows, st);
  }
}

void k_zfft_inverse(const KPlan& pl, KWork& w, const double2* planes, const SlabLayout& L, const int* slot_of,
                    cudaStream_t st) {
  const int rows = L.xlo[L.nslab] - L.xlo[0];
  if (rows <= 0) return;
  switch (zcols(pl.dv.M)) {
    case 4: zinv_launch<4>(pl, w, planes, L, slot_of, rows, st); break;
    case 8: zinv_launch<8>(pl, w, planes, L, slot_of, rows, st); break;
    case 16: zinv_launch<16>(pl, w, planes, L, slot_of, rows, st); break;
    case 32: zinv_launch<32>(pl, w, planes, L, slot_of, rows, st); break;
    default: zinv_launch<64>(pl, w, planes, L, slot_of, rows, st);
  }
}

// Column-pass block size: the warp multiple <= kColMaxThreads with the fewest butterfly rounds
// over the FFT's stages (stage s has CB W / R_s butterflies), then the fewest threads -- e.g. the
// 320-point J columns (radices 5, 8, 8) x 8 take 320 threads: 2 + 1 + 1 rounds instead of 2 + 2 + 2
static int col_threads(const FftDesc& f, int CB) {
  int best = kFftThreads, best_rounds = 1 << 30;
  for (int t = 128; t <= kColMaxThreads; t += 32) {
    int rounds = 0;
    for (int s = 0; s < f.nst; ++s) rounds += (int)ceil_div((int64_t)CB * (f.n / f.rad[s]), t);
    if (rounds < best_rounds) {
      best_rounds = rounds;
      best = t;
    }
  }
  return best;
}

template <int CB, int SHAPE>
static void colpass_launch_sh(const KPlan& pl, KWork& w, int nplanes, int W, const FftDesc& f, const double2* tw,
                              int64_t base, int kernel_class, PlaneSel S, cudaStream_t st) {
  const size_t smc = 2 * (size_t)CB * (W + 1) * sizeof(double2) + (kernel_class ? (size_t)CB * W * sizeof(double) : 0);
  set_smem((const void*)k_colpass<CB, SHAPE>, smc);
  k_colpass<CB, SHAPE><<<dim3((unsigned)ceil_div(W, CB), nplanes), col_threads(f, CB), smc, st>>>(
      pl.dv.Mt, W, base, f, tw, w.T, kernel_class, pl.d_khat, pl.d_exJ, pl.d_k2J, (const double2*)pl.d_pl, S);
  SE1P_LAUNCH_CHECK();
}
template <int CB>
static void colpass_launch(const KPlan& pl, KWork& w, int nplanes, int W, const FftDesc& f, const double2* tw,
                           int64_t base, int kernel_class, PlaneSel S, cudaStream_t st) {
  const int shape = SE1P_FFT_CT ? fft_plan_shape(f) : kPlanGeneric;
  if (shape == kPlan320)
    colpass_launch_sh<CB, kPlan320>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st);
  else if (shape == kPlan576)
    colpass_launch_sh<CB, kPlan576>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st);
  else
    colpass_launch_sh<CB, kPlanGeneric>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st);
}

static void mode_class(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, PlaneSel S, int nplanes,
                       int W, const FftDesc& f, int twoff, int64_t base, int kernel_class, cudaStream_t st) {
  if (nplanes <= 0) return;
  const int Mt = pl.dv.Mt;
  const int RB = rows_for(W), CB = cols_for(W);
#if SE1P_PERSIST & 4
  {
    const double2* tw = pl.d_tw + twoff;
    const int nxb = (int)ceil_div(Mt, RB);
    // compile-time plans where the shape and the rows per item match (C5: 320 x 4, 576 x 2)
    const int shape = SE1P_FFT_CT ? fft_plan_shape(f) : kPlanGeneric;
    auto rows = [&](auto sh, auto nr, bool inv) {
      constexpr int SH = decltype(sh)::value, NR = decltype(nr)::value;
      if (!inv) {
        RowFwdPass<SH, NR> R{nxb * nplanes, RB * W, nxb, Mt, W, RB, base, f, tw, planes, w.T, L, S};
        persist_launch<RowFwdPass<SH, NR>, SE1P_FFT_MINB_2D>(R, st);
      } else {
        RowInvPass<SH, NR> Q{nxb * nplanes, RB * W, nxb, Mt, W, RB, base, f, tw, w.T, planes, L, S};
        persist_launch<RowInvPass<SH, NR>, SE1P_FFT_MINB_2D>(Q, st);
      }
    };
    auto rows_dispatch = [&](bool inv) {
      if (shape == kPlan320 && RB == 4)
        rows(std::integral_constant<int, kPlan320>(), std::integral_constant<int, 4>(), inv);
      else if (shape == kPlan576 && RB == 2)
        rows(std::integral_constant<int, kPlan576>(), std::integral_constant<int, 2>(), inv);
      else
        rows(std::integral_constant<int, kPlanGeneric>(), std::integral_constant<int, 1>(), inv);
    };
    rows_dispatch(false);
#if SE1P_PERSIST & 8
    const int cb = W > 400 ? SE1P_PCOLS_LARGE : SE1P_PCOLS_SMALL;
    auto col = [&](auto cbc) {
      constexpr int C = decltype(cbc)::value;
      ColPass<C> P{};
      P.ncb = (int)ceil_div(W, C);
      P.n_items = P.ncb * nplanes;
      P.slot = C * (W + 1) + (kernel_class ? (C * W + 1) / 2 : 0);
      P.Mt = Mt;
      P.W = W;
      P.kernel_class = kernel_class;
      P.base = base;
      P.f = f;
      P.tw = tw;
      P.T = w.T;
      P.khat = pl.d_khat;
      P.exJ = pl.d_exJ;
      P.k2J = pl.d_k2J;
      P.pl = (const double2*)pl.d_pl;
      P.S = S;
      persist_launch<ColPass<C>, SE1P_FFT_MINB_2D>(P, st);
    };
    if (cb == 2) col(std::integral_constant<int, 2>());
    else if (cb == 8) col(std::integral_constant<int, 8>());
    else col(std::integral_constant<int, 4>());
#else
    switch (CB) {
      case 2: colpass_launch<2>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st); break;
      case 4: colpass_launch<4>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st); break;
      case 16: colpass_launch<16>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st); break;
      default: colpass_launch<8>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st);
    }
#endif
    rows_dispatch(true);
    return;
  }
#endif
  const size_t smr = 2 * (size_t)RB * W * sizeof(double2);
  set_smem((const void*)k_rowfwd, smr);
  set_smem((const void*)k_rowinv, smr);
  const double2* tw = pl.d_tw + twoff;
  k_rowfwd<<<dim3((unsigned)ceil_div(Mt, RB), nplanes), kFftThreads, smr, st>>>(Mt, W, base, RB, f, tw, planes, w.T, L, S);
  SE1P_LAUNCH_CHECK();
  switch (CB) {
    case 2: colpass_launch<2>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st); break;
    case 4: colpass_launch<4>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st); break;
    case 16: colpass_launch<16>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st); break;
    default: colpass_launch<8>(pl, w, nplanes, W, f, tw, base, kernel_class, S, st);
  }
  k_rowinv<<<dim3((unsigned)ceil_div(Mt, RB), nplanes), kFftThreads, smr, st>>>(Mt, W, base, RB, f, tw, w.T, planes, L, S);
  SE1P_LAUNCH_CHECK();
}

// Kernel planes (k3 = 0 and the I modes, global index < n_kernel) and J planes.  Null maps: all
// planes, global index = slot.  Otherwise glK/liK (nK entries) and glJ/liJ (nJ entries) are
// device arrays of global plane indices and their slots in the buffer.
void k_mode_stage(const KPlan& pl, KWork& w, double2* planes, const SlabLayout& L, const int* glK, const int* liK,
                  int nK, const int* glJ, const int* liJ, int nJ, cudaStream_t st) {
  const int Mt = pl.dv.Mt;
  if (!glK) nK = pl.n_kernel;
  if (!glJ) nJ = pl.n_planes - pl.n_kernel;
  const int64_t baseJ = (int64_t)nK * Mt * pl.LK;
#if SE1P_MODES_TWO_STREAMS
  // the two plane classes are independent (disjoint planes and T regions) and each pass is
  // latency bound: the kernel planes run on a second stream beside the J planes
  if (nK > 0 && nJ > 0) {
    if (!w.side) {
      SE1P_CUDA_TRY(cudaStreamCreateWithFlags(&w.side, cudaStreamNonBlocking));
      SE1P_CUDA_TRY(cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming));
      SE1P_CUDA_TRY(cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming));
    }
    SE1P_CUDA_TRY(cudaEventRecord(w.ev_fork, st));
    SE1P_CUDA_TRY(cudaStreamWaitEvent(w.side, w.ev_fork, 0));
    mode_class(pl, w, planes, L, PlaneSel{glK, liK, 0}, nK, pl.LK, pl.fK, pl.twK, 0, 1, w.side);
#if SE1P_MODES_TWO_STREAMS > 1
    if (nJ >= 8) {   // the J planes in two halves on two streams
      if (!w.side2) {
        SE1P_CUDA_TRY(cudaStreamCreateWithFlags(&w.side2, cudaStreamNonBlocking));
        SE1P_CUDA_TRY(cudaEventCreateWithFlags(&w.ev_join2, cudaEventDisableTiming));
      }
      SE1P_CUDA_TRY(cudaStreamWaitEvent(w.side2, w.ev_fork, 0));
      // SE1P_MODES_JSPLIT chunks, alternating between the two streams (smaller chunks keep each
      // chunk's row-transformed planes T resident in L2 between its three passes)
      const int nch = std::max(2, std::min(SE1P_MODES_JSPLIT, nJ / 4));
      for (int ch = 0; ch < nch; ++ch) {
        const int a0 = (int)((int64_t)nJ * ch / nch), a1 = (int)((int64_t)nJ * (ch + 1) / nch);
        const PlaneSel Sc{glJ ? glJ + a0 : nullptr, liJ ? liJ + a0 : nullptr, pl.n_kernel + a0};
        mode_class(pl, w, planes, L, Sc, a1 - a0, pl.prm.SJ, pl.fJ, pl.twJ, baseJ + (int64_t)a0 * Mt * pl.prm.SJ, 0,
                   (ch & 1) ? w.side2 : st);
      }
      SE1P_CUDA_TRY(cudaEventRecord(w.ev_join2, w.side2));
      SE1P_CUDA_TRY(cudaStreamWaitEvent(st, w.ev_join2, 0));
    } else
#endif
      mode_class(pl, w, planes, L, PlaneSel{glJ, liJ, pl.n_kernel}, nJ, pl.prm.SJ, pl.fJ, pl.twJ, baseJ, 0, st);
    SE1P_CUDA_TRY(cudaEventRecord(w.ev_join, w.side));
    SE1P_CUDA_TRY(cudaStreamWaitEvent(st, w.ev_join, 0));
    return;
  }
#endif
  mode_class(pl, w, planes, L, PlaneSel{glK, liK, 0}, nK, pl.LK, pl.fK, pl.twK, 0, 1, st);
  mode_class(pl, w, planes, L, PlaneSel{glJ, liJ, pl.n_kernel}, nJ, pl.prm.SJ, pl.fJ, pl.twJ, baseJ, 0, st);
}

// ------------------------------------------------------------------ plan-time kernel spectra
// sig: (S/2+1)^2 table of the scaling function over |a'|,|b'| (host computed).
// Step A: tmp[d][m2] = sum_{m1} mult(m1) sig[m1][m2] cos(2 pi m1 d/S), d < Mt, m2 <= S/2.
__global__ void k_kern_a(int S, int Mt, const double* __restrict__ sig, double* __restrict__ tmp) {
  const int H = S / 2 + 1;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)Mt * H) return;
  const int d = (int)(id / H), m2 = (int)(id - (int64_t)d * H);
  double acc = 0.0;
  for (int m1 = 0; m1 < H; ++m1) {
    const double mult = (m1 == 0 || 2 * m1 == S) ? 1.0 : 2.0;
    const long long r = ((long long)m1 * d) % S;
    acc = fma(mult * sig[(int64_t)m1 * H + m2], cospi(2.0 * (double)r / (double)S), acc);
  }
  tmp[id] = acc;
}

// Step B: K[d1][d2] = (1/S^2) sum_{m2} mult(m2) tmp[d1][m2] cos(2 pi m2 d2/S), written into the
// LK x LK complex array at (+-d1 mod LK, +-d2 mod LK).
__global__ void k_kern_b(int S, int Mt, int LK, const double* __restrict__ tmp, double2* __restrict__ KL) {
  const int H = S / 2 + 1;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)Mt * Mt) return;
  const int d1 = (int)(id / Mt), d2 = (int)(id - (int64_t)d1 * Mt);
  double acc = 0.0;
  for (int m2 = 0; m2 < H; ++m2) {
    const double mult = (m2 == 0 || 2 * m2 == S) ? 1.0 : 2.0;
    const long long r = ((long long)m2 * d2) % S;
    acc = fma(mult * tmp[(int64_t)d1 * H + m2], cospi(2.0 * (double)r / (double)S), acc);
  }
  acc /= (double)S * (double)S;
  const int i1[2] = {d1, (LK - d1) % LK}, i2[2] = {d2, (LK - d2) % LK};
  for (int s1 = 0; s1 < 2; ++s1)
    for (int s2 = 0; s2 < 2; ++s2) KL[(int64_t)i1[s1] * LK + i2[s2]] = make_double2(acc, 0.0);
}

// In-place FFT of the rows of an n x n complex matrix (plan-time helper).
__global__ void k_fft_rows_inplace(int n, int RB, FftDesc f, const double2* __restrict__ tw, double2* __restrict__ A) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* tmp = sm + RB * n;
  const int r0 = blockIdx.x * RB, nr = min(RB, n - r0);
  for (int idx = threadIdx.x; idx < RB * n; idx += blockDim.x)
    buf[idx] = (idx / n < nr) ? A[(int64_t)r0 * n + idx] : make_double2(0.0, 0.0);
  __syncthreads();
  double2* out = fft_rows<-1>(buf, tmp, f, tw, RB, n, threadIdx.x, blockDim.x);
  for (int idx = threadIdx.x; idx < nr * n; idx += blockDim.x) A[(int64_t)r0 * n + idx] = out[idx];
}

__global__ void k_transpose_scale_real(int n, double scale, const double2* __restrict__ A, double* __restrict__ out) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)n * n) return;
  const int i = (int)(id / n), j = (int)(id - (int64_t)i * n);
  out[id] = A[(int64_t)j * n + i].x * scale;
}

__global__ void k_transpose(int n, const double2* __restrict__ A, double2* __restrict__ B) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)n * n) return;
  const int i = (int)(id / n), j = (int)(id - (int64_t)i * n);
  B[id] = A[(int64_t)j * n + i];
}

// Device part of the kernel spectrum: sig (host table, device copy) -> khat_out [LK][LK].
void build_kernel_spectrum(const KPlan& pl, int S, const double* d_sig, double* khat_out, double scale,
                           const KernScratch& ks, cudaStream_t st) {
  const int Mt = pl.dv.Mt, LK = pl.LK, H = S / 2 + 1;
  double* tmp = ks.tmp;
  double2 *A = ks.A, *B = ks.B;
  SE1P_CUDA_TRY(cudaMemsetAsync(A, 0, sizeof(double2) * (size_t)LK * LK, st));
  k_kern_a<<<(unsigned)ceil_div((int64_t)Mt * H, 128), 128, 0, st>>>(S, Mt, d_sig, tmp);
  SE1P_LAUNCH_CHECK();
  k_kern_b<<<(unsigned)ceil_div((int64_t)Mt * Mt, 128), 128, 0, st>>>(S, Mt, LK, tmp, A);
  SE1P_LAUNCH_CHECK();
  const int RB = rows_for(LK);
  const size_t sm = 2 * (size_t)RB * LK * sizeof(double2);
  set_smem((const void*)k_fft_rows_inplace, sm);
  const double2* tw = pl.d_tw + pl.twK;
  k_fft_rows_inplace<<<(unsigned)ceil_div(LK, RB), 256, sm, st>>>(LK, RB, pl.fK, tw, A);
  SE1P_LAUNCH_CHECK();
  k_transpose<<<(unsigned)ceil_div((int64_t)LK * LK, 256), 256, 0, st>>>(LK, A, B);
  SE1P_LAUNCH_CHECK();
  k_fft_rows_inplace<<<(unsigned)ceil_div(LK, RB), 256, sm, st>>>(LK, RB, pl.fK, tw, B);
  SE1P_LAUNCH_CHECK();
  // B = transpose of the 2D spectrum; transpose back while taking the (real) value
  k_transpose_scale_real<<<(unsigned)ceil_div((int64_t)LK * LK, 256), 256, 0, st>>>(LK, scale, B, khat_out);
  SE1P_LAUNCH_CHECK();
}

}  // namespace se1p
