/*
 * se1p.h -- C ABI of the B200-native SE1P k-space library (libse1p.so).
 *
 * Method: Saffar Shamshirgar & Tornberg, "The Spectral Ewald method for singly periodic
 * domains", arXiv:1611.09538.  "P:n" cites line n of the paper's text.
 *
 * Problem (Eq. (1), with P_1 periodicity P:79): N point charges q_n at x_n in
 * [0,L1) x [0,L2) x [0,L3), periodic along axis 3 (z) only, free along axes 1,2.
 * The library evaluates the Ewald1P split of the potential at every charge location:
 *   se1p_kspace  ->  phi^F  = phi^{F,k3!=0} + phi^{F,k3=0}   (Alg. 1; Eqs. (4),(5))
 *   se1p_real    ->  phi^R + phi^self                       (Eq. (3), Eq. (6))
 * Their sum is the full potential phi of Eq. (2).
 *
 * Conventions for every entry point
 *   - x: double[3*N], interleaved x0,y0,z0,x1,...; q: double[N]; phi_out: double[N].
 *     The caller owns all three.  Inputs are never modified (z is folded into [0,L3)
 *     internally).  phi_out is overwritten (phi_out[n] belongs to particle n).
 *   - Pointers are CUDA DEVICE pointers on the current device unless opts->host_io != 0,
 *     in which case they are host pointers and the library copies in and out (the copies
 *     are part of the call).
 *   - All arithmetic is IEEE fp64.  Results are bitwise reproducible for identical inputs
 *     (no floating-point atomics; every reduction has a fixed order).
 *   - The plain entries (se1p_kspace, se1p_real) are synchronous and return a complete
 *     status including CUDA errors.  The _ex entries enqueue on `stream` (cudaStream_t,
 *     NULL = legacy default stream) and, with opts->sync == 0, return after enqueueing;
 *     argument errors are still returned synchronously.
 *   - On any non-OK return, se1p_last_error() gives a thread-local message.
 *   - Thread safety: calls on different threads are serialised by an internal mutex
 *     (plans and workspaces are per device and shared).  Calls may use different streams:
 *     each call's stream first waits (cudaStreamWaitEvent) for the work the previous call on
 *     the same device enqueued, so stream-ordered (sync == 0) calls on two streams never
 *     overlap on the shared workspace.
 */
#ifndef SE1P_H
#define SE1P_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SE1P_OK = 0,
  SE1P_EINVAL = 1,       /* null pointer, N < 1, xi <= 0, L <= 0, rc <= 0, M < 2            */
  SE1P_EDOMAIN = 2,      /* an x or y coordinate outside [0,L1) x [0,L2)  (free axes)          */
  SE1P_ENONNEUTRAL = 3,  /* |sum q| > 1e-12 * sum |q|; Eq. (5) needs neutrality */
  SE1P_EPARAM = 4,       /* L1/h or L2/h not an integer, L1/h != L2/h, P < 2 or P > M,
                            eta not in (0,1), n_local > M/2, FFT extent < M+P or
                            with a prime factor > 61                                         */
  SE1P_ENOMEM = 5,
  SE1P_ECUDA = 6,
  SE1P_ENCCL = 7
} se1p_status;

/* Options for the _ex entries.  Zero-initialise and set what you need; every 0 means
   "default".  Padded FFT extents are integers (reading R-5: the paper's s0, s_l are
   factors relative to M~ = M_free + P and it asks for s M~ to be an integer). */
typedef struct se1p_opts {
  int Ntilde;       /* FFT extent of the free axes for the k3 in J modes (s = 1);
                       0 -> planner (>= M~, FFT-friendly, widened per DESIGN.md).         */
  int S0;           /* padded extent for k3 = 0 (the paper's s0 M~); 0 -> from s0         */
  int SI;           /* padded extent for k3 in I (the paper's s_l M~); 0 -> from sf       */
  int host_io;      /* 1: x, q, phi_out are host pointers (copied in/out inside the call) */
  int skip_checks;  /* 1: skip the device-side domain and neutrality checks               */
  int sync;         /* 1: synchronise the stream before returning (plain entries do)     */
  int reserved[10];
} se1p_opts;

/* Derived sizes of a k-space plan (for reporting and tests). */
typedef struct se1p_plan_info {
  double h;         /* grid step L3/M (Alg. 1 step 1)                              */
  double eta;       /* Gaussian split parameter (Eq. (comp_eta))                    */
  int M;            /* periodic-axis points                                               */
  int Mfree;        /* L1/h = L2/h                                                        */
  int Mt;           /* M~ = Mfree + P                                             */
  int P;
  int n_local;      /* n_l: |k3| <= 2 pi n_l/L3 are upsampled (Eq. (I))             */
  int Ntilde;       /* J-mode FFT extent                                                  */
  int S0, SI;       /* padded extents of the k3 = 0 and I modes                            */
  int LK;           /* FFT extent used on the device for the upsampled modes (>= 2 M~ - 1):
                       their padded transform is applied as an exact aperiodic convolution
                       with a plan-time kernel.                   */
  int n_kernel_planes;  /* planes handled through LK (k3 = 0 and the I modes, k3 >= 0)   */
  int n_planes;         /* M/2 + 1 (Hermitian half along z)                              */
  int64_t grid_points;  /* M~^2 * M real grid points                                     */
  int64_t workspace_bytes;
  double plan_ms;       /* host wall time of the plan build (tables, kernel spectra); paid once
                           per parameter set, not per call                                   */
} se1p_plan_info;

/* k-space potential phi^F (Alg. 1 OUTPUT): no real-space and no self term.
     M        grid points along the periodic axis; h = L[2]/M.  The free axes are solved on the
              square [0, max(L[0],L[1]))^2, whose side must be an integer multiple of h; a
              rectangular box is embedded in it (phi^F is free-space in x, y, so
              the embedding does not change it; reading R-19).
     P        Gaussian support points per dimension
     eta      <= 0 -> P xi^2 h^2/(0.95^2 pi) (Eq. (comp_eta))
     s0, sf   upsampling factors of k3 = 0 and of the I modes (Eq. (upsamplings));
              <= 0 -> planner default.  Padded extents are ceil(s M~).
     n_local  n_l (Eq. (I)); < 0 -> planner default.
   sf == s0 with n_local == M/2 reproduces the plain upsampled FFT.              */
int se1p_kspace(const double* x, const double* q, int64_t N, const double L[3], double xi,
                int M, int P, double eta, double s0, double sf, int n_local, double* phi_out);

int se1p_kspace_ex(const se1p_opts* opts, void* stream, const double* x, const double* q,
                   int64_t N, const double L[3], double xi, int M, int P, double eta,
                   double s0, double sf, int n_local, double* phi_out);

/* ---------------------------------------------------------------------------------------
 * Mode-sharded k-space over R ranks.  One rank per GPU;
 * the caller moves the plane buffers between ranks (all-to-all) and sums phi_partial (all-reduce).
 * Every rank holds the full x, q (device pointers).  The free axis x of the extended grid
 * (M~ = M_free + P rows) is cut into R slabs [slab_lo[r], slab_lo[r+1]), bounds multiples of 16
 * (the last may be M~); the M/2+1 k3 planes (Hermitian half, reading R-7) are owned by ranks.
 *
 * Plane buffers hold complex doubles (re, im pairs):
 *   slab buffer   (forward output / backward input) of rank r: [M/2+1 slots][W_r][M~], W_r the slab
 *                 width; slot i holds plane plane_order[i].  With plane_order grouping the planes
 *                 by owner (rank 0's planes first), the chunk for owner r' is contiguous.
 *   split buffer  (se1p_kspace_modes) of an owner with n_own planes: the concatenation over source
 *                 slabs r of [n_own][W_r][M~] -- exactly what an all-to-all of the slab buffers
 *                 delivers; the mode stage runs in place and the same all-to-all in reverse
 *                 returns every rank its slab buffer.
 *
 * se1p_kspace_slab_forward: Alg. 1 steps 2-3a (AFT step 1 P:749) restricted to the slab:
 *   compacts the particles whose stencils meet the slab's tiles, bins and sorts those, grids the
 *   slab's x rows (output-stationary tiles, so no reduction between ranks) and transforms them
 *   along z.  planes_out: slab buffer (caller owned).  Synchronises the stream once (the
 *   compacted count sizes the sort).
 * se1p_kspace_modes: Alg. 2 steps 2-4, the scaling of Alg. 1 step 4 and Alg. 3 steps 1-3
 *    for the n_own planes plane_ids[] (global k3 indices 0..M/2) held in the
 *   split buffer `planes` described by nslab, slab_lo[0..nslab] (slab_lo[0] = 0, slab_lo[nslab] = M~).
 * se1p_kspace_slab_backward: Alg. 3 steps 4-5 for the slab rows and the gather
 *   (Alg. 1 step 6) over the slab's tiles: phi_partial[n] (user order, N doubles) is the
 *   slab's share of phi^F at particle n; the sum over all slabs is se1p_kspace's result.  Uses the
 *   particle state of the last se1p_kspace_slab_forward on this device with the same N and
 *   parameters (SE1P_EINVAL otherwise).
 * An empty slab (x_lo == x_hi) is allowed; its buffers may then be NULL.
 * All three are stream-ordered like the _ex entries (opts->sync), take device pointers only
 * (opts->host_io is rejected) and share the device's workspace: issue them on one stream.
 * --------------------------------------------------------------------------------------- */
int se1p_kspace_slab_forward(const se1p_opts* opts, void* stream, const double* x, const double* q,
                             int64_t N, const double L[3], double xi, int M, int P, double eta,
                             double s0, double sf, int n_local, int x_lo, int x_hi,
                             const int* plane_order, void* planes_out);

int se1p_kspace_modes(const se1p_opts* opts, void* stream, const double L[3], double xi, int M, int P,
                      double eta, double s0, double sf, int n_local, int n_own, const int* plane_ids,
                      int nslab, const int* slab_lo, void* planes);

int se1p_kspace_slab_backward(const se1p_opts* opts, void* stream, int64_t N, const double L[3],
                              double xi, int M, int P, double eta, double s0, double sf, int n_local,
                              int x_lo, int x_hi, const int* plane_order, const void* planes_in,
                              double* phi_partial);

/* Real-space erfc sum truncated at |x_m - x_n + alpha L3 e3| <= rc over z-images alpha
   (Eq. (3); truncation P:120; cell lists P:161-162) plus the self term
   -2 xi q_m/sqrt(pi) (Eq. (6)).  Any rc > 0 (all images within rc are included). */
int se1p_real(const double* x, const double* q, int64_t N, const double L[3], double xi,
              double rc, double* phi_out);

/* se1p_real_ex / se1p_real_field_ex with opts->reserved[4] = R > 1 and opts->reserved[5] = r
   (0 <= r < R): part r of R of the sum -- the targets are split into R near-equal parts (the
   warp kernel's target groups in sorted order) and only part r's entries of phi_out (and
   field_out) are computed; the others are set to 0, so the R parts sum exactly (bitwise) to the
   whole.  For ranks sharing the real-space sum (dist.real: each rank its part, one all-reduce).
   reserved[4] = 0 or 1: the whole sum.  Errors: SE1P_EINVAL for R < 0 or r outside [0, R). */
int se1p_real_ex(const se1p_opts* opts, void* stream, const double* x, const double* q,
                 int64_t N, const double L[3], double xi, double rc, double* phi_out);

/* Electric field E = -grad phi at the particles (force on particle n: F_n = q_n E_n), the
   derivative the paper's force expressions take: SURVEY.md 8(f) NEXT-1.
   se1p_kspace_field_ex: the k-space field E^F = -grad phi^F of Alg. 1 -- the same grid H~
     (steps 1-5) gathered with the gradient of the Gaussian window (step 6 differentiated,
     P:270-275: d/dx_n e^{-alpha|x-x_n|^2} = 2 alpha (x - x_n) e^{-alpha|x-x_n|^2}).
   se1p_real_field_ex: E^R = -grad phi^R of Eq. (3) with the same truncation as se1p_real
     (the self term has no gradient).
   field_out: [N][3] doubles (x, y, z components) in the caller's particle order, required;
   phi_out: N doubles or NULL -- when given, the potential of the matching non-field call is
   written too (same values).  Arguments, ownership, opts and errors as the _ex entries above.
   opts->reserved[2] must be 0. */
int se1p_kspace_field_ex(const se1p_opts* opts, void* stream, const double* x, const double* q,
                         int64_t N, const double L[3], double xi, int M, int P, double eta,
                         double s0, double sf, int n_local, double* phi_out, double* field_out);

int se1p_real_field_ex(const se1p_opts* opts, void* stream, const double* x, const double* q,
                       int64_t N, const double L[3], double xi, double rc, double* phi_out,
                       double* field_out);

/* Energy, potentials and forces of the full singly periodic sum (Eq. (2), and its
   gradient): phi = phi^F + phi^R + phi^self, E = E^F + E^R (the two field entries above, with rc
   for the real-space term), F_n = q_n E_n (reading R-17) and the energy
   U = 1/2 sum_n q_n phi_n, reduced on the device in a fixed order (bitwise
   reproducible).  U_out: 1 double; phi_out: N doubles or NULL; F_out: [N][3] doubles, required.
   All are device pointers, or host pointers with opts->host_io (then the call is synchronous).
   Arguments and errors as se1p_kspace_ex and se1p_real_ex (rc > 0). */
int se1p_energy_forces(const se1p_opts* opts, void* stream, const double* x, const double* q, int64_t N,
                       const double L[3], double xi, double rc, int M, int P, double eta, double s0,
                       double sf, int n_local, double* U_out, double* phi_out, double* F_out);

/* Resolve the plan the k-space call with these arguments would use (no device work
   beyond plan creation).  Returns SE1P_OK or the same errors as se1p_kspace_ex. */
int se1p_plan_query(const se1p_opts* opts, const double L[3], double xi, int M, int P,
                    double eta, double s0, double sf, int n_local, se1p_plan_info* info);

/* Multi-tier adaptive upsampling (generalises the paper's three tiers
   s0 / s_l / 1 of Eq. (upsamplings), and its Table 2 "plain upsampled FFT"):
   mode |k3| = 2 pi n/L3, n = 1..n_local, uses the padded extent S_modes[n-1] (each >= M~; the
   paper's s(n) M~), k3 = 0 uses S0 (opts->S0, or s0), |k3| > 2 pi n_local/L3 the J extent.
   n_local must be given (>= 0); S_modes holds n_local ints (host).  Other arguments, ownership
   and errors as se1p_kspace_ex.  On this device path every upsampled mode costs the same
   exact-convolution transform whatever its extent, so the tiers set the
   discretisation (and error), not the run time. */
int se1p_kspace_tiers_ex(const se1p_opts* opts, void* stream, const double* x, const double* q,
                         int64_t N, const double L[3], double xi, int M, int P, double eta,
                         double s0, int n_local, const int* S_modes, double* phi_out);

/* SE3P baseline (the paper's Ex. 5, compares SE1P with the
   triply periodic SE3P): the k-space part of the triply periodic Ewald sum with tin-foil boundary,
     phi^F(x_m) = (4 pi/V) sum_{k != 0} e^{-k^2/4 xi^2}/k^2 sum_n q_n cos(k.(x_m - x_n)),
   by Spectral Ewald: the same gridding and gather as se1p_kspace (Gaussians of Eq. (spread_1p)
   truncated to P^3 nodes, h = L[2]/M, eta as in se1p_kspace), a plain 3D FFT of the
   M_free x M_free x M periodic grid (no upsampling) and the scaling e^{-(1-eta)k^2/4xi^2}/k^2
   (k = 0 dropped).  P must be even; x, y in [0,L1) x [0,L2) (any z).  Same pointers, ownership,
   opts and errors as se1p_kspace_ex; L1 != L2 -> SE1P_EPARAM (the periodic cross-section must be
   square in this build). */
int se1p_kspace3p_ex(const se1p_opts* opts, void* stream, const double* x, const double* q,
                     int64_t N, const double L[3], double xi, int M, int P, double eta,
                     double* phi_out);

/* Parameters from an absolute rms error tolerance: the paper's recipe
   "Parameter selection" -- rc and kinf by inverting the Kolafa-Perram estimates
   (Eqs. (rc), (kinf), Lambert W), M = 2 kinf (even, FFT-friendly, max(L1,L2)/h
   integer), P the smallest even integer with A e^{-c^2 pi P/2} <= tol (Eq.
   (approximation_error_oneterm), c = 0.95), eta, s_l from e^{-2 pi s_l} < tol
   (P:697), n_l = ceil(M/10), s0 = 1 + sqrt(2).  Host-only (no device
   work).  Non-cubic boxes: DESIGN.md reading R-18.  Q = sum q_n^2; xi is the caller's choice
   (the paper balances real- and k-space run time).  Each estimate is inverted at a share
   of tol (real space tol/2, k-space truncation and aliasing tol/10, window tol/100) and M is
   raised until eta <= 0.8 (reading R-18), so the measured rms error meets tol.
   Errors: SE1P_EINVAL (null, Q/xi/L <= 0, tol not in (0,1)), SE1P_EPARAM (no admissible M <=
   8192). */
typedef struct se1p_tol_plan {
  double xi, tol, Q;
  double rc;                 /* real-space cutoff, Eq. (rc)                                  */
  double kinf;               /* Eq. (kinf) (unrounded)                                       */
  int M, P, Mfree, Mt;       /* periodic points, support, max(L1,L2)/h, M~ = Mfree + P      */
  double h, eta;
  int n_local;               /* n_l                                                          */
  double s_l, s0;            /* upsampling factors                                           */
  int SI, S0, Ntilde;        /* extents for se1p_opts (SI = ceil(s_l M~), S0 = ceil(s0 M~))  */
  double est_real, est_fourier, est_approx;   /* the three estimates at the chosen values   */
} se1p_tol_plan;

int se1p_plan_from_tol(const double L[3], double Q, double xi, double tol, se1p_tol_plan* out);

/* The erfc table of the real-space kernel (host only, no device needed; for inspection and
   tests).  On kRealK = *intervals equal intervals of [0, rc], erfc(xi r) is the polynomial
   sum_n c[n][i] (r - (i + 1/2) rc/K)^n of degree *degree (Chebyshev interpolant, within 2e-16 of
   erfc in absolute terms); *degree = 0 means xi rc is beyond the table and
   the thread-per-target kernel is used.  coeffs: caller-owned, (degree + 1) * intervals doubles,
   coefficient-major c[n][i]; written only if capacity is large enough (query with coeffs = NULL).
   Errors: SE1P_EINVAL for null degree/intervals or xi, rc <= 0. */
int se1p_real_table(double xi, double rc, int* degree, int* intervals, double* coeffs, int capacity);

/* Per-stage device time of the last _ex call on this thread, in milliseconds, measured
   with CUDA events on the call's stream when opts->reserved[0] == 1 (profiling mode).
   Stages: 0 bin/sort, 1 particle records (window weights), 2 gridding tiles, 3 z-FFT,
   4 mode stage, 5 inverse z-FFT, 6 gather tiles, 7 gather slot sum.  Returns stages written. */
int se1p_last_stage_times(double* ms, int max_stages);

/* Number of kernels the library launched in the last call on this thread. */
int se1p_last_launch_count(void);

/* Testing hook: with opts->reserved[1] = s (1..4) a k-space call stops after stage s
   (1 gridding, 2 z-FFT, 3 mode stage, 4 inverse z-FFT) and leaves phi_out untouched.
   se1p_debug_copy then copies `count` elements of workspace buffer `which` (0: real grid
   [M~][M~][M] doubles, 1: k3 planes [M/2+1][M~][M~] complex as double pairs) to host memory.
   Returns SE1P_OK or SE1P_EINVAL if the buffer is smaller than requested. */
int se1p_debug_copy(int which, double* host_dst, int64_t count);

/* Free all plans and workspaces of the current device. */
void se1p_release(void);

/* Device-memory hook (SURVEY.md 8(b) "Ownership": the Python layer routes the library's memory
   to torch's caching allocator).  Every plan, workspace and table the library allocates from now
   on comes from alloc(bytes, ctx) (must return device memory of the current device, >= 256-byte
   aligned, or NULL -> SE1P_ENOMEM) and goes back through release(ptr, ctx).  Before a pointer is
   released the library synchronises the device, so the hook may reuse it at once.  The call
   first frees everything allocated so far on every device (through the allocator that made it),
   then installs the hook; alloc = release = NULL restores cudaMalloc / cudaFree.  Not to be
   called while another thread is inside the library.  Returns SE1P_OK, or SE1P_EINVAL if
   exactly one of alloc, release is NULL (nothing changes then). */
int se1p_set_allocator(void* (*alloc)(size_t bytes, void* ctx), void (*release)(void* ptr, void* ctx), void* ctx);

const char* se1p_last_error(void);
const char* se1p_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SE1P_H */
