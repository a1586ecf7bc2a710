// tiles.cuh -- shared machinery of the gridding and gather sweep kernels (sweep.cu).
//
// Gridding (Alg. 1 step 2, Eq. (spread_1p)) is, per output tile, the contraction
//   H[(x,y), z] += sum_p (q_p wx_p[x] wy_p[y]) wz_p[z]
// and the gather (Alg. 1 step 6, Eq. (se1p_complete_discretized)) the contraction
//   T[(x,y), p] = sum_z H~[(x,y), z] wz_p[z],   phi_p += sum_(x,y) wx_p[x] wy_p[y] T[(x,y), p].
// Both run on the FP64 tensor pipe with mma.sync m16n8k8 f64 (SASS DMMA): tcgen05.mma has no
// f64 kind, so DMMA is the sm_100a fp64 matrix path (same 37 TFLOP/s as DFMA, 4-16x fewer
// instructions per FMA).  The mma wrappers are plain (not volatile) asm: an MMA is a pure
// function of its operands, so the compiler may schedule the surrounding loads across it.
#pragma once
#include "kspace.cuh"

namespace se1p {

constexpr int kTXY = 16;        // CTA tile extent in x and y (grid nodes)
constexpr int kBXY = 4;         // particle bins: xy columns of kBXY x kBXY cells, z-sorted inside

// Doubles per particle record (sweep.cu, k_records).
int rec_doubles(int P);

__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double (&a)[4], double b0, double b1) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0), "d"(b1));
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], const double (&a)[2], double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(b0));
}

__device__ __forceinline__ void dmma_16x8x16(double (&c)[4], const double (&a)[8], double b0, double b1, double b2,
                                             double b3) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b0), "d"(b1),
        "d"(b2), "d"(b3));
}

__device__ __forceinline__ int fdiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
__device__ __forceinline__ int pmod(int a, int m) { int r = a % m; return r < 0 ? r + m : r; }

}  // namespace se1p
