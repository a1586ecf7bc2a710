// tiles.cuh -- shared machinery of the DMMA gridding and gather kernels (tiles.cu).
//
// CTA tile: 16 (x) x 16 (y) columns of the extended grid x TZ (z) nodes, 16 warps; warp w owns
// the 4 x 4 column block (4 (w&3), 4 (w>>2)) over all TZ nodes.  Gridding is the contraction
//   H[(x,y), z] += sum_p (wx_p[x] wy_p[y]) (q_p wz_p[z])                 (Eq. (spread_1p))
// and the gather the contraction T[(x,y), p] = sum_z H~[(x,y), z] wz_p[z] followed by
// phi_p += sum_(x,y) wx_p[x] wy_p[y] T[(x,y), p]                          (Eq. (se1p_complete_
// discretized)); both run on the FP64 tensor pipe (mma.sync m16n8k4 f64, SASS DMMA).
#pragma once
#include "kspace.cuh"

namespace se1p {

constexpr int kTXY = 16;        // CTA x and y extent (grid nodes)
constexpr int kWarps = 16;      // 4 x 4 column blocks of 4 x 4
constexpr int kStage = 64;      // particles staged per batch
constexpr int kSX = 20;         // smem row stride of x/y weights (doubles, = 4 mod 16: no bank conflicts)

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ int fdiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
__device__ __forceinline__ int pmod(int a, int m) { int r = a % m; return r < 0 ? r + m : r; }

}  // namespace se1p
