// Do DFMA (CUDA-core FP64) and DMMA (FP64 tensor) share execution resources on sm_100a?
// Half the warps run DMMA, half run DFMA; compare the combined rate with each alone.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(double* out, int iters, int mode) {   // mode 0: all DMMA, 1: all DFMA, 2: half/half
  const int w = threadIdx.x >> 5;
  const bool do_mma = (mode == 0) || (mode == 2 && (w & 1) == 0);
  double s = 0;
  if (do_mma) {
    double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 1.0, b = 0.5;
    double c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  } else {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], 0.999, 1e-3);
    }
    for (int j = 0; j < 8; ++j) s += x[j];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  // per DMMA warp-iteration: 4 x 512 FMA ; per DFMA warp-iteration: 128 x 32 FMA = 4096 FMA
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<148, 512>>>(out, 10, mode);
    cudaEventRecord(e0);
    mix<<<148, 512>>>(out, iters, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mma_w = mode == 0 ? 16 : (mode == 2 ? 8 : 0), fma_w = mode == 1 ? 16 : (mode == 2 ? 8 : 0);
    double fmas = 148.0 * iters * (mma_w * 2048 + fma_w * 4096);
    printf("mode %d (%s): %.3f ms, %.1f TFLOP/s combined\n", mode, mode == 0 ? "DMMA only" : mode == 1 ? "DFMA only" : "half/half",
           ms, 2 * fmas / ms * 1e-9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
