// The sweep kernels' gridding k-step in isolation: per k-step 3 m16n8k8 f64 MMAs (6 accumulators
// x 2 K halves = 12 SASS DMMA.8x8x4) with operands from shared memory, A formed by 4 DMULs.
// Variants: 0 DMMA only (register operands), 1 + shared-memory B, 2 + shared-memory A factors and
// the DMULs, 3 = 2 with the next k-step's operands loaded before the MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kstep kstep.cu && ./kstep
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[4], double b0, double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0), "d"(b1));
}

template <int V>
__global__ void kern(double* out, int iters) {
  __shared__ double rows[96 * 56];
  for (int i = threadIdx.x; i < 96 * 56; i += blockDim.x) rows[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3, w = threadIdx.x >> 5;
  double c[3][4] = {};
  double a[4] = {1.0, 1.0, 1.0, 1.0};
  double b[3][2] = {{0.5, 0.5}, {0.5, 0.5}, {0.5, 0.5}};
  int e0 = (w * 8 + tg) % 96, e1 = (w * 8 + tg + 4) % 96;
  for (int it = 0; it < iters; ++it) {
    if (V >= 1) {
      const double* r0 = rows + e0 * 56;
      const double* r1 = rows + e1 * 56;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        b[j][0] = r0[32 + 8 * j + g];
        b[j][1] = r1[32 + 8 * j + g];
      }
      if (V >= 2) {
        const double y0 = r0[16 + g], y1 = r1[16 + g];
        a[0] = r0[g >> 2] * y0;
        a[1] = r0[(g >> 2) + 2] * y0;
        a[2] = r1[g >> 2] * y1;
        a[3] = r1[(g >> 2) + 2] * y1;
      }
      e0 = (e0 + 8) % 96;
      e1 = (e1 + 8) % 96;
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) dmma(c[j], a, b[j][0], b[j][1]);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 3; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(const char* name, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 16, 24}) {
    const int grid = 148, iters = 4000;
    kern<V><<<grid, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    kern<V><<<grid, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 3 * 1024 * (double)iters * grid * warps;
    printf("%s warps/SM=%2d: %.2f TFLOP/s\n", name, warps, flops / ms * 1e-9);
  }
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  run<0>("dmma only       ", out);
  run<1>("+ smem B        ", out);
  run<2>("+ smem A, DMUL  ", out);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
