// FP64 throughput microbenchmark on sm_100a: DFMA (CUDA cores) vs DMMA (mma.sync f64).
// Used once to choose the gridding/gather kernel design; not part of the product path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + j * 1e-6;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 0.5;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bs : {256, 512}) for (int bpsm : {2, 4, 8}) {
    int grid = p.multiProcessorCount * bpsm, iters = 2000;
    dfma_kernel<<<grid, bs>>>(out, 10, 0.999, 1e-3);
    cudaEventRecord(e0); dfma_kernel<<<grid, bs>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * grid * bs;
    printf("DFMA bs=%d grid=%d: %.3f ms  %.2f TFLOP/s\n", bs, grid, ms, flops / ms * 1e-9);
  }
  for (int bs : {128, 256}) for (int bpsm : {2, 4, 8}) {
    int grid = p.multiProcessorCount * bpsm, iters = 500;
    dmma_m8n8k4_kernel<<<grid, bs>>>(out, 10);
    cudaEventRecord(e0); dmma_m8n8k4_kernel<<<grid, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * 16 * (double)iters * grid * (bs / 32);
    printf("DMMA m8n8k4 bs=%d grid=%d: %.3f ms  %.2f TFLOP/s\n", bs, grid, ms, flops / ms * 1e-9);
  }
  for (int bs : {128, 256}) for (int bpsm : {2, 4}) {
    int grid = p.multiProcessorCount * bpsm, iters = 200;
    dmma_m16n8k16_kernel<<<grid, bs>>>(out, 10);
    cudaEventRecord(e0); dmma_m16n8k16_kernel<<<grid, bs>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 4 * 4 * (double)iters * grid * (bs / 32);
    printf("DMMA m16n8k16 bs=%d grid=%d: %.3f ms  %.2f TFLOP/s\n", bs, grid, ms, flops / ms * 1e-9);
  }
  cudaError_t err = cudaGetLastError(); printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
