// Throughput of the f64 mma.sync shapes on sm_100a (m8n8k4, m16n8k4, m16n8k8, m16n8k16).
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void kern(double* out, int iters) {
  double a[8], b[4], c[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + j * 1e-6 + threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 0.5;
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      if (SHAPE == 3)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
void run(const char* name, double fma_per_inst, double* out, int nsm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 16, 32}) {
    int grid = nsm, iters = 2000;
    kern<SHAPE><<<grid, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    kern<SHAPE><<<grid, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * fma_per_inst * 8 * (double)iters * grid * warps;
    printf("%s warps/SM=%d: %.2f TFLOP/s (%.1f SM-cycles/inst at 1.965 GHz)\n", name, warps, flops / ms * 1e-9,
           ms * 1e-3 * 1.965e9 / (8.0 * iters * warps));
  }
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  run<0>("m8n8k4  ", 256, out, 148);
  run<1>("m16n8k4 ", 512, out, 148);
  run<2>("m16n8k8 ", 1024, out, 148);
  run<3>("m16n8k16", 2048, out, 148);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
