// Verify the register layouts assumed for mma.sync m16n8k8 / m16n8k16 f64 on sm_100a:
//   A (16 x K): a[2j] = A[gid][tig + 4j], a[2j+1] = A[gid + 8][tig + 4j]
//   B (K x 8):  b[j]  = B[tig + 4j][gid]
//   C (16 x 8): c0,c1 = C[gid][2 tig + {0,1}], c2,c3 = C[gid + 8][2 tig + {0,1}]
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

template <int K>
__global__ void k(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
  for (int j = 0; j < K / 4; ++j) {
    a[2 * j] = A[gid * K + tig + 4 * j];
    a[2 * j + 1] = A[(gid + 8) * K + tig + 4 * j];
    b[j] = B[(tig + 4 * j) * 8 + gid];
  }
  if (K == 8)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  if (K == 16)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4 % (K / 2)]), "d"(a[5 % (K / 2)]), "d"(a[6 % (K / 2)]), "d"(a[7 % (K / 2)]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2 % (K / 4)]), "d"(b[3 % (K / 4)]));
  C[gid * 8 + 2 * tig] = c[0];
  C[gid * 8 + 2 * tig + 1] = c[1];
  C[(gid + 8) * 8 + 2 * tig] = c[2];
  C[(gid + 8) * 8 + 2 * tig + 1] = c[3];
}

template <int K>
int check() {
  double hA[16 * K], hB[K * 8], hC[128], ref[128];
  for (int i = 0; i < 16 * K; ++i) hA[i] = std::sin(1.0 + i * 0.37);
  for (int i = 0; i < K * 8; ++i) hB[i] = std::cos(0.3 + i * 0.71);
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int kk = 0; kk < K; ++kk) s += hA[m * K + kk] * hB[kk * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&C, sizeof hC);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  k<K><<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, sizeof hC, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("m16n8k%d layout max err %.3e (%s)\n", K, err, err < 1e-12 ? "OK" : "MISMATCH");
  return err < 1e-12 ? 0 : 1;
}

int main() { return check<8>() + check<16>(); }
