// common.cuh -- shared device/host definitions of libse1p (the CUDA path).
// No code here is shared with oracle/ (the two are independent by construction).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

namespace se1p {

constexpr double kPi = 3.141592653589793238462643383279502884;

struct Status {
  int code = 0;
  std::string msg;
};

// Error helpers: library entry points translate these into se1p_status codes.
struct Error {
  int code;
  std::string msg;
};

#define SE1P_CUDA_TRY(expr)                                                           \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw ::se1p::Error{6, std::string(#expr) + ": " + cudaGetErrorString(_e)};      \
  } while (0)

#define SE1P_LAUNCH_CHECK()                                                           \
  do {                                                                                \
    cudaError_t _e = cudaGetLastError();                                              \
    if (_e != cudaSuccess)                                                            \
      throw ::se1p::Error{6, std::string("kernel launch: ") + cudaGetErrorString(_e)}; \
    ::se1p::count_launch();                                                           \
  } while (0)

void count_launch();

// Device memory of the library (workspaces, plans, tables): cudaMalloc/cudaFree, or the hook
// installed by se1p_set_allocator (include/se1p.h).  dev_alloc throws Error{5} on failure.
void* dev_alloc(size_t bytes);
void dev_free(void* p);
template <typename T>
inline void dev_alloc(T*& p, size_t count) { p = static_cast<T*>(dev_alloc(sizeof(T) * count)); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Floor of a double as int64 (particles are in range; z is folded first).
__device__ __forceinline__ int64_t ifloor(double v) { return (int64_t)floor(v); }

}  // namespace se1p
