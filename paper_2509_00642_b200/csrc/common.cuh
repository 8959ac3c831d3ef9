// Shared helpers for the HADIS B200 kernels (sm_100a).
//
// Every floating-point expression that must reproduce a reference (Python /
// numpy) value bit for bit is written with explicit round-to-nearest
// intrinsics (__dmul_rn / __dadd_rn / __ddiv_rn) AND the library is built
// with -fmad=false, so no multiply-add is ever contracted into an FMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hadis_b200.h"

#define HADIS_CUDA_TRY(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) { hadis_set_cuda_error(_e); return HADIS_ERR_CUDA; } \
  } while (0)

#define HADIS_LAUNCH_CHECK() HADIS_CUDA_TRY(cudaGetLastError())

void hadis_set_cuda_error(cudaError_t e);
void hadis_count_launches(int k);  // bookkeeping for hadis_kernel_launches()

namespace hadis {

constexpr int kNumSMs = 148;  // B200; grids are sized as multiples of this

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Order-preserving map double -> uint64 (total order; -0.0 folded onto +0.0
// so it compares equal to 0.0 exactly like Python floats do).
__host__ __device__ inline uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = (uint64_t)__double_as_longlong(x);
#else
  __builtin_memcpy(&b, &x, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__host__ __device__ inline double from_order_key(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
#ifdef __CUDA_ARCH__
  x = __longlong_as_double((long long)b);
#else
  __builtin_memcpy(&x, &b, 8);
#endif
  return x;
}

// #{u[i] < x} over sorted unique u[0..n) ; NaN -> 0 (h > theta is never true)
__device__ __forceinline__ int count_less(const double* u, int n, double x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (u[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// #{u[i] <= x} over sorted unique u ; NaN -> n (s < tau is never true)
__device__ __forceinline__ int count_less_equal(const double* u, int n, double x) {
  if (x != x) return n;
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (u[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// prune.cu: ascending sort of (k1, k2, index) keys (k2 may be null)
size_t sort_workspace_bytes(int64_t n);
int sort_keys(const double* k1, const double* k2, int64_t n, void* workspace, cudaStream_t st,
              const uint32_t** sorted_idx, const unsigned long long** sorted_k2);

}  // namespace hadis
