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
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when `func` needs more
// than it was last granted on the current device: the call can cost
// milliseconds of host time, and eager pipelines launch ~40 kernels per build.
cudaError_t hadis_ensure_smem(const void* func, size_t bytes);
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

// ---------------------------------------------------------------------------
// Blackwell async-copy plumbing: 1-D bulk copies (TMA engine, UBLKCP) into
// shared memory completing on mbarriers (full / empty ring barriers).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// make mbarrier inits visible to the async proxy (the bulk-copy engine)
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// the same on a precomputed shared-window address
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// global -> shared bulk copy of `bytes` (multiple of 16, both ends 16-byte
// aligned), completing `bytes` transactions on `bar`; streamed data: L2
// evict-first
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// bulk L2 prefetch (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// named barrier over `threads` threads (a subset of the CTA, e.g. consumer warps)
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// prune.cu: ascending sort of (k1, k2, index) keys (k2 may be null)
size_t sort_workspace_bytes(int64_t n);
int sort_keys(const double* k1, const double* k2, int64_t n, void* workspace, cudaStream_t st,
              const uint32_t** sorted_idx, const unsigned long long** sorted_k2);

}  // namespace hadis
