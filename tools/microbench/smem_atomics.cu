// Pure shared-memory atomic throughput on B200 (no global traffic in the loop):
// how many ATOMS lanes per clock per SM for u32 add / u64 add (CAS loop) over
// random addresses in a 1025-bin (or larger) per-CTA histogram.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t xs(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

template <int MODE>
__global__ void k(int iters, int nbins, unsigned long long* out) {
  extern __shared__ unsigned long long sm[];
  uint32_t* s32 = (uint32_t*)sm;
  for (int i = threadIdx.x; i < nbins * 2; i += blockDim.x) s32[i] = 0;
  __syncthreads();
  uint32_t r = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
    r = xs(r);
    const uint32_t b = r & (nbins - 1);
    if (MODE == 0) atomicAdd(&s32[b], 1u);
    if (MODE == 1) { atomicAdd(&s32[b], 1u); atomicAdd(&s32[nbins + b], r >> 8); }
    if (MODE == 2) atomicAdd(&sm[b], (unsigned long long)(r >> 4));
    if (MODE == 3) { atomicAdd(&s32[b], 1u); atomicAdd(&s32[nbins + b], r >> 8); atomicAdd(&s32[(b ^ 1)], r & 255); }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s32[0];
}

int main() {
  unsigned long long* out; cudaMalloc(&out, 148 * 64 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096;
  for (int nb : {1024, 4096, 16384}) {
    for (int mode = 0; mode < 4; ++mode) {
      for (int bpsm : {1, 2, 4}) {
        size_t smem = (size_t)nb * 8;
        auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int grid = 148 * bpsm, thr = 1024 / bpsm < 256 ? 256 : 1024 / bpsm;
        f<<<grid, thr, smem>>>(8, nb, out);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        f<<<grid, thr, smem>>>(iters, nb, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double upd = (double)grid * thr * iters;
        double per_clk_sm = upd / (ms * 1e-3) / 148 / 1.965e9;
        printf("bins %6d mode %d (%s) blk/SM %d thr %4d: %7.3f ms  %8.1f G upd/s  %6.2f upd/clk/SM  %s\n",
               nb, mode, mode == 0 ? "u32" : mode == 1 ? "2xu32" : mode == 2 ? "u64cas" : "3xu32",
               bpsm, thr, ms, upd / ms / 1e6, per_clk_sm, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
