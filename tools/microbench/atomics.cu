// Microbenchmark: scattered histogram updates on B200 (sm_100a).
// Informs the K1 (bin + histogram) design: global L2 atomics vs shared-memory
// privatised atomics vs plain streaming reads, at the bin counts of the
// BASELINE configs ((K+1)^2 = 4225, 66049, 263169, 1050625).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// streaming read baseline: sum of doubles
__global__ void k_stream(const double2* __restrict__ a, size_t n2, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = a[i]; acc += v.x + v.y;
  }
  if (acc == 12345.678) *out = acc;
}

// global: count u32 + sum u64 per bin, random bins
__global__ void k_global2(const double* __restrict__ s, size_t n, uint32_t nbins,
                          uint32_t* cnt, unsigned long long* sum) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double v = s[i];
    uint32_t b = hash32((uint32_t)i ^ (uint32_t)(v * 1e6)) % nbins;
    atomicAdd(cnt + b, 1u);
    atomicAdd(sum + b, (unsigned long long)(v * 1099511627776.0));
  }
}
// global: single packed u64 per bin
__global__ void k_global1(const double* __restrict__ s, size_t n, uint32_t nbins, unsigned long long* sum) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double v = s[i];
    uint32_t b = hash32((uint32_t)i ^ (uint32_t)(v * 1e6)) % nbins;
    atomicAdd(sum + b, (unsigned long long)(v * 1099511627776.0) + (1ull << 44));
  }
}
// smem privatised: count u32 + sum u64, flush at end
__global__ void k_smem2(const double* __restrict__ s, size_t n, uint32_t nbins,
                        uint32_t* cnt, unsigned long long* sum) {
  extern __shared__ unsigned long long sm[];
  unsigned long long* ssum = sm;
  uint32_t* scnt = (uint32_t*)(sm + nbins);
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) { ssum[b] = 0; scnt[b] = 0; }
  __syncthreads();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double v = s[i];
    uint32_t b = hash32((uint32_t)i ^ (uint32_t)(v * 1e6)) % nbins;
    atomicAdd(scnt + b, 1u);
    atomicAdd(ssum + b, (unsigned long long)(v * 1099511627776.0));
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
    if (scnt[b]) { atomicAdd(cnt + b, scnt[b]); atomicAdd(sum + b, ssum[b]); }
  }
}
// smem privatised, count only u32
__global__ void k_smem1(const double* __restrict__ s, size_t n, uint32_t nbins, uint32_t* cnt) {
  extern __shared__ unsigned long long sm[];
  uint32_t* scnt = (uint32_t*)sm;
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) scnt[b] = 0;
  __syncthreads();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double v = s[i];
    uint32_t b = hash32((uint32_t)i ^ (uint32_t)(v * 1e6)) % nbins;
    atomicAdd(scnt + b, 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) if (scnt[b]) atomicAdd(cnt + b, scnt[b]);
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d L2 %d MB smem/block optin %zu KB clock %d MHz memclk %d MHz bus %d\n",
         p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin >> 10,
         p.clockRate / 1000, p.memoryClockRate / 1000, p.memoryBusWidth);
  const size_t n = 150ull * 1000 * 1000;  // c4: 10M records x 15 light models
  double* s; CK(cudaMalloc(&s, n * 8));
  std::vector<double> hs(1 << 20);
  for (size_t i = 0; i < hs.size(); i++) hs[i] = (double)((i * 2654435761u) % 1000003) / 1000003.0;
  for (size_t off = 0; off < n; off += hs.size()) {
    size_t c = std::min(hs.size(), n - off);
    CK(cudaMemcpy(s + off, hs.data(), c * 8, cudaMemcpyHostToDevice));
  }
  uint32_t maxbins = 1050625 * 4;
  uint32_t* cnt; unsigned long long* sum; double* out;
  CK(cudaMalloc(&cnt, maxbins * 4)); CK(cudaMalloc(&sum, maxbins * 8)); CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  auto tm = [&](auto launch, const char* name, double bytes_or_updates, bool isbytes) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    cudaError_t err = cudaGetLastError();
    if (isbytes) printf("%-44s %8.3f ms  %8.1f GB/s %s\n", name, ms, bytes_or_updates / ms / 1e6, cudaGetErrorString(err));
    else printf("%-44s %8.3f ms  %8.2f Gupd/s %s\n", name, ms, bytes_or_updates / ms / 1e6, cudaGetErrorString(err));
  };
  tm([&] { k_stream<<<sms * 8, 256>>>((const double2*)s, n / 2, out); }, "stream read 1.2 GB", n * 8.0, true);
  uint32_t bins_list[] = {1025, 4225, 66049, 263169, 1050625, 4202500};
  for (uint32_t nb : bins_list) {
    char nm[128];
    cudaMemset(cnt, 0, maxbins * 4); cudaMemset(sum, 0, maxbins * 8);
    snprintf(nm, sizeof nm, "global u32+u64 bins=%u", nb);
    tm([&] { k_global2<<<sms * 8, 256>>>(s, n, nb, cnt, sum); }, nm, (double)n, false);
    snprintf(nm, sizeof nm, "global packed u64 bins=%u", nb);
    tm([&] { k_global1<<<sms * 8, 256>>>(s, n, nb, sum); }, nm, (double)n, false);
    size_t sm2 = (size_t)nb * 12, sm1 = (size_t)nb * 4;
    if (sm2 <= 200 * 1024) {
      cudaFuncSetAttribute(k_smem2, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      int per = (int)((220 * 1024) / sm2); if (per > 8) per = 8; if (per < 1) per = 1;
      snprintf(nm, sizeof nm, "smem u32+u64 bins=%u (blk/SM~%d)", nb, per);
      tm([&] { k_smem2<<<sms * per, 512, sm2>>>(s, n, nb, cnt, sum); }, nm, (double)n, false);
    }
    if (sm1 <= 200 * 1024) {
      cudaFuncSetAttribute(k_smem1, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      int per = (int)((220 * 1024) / sm1); if (per > 8) per = 8; if (per < 1) per = 1;
      snprintf(nm, sizeof nm, "smem u32 bins=%u (blk/SM~%d)", nb, per);
      tm([&] { k_smem1<<<sms * per, 512, sm1>>>(s, n, nb, cnt); }, nm, (double)n, false);
    }
  }
  return 0;
}
