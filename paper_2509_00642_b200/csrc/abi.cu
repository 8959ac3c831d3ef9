// ABI housekeeping: version, status strings, last CUDA error.
#include <cstring>

#include "common.cuh"

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

static thread_local char g_last_cuda_error[256] = "";
static std::atomic<long long> g_launches{0};

void hadis_count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

extern "C" int64_t hadis_kernel_launches(void) { return g_launches.load(); }

void hadis_set_cuda_error(cudaError_t e) {
  std::strncpy(g_last_cuda_error, cudaGetErrorString(e), sizeof(g_last_cuda_error) - 1);
}

cudaError_t hadis_ensure_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& g = granted[{dev, func}];
  if (bytes <= g) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) g = bytes;
  return e;
}

extern "C" int hadis_abi_version(void) { return HADIS_ABI_VERSION; }

extern "C" const char* hadis_last_cuda_error(void) { return g_last_cuda_error; }

extern "C" const char* hadis_status_string(int status) {
  switch (status) {
    case HADIS_OK: return "ok";
    case HADIS_ERR_ARG: return "invalid argument";
    case HADIS_ERR_RECORDS: return "records: hardness must be finite and within [0, 1]";
    case HADIS_ERR_CAPACITY: return "capacity exceeded";
    case HADIS_ERR_CUDA: return "cuda error";
    case HADIS_ERR_NO_ROWS: return "fallback: no serveable rows";
    case HADIS_ERR_NEG_DEMAND: return "solve: negative demand";
    case HADIS_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}
