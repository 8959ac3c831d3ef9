// Generic latency/quality Pareto prune (catalog.py:171-192) on the GPU.
//
// pareto_prune sorts rows by (latency, quality, original index) and keeps a
// row iff its quality is strictly below every quality before it.  Here:
//   1. keys -> (order_key(lat), order_key(qual), idx)   (total order, -0.0 == 0.0)
//   2. sort: CTA-local bitonic sort of 2048-key tiles in shared memory, then
//      log2(n / 2048) merge passes where every key finds its output slot by a
//      binary search in the partner run (keys are unique, so ranks are exact)
//   3. exclusive prefix-min of quality in sorted order; keep iff qual < prefix
//   4. order-preserving compaction of kept original indices
#include <cmath>

#include "common.cuh"

namespace hadis {

constexpr int kTile = 2048;
constexpr int kPruneThreads = 1024;

struct Key3 {
  unsigned long long a, b;
  uint32_t i;
};

__device__ __forceinline__ bool key_less(unsigned long long a1, unsigned long long b1, uint32_t i1,
                                         unsigned long long a2, unsigned long long b2, uint32_t i2) {
  return a1 < a2 || (a1 == a2 && (b1 < b2 || (b1 == b2 && i1 < i2)));
}

__global__ void __launch_bounds__(kPruneThreads)
tile_sort_kernel(const double* __restrict__ lat, const double* __restrict__ qual, int64_t n,
                 unsigned long long* __restrict__ ka, unsigned long long* __restrict__ kb,
                 uint32_t* __restrict__ ki) {
  __shared__ unsigned long long sa[kTile];
  __shared__ unsigned long long sb[kTile];
  __shared__ uint32_t si[kTile];
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int j = threadIdx.x; j < kTile; j += blockDim.x) {
    const int64_t g = base + j;
    if (g < n) {
      sa[j] = order_key(lat[g]);
      sb[j] = qual ? order_key(qual[g]) : 0ull;
      si[j] = (uint32_t)g;
    } else {
      sa[j] = ~0ull; sb[j] = ~0ull; si[j] = 0xffffffffu;
    }
  }
  __syncthreads();
  for (int size = 2; size <= kTile; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = key_less(sa[j], sb[j], si[j], sa[i], sb[i], si[i]);
          if (gt == up) {
            unsigned long long t = sa[i]; sa[i] = sa[j]; sa[j] = t;
            t = sb[i]; sb[i] = sb[j]; sb[j] = t;
            uint32_t u = si[i]; si[i] = si[j]; si[j] = u;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = threadIdx.x; j < kTile; j += blockDim.x) {
    const int64_t g = base + j;
    if (g < n) { ka[g] = sa[j]; kb[g] = sb[j]; ki[g] = si[j]; }
  }
}

// merge runs of length `run` pairwise: each element's output rank is its own
// position plus its rank in the partner run
__global__ void merge_pass_kernel(const unsigned long long* __restrict__ ia,
                                  const unsigned long long* __restrict__ ib,
                                  const uint32_t* __restrict__ ii, int64_t n, int64_t run,
                                  unsigned long long* __restrict__ oa,
                                  unsigned long long* __restrict__ ob, uint32_t* __restrict__ oi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += stride) {
    const int64_t pair_base = (g / (2 * run)) * (2 * run);
    const bool left = (g - pair_base) < run;
    const int64_t own0 = left ? pair_base : pair_base + run;
    const int64_t oth0 = left ? pair_base + run : pair_base;
    const int64_t oth1 = min(n, oth0 + run);
    const int64_t own_pos = g - own0;
    const unsigned long long a = ia[g], b = ib[g];
    const uint32_t i = ii[g];
    int64_t lo = oth0, hi = oth1 > oth0 ? oth1 : oth0;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (key_less(ia[mid], ib[mid], ii[mid], a, b, i)) lo = mid + 1; else hi = mid;
    }
    const int64_t at = pair_base + own_pos + (lo - oth0);
    oa[at] = a; ob[at] = b; oi[at] = i;
  }
}

// single CTA: prefix-min keep flags, then order-preserving compaction
__global__ void __launch_bounds__(kPruneThreads)
keep_compact_kernel(const unsigned long long* __restrict__ kb, const uint32_t* __restrict__ ki,
                    int64_t n, int64_t* __restrict__ out_idx, int64_t* __restrict__ out_count) {
  __shared__ unsigned long long part_min[kPruneThreads];
  __shared__ unsigned long long part_cnt[kPruneThreads];
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per;
  const int64_t hi = min(n, lo + per);
  unsigned long long m = ~0ull;
  for (int64_t i = lo; i < hi; ++i) m = min(m, kb[i]);
  part_min[threadIdx.x] = m;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    unsigned long long o = threadIdx.x >= off ? part_min[threadIdx.x - off] : ~0ull;
    __syncthreads();
    part_min[threadIdx.x] = min(part_min[threadIdx.x], o);
    __syncthreads();
  }
  // quality order keys: strict "<" on doubles == strict "<" on keys (-0.0 folded)
  unsigned long long run = threadIdx.x > 0 ? part_min[threadIdx.x - 1] : ~0ull;
  unsigned long long kept = 0;
  for (int64_t i = lo; i < hi; ++i) {
    if (kb[i] < run) { ++kept; run = kb[i]; }
  }
  part_cnt[threadIdx.x] = kept;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    unsigned long long o = threadIdx.x >= off ? part_cnt[threadIdx.x - off] : 0ull;
    __syncthreads();
    part_cnt[threadIdx.x] += o;
    __syncthreads();
  }
  unsigned long long at = part_cnt[threadIdx.x] - kept;
  run = threadIdx.x > 0 ? part_min[threadIdx.x - 1] : ~0ull;
  for (int64_t i = lo; i < hi; ++i) {
    if (kb[i] < run) { out_idx[at++] = ki[i]; run = kb[i]; }
  }
  if (threadIdx.x == blockDim.x - 1) out_count[0] = (int64_t)part_cnt[blockDim.x - 1];
}

// Sort n (k1, k2, index) keys ascending (k2 may be null); ws must hold
// sort_workspace_bytes(n).  *sorted_idx / *sorted_k2 point into ws on return.
size_t sort_workspace_bytes(int64_t n) { return 2 * (((size_t)n * 20 + 255) & ~(size_t)255); }

int sort_keys(const double* k1, const double* k2, int64_t n, void* workspace, cudaStream_t st,
              const uint32_t** sorted_idx, const unsigned long long** sorted_k2) {
  char* ws = (char*)workspace;
  unsigned long long* a0 = (unsigned long long*)ws;
  unsigned long long* b0 = a0 + n;
  uint32_t* i0 = (uint32_t*)(b0 + n);
  unsigned long long* a1 = (unsigned long long*)(ws + (((size_t)n * 20 + 255) & ~(size_t)255));
  unsigned long long* b1 = a1 + n;
  uint32_t* i1 = (uint32_t*)(b1 + n);
  const int64_t tiles = ceil_div(n, kTile);
  tile_sort_kernel<<<(unsigned)tiles, kPruneThreads, 0, st>>>(k1, k2, n, a0, b0, i0);
  HADIS_LAUNCH_CHECK();
  int launches = 1;
  bool in0 = true;
  for (int64_t run = kTile; run < n; run <<= 1) {
    int64_t grid = ceil_div(n, 256);
    if (grid > kNumSMs * 8) grid = kNumSMs * 8;
    if (in0) merge_pass_kernel<<<(unsigned)grid, 256, 0, st>>>(a0, b0, i0, n, run, a1, b1, i1);
    else merge_pass_kernel<<<(unsigned)grid, 256, 0, st>>>(a1, b1, i1, n, run, a0, b0, i0);
    HADIS_LAUNCH_CHECK();
    ++launches;
    in0 = !in0;
  }
  hadis_count_launches(launches);
  *sorted_idx = in0 ? i0 : i1;
  if (sorted_k2) *sorted_k2 = in0 ? b0 : b1;
  return HADIS_OK;
}

}  // namespace hadis

using namespace hadis;

extern "C" size_t hadis_pareto_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return sort_workspace_bytes(n);
}

extern "C" int hadis_pareto_prune(const double* lat, const double* qual, int64_t n,
                                  int64_t* out_idx, int64_t* out_count, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (n <= 0 || n > 0xffffffffll || !lat || !qual || !out_idx || !out_count || !workspace)
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_pareto_workspace_bytes(n)) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t* idx = nullptr;
  const unsigned long long* kb = nullptr;
  const int rc = sort_keys(lat, qual, n, workspace, st, &idx, &kb);
  if (rc != HADIS_OK) return rc;
  keep_compact_kernel<<<1, kPruneThreads, 0, st>>>(kb, idx, n, out_idx, out_count);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}
