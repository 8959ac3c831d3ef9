// Record store layout + K1 (bin + 2-D histogram) from hardness-sorted records.
//
// Ingest (once per record set, hadis_records_sort): records are ordered by
// hardness (ties by original index, so the layout is deterministic) and the
// score rows are gathered into the same order.  The original-order arrays
// stay with the caller for the numpy-exact fidelity emulation.
//
// Then, for ANY threshold grid, bh(q) = #{u < h[q]} is constant on a
// contiguous run of sorted records (a "row"), so K1 needs no global atomics:
// one CTA owns (row k, light model l, record range) and accumulates the row's
// bs-histogram (counts + fixed-point hardness) in shared memory with 32-bit
// ATOMS, then writes it out -- plain stores when it owns the whole row.
// Bins are (count, three 16-bit hardness limbs) with hardness in <= 48-bit
// fixed point; a CTA sees at most kRowChunk records, so no limb can overflow.
#include <cmath>

#include "common.cuh"

namespace hadis {

constexpr int kK1Threads = 256;
constexpr int kRowChunk = 32768;      // records per CTA: 32768 * 2^16 = 2^31 per limb
constexpr int kGuide = 4096;          // score guide table buckets over [0, 1]

__global__ void gather_kernel(const double* __restrict__ h, const double* __restrict__ scores,
                              int64_t n, int n_rows, const uint32_t* __restrict__ idx,
                              double* __restrict__ h_sorted, double* __restrict__ s_sorted,
                              uint32_t* __restrict__ perm, uint32_t* __restrict__ bad) {
  uint32_t my_bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t q = idx[i];
    const double hq = h[q];
    my_bad += !(hq >= 0.0 && hq <= 1.0);
    h_sorted[i] = hq;
    if (perm) perm[i] = q;
    for (int l = 0; l < n_rows; ++l) s_sorted[(int64_t)l * n + i] = scores[(int64_t)l * n + q];
  }
  if (my_bad) atomicAdd(bad, my_bad);
}

// row boundaries: rb[k] = #{h <= u[k-1]} (rb[0] = 0, rb[U+1] = n); rows with
// more than kRowChunk records are split into chunks; item_off = prefix of chunks
__global__ void __launch_bounds__(1024)
row_plan_kernel(const double* __restrict__ hs, int64_t n, const double* __restrict__ thr, int U,
                int64_t* __restrict__ rb, int64_t* __restrict__ item_off,
                uint16_t* __restrict__ guide) {
  for (int k = threadIdx.x; k <= U + 1; k += blockDim.x) {
    int64_t pos;
    if (k == 0) pos = 0;
    else if (k == U + 1) pos = n;
    else {                                  // upper_bound(u[k-1]) over sorted hardness
      const double u = thr[k - 1];
      int64_t lo = 0, hi = n;
      while (lo < hi) { const int64_t mid = (lo + hi) >> 1; if (hs[mid] <= u) lo = mid + 1; else hi = mid; }
      pos = lo;
    }
    rb[k] = pos;
  }
  // guide[j] = #{u <= j / kGuide}: search for bs = #{u <= s} starts there
  for (int j = threadIdx.x; j <= kGuide; j += blockDim.x) {
    const double x = (double)j / kGuide;
    int lo = 0, hi = U;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (thr[mid] <= x) lo = mid + 1; else hi = mid; }
    guide[j] = (uint16_t)lo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int k = 0; k <= U; ++k) {
      item_off[k] = acc;
      const int64_t len = rb[k + 1] - rb[k];
      acc += len > 0 ? ceil_div(len, kRowChunk) : 0;
    }
    item_off[U + 1] = acc;
  }
}

// #{u <= s} via the guide table (s in [0, 1]) or binary search otherwise
__device__ __forceinline__ int score_bin(const double* u, int U, const uint16_t* guide, double s) {
  if (s >= 0.0 && s <= 1.0) {
    const int j = (int)(s * kGuide);
    int lo = guide[j], hi = guide[j < kGuide ? j + 1 : kGuide];
    if (hi - lo <= 4) {
      while (lo < hi && u[lo] <= s) ++lo;
      return lo;
    }
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (u[mid] <= s) lo = mid + 1; else hi = mid; }
    return lo;
  }
  return count_less_equal(u, U, s);
}

// grid: (item slots, light slots); one CTA = one chunk of one row for one model
__global__ void __launch_bounds__(kK1Threads)
row_hist_kernel(const double* __restrict__ hs, const double* __restrict__ ss, int64_t n,
                const double* __restrict__ thr, int U, const uint16_t* __restrict__ g_guide,
                const int64_t* __restrict__ rb, const int64_t* __restrict__ item_off,
                double hscale, uint32_t* __restrict__ g_cnt, unsigned long long* __restrict__ g_hsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B1 = U + 1;
  double* s_thr = reinterpret_cast<double*>(smem);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_thr + U);
  uint32_t* s_l0 = s_cnt + B1;
  uint32_t* s_l1 = s_l0 + B1;
  uint32_t* s_l2 = s_l1 + B1;
  uint16_t* s_guide = reinterpret_cast<uint16_t*>(s_l2 + B1);
  const int64_t items = item_off[U + 1];
  const int64_t item = blockIdx.x;
  if (item >= items) return;
  // row k = last row with item_off[k] <= item
  int lo = 0, hi = U + 1;
  while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (item_off[mid] <= item) lo = mid; else hi = mid - 1; }
  const int k = lo;
  const int64_t chunk = item - item_off[k];
  const int64_t r0 = rb[k] + chunk * kRowChunk;
  const int64_t r1 = min(rb[k + 1], r0 + kRowChunk);
  const bool whole_row = (r0 == rb[k]) && (r1 == rb[k + 1]);
  const int l = blockIdx.y;
  for (int i = threadIdx.x; i < U; i += blockDim.x) s_thr[i] = thr[i];
  for (int i = threadIdx.x; i < B1; i += blockDim.x) {
    s_cnt[i] = 0; s_l0[i] = 0; s_l1[i] = 0; s_l2[i] = 0;
  }
  for (int i = threadIdx.x; i <= kGuide; i += blockDim.x) s_guide[i] = g_guide[i];
  __syncthreads();
  const double* srow = ss + (int64_t)l * n;
  for (int64_t q = r0 + threadIdx.x; q < r1; q += blockDim.x) {
    const double hq = hs[q];
    const double sq = srow[q];
    const unsigned long long hf =
        (unsigned long long)__dmul_rn(hq >= 0.0 && hq <= 1.0 ? hq : 0.0, hscale);
    const int b = score_bin(s_thr, U, s_guide, sq);
    atomicAdd(&s_cnt[b], 1u);
    atomicAdd(&s_l0[b], (uint32_t)(hf & 0xffffu));
    atomicAdd(&s_l1[b], (uint32_t)((hf >> 16) & 0xffffu));
    atomicAdd(&s_l2[b], (uint32_t)(hf >> 32));
  }
  __syncthreads();
  uint32_t* gc = g_cnt + ((int64_t)l * B1 + k) * B1;
  unsigned long long* gh = g_hsum + ((int64_t)l * B1 + k) * B1;
  for (int i = threadIdx.x; i < B1; i += blockDim.x) {
    const uint32_t c = s_cnt[i];
    const unsigned long long v = (unsigned long long)s_l0[i] +
                                 ((unsigned long long)s_l1[i] << 16) +
                                 ((unsigned long long)s_l2[i] << 32);
    if (whole_row) {
      gc[i] = c;
      gh[i] = v;
    } else if (c) {
      atomicAdd(&gc[i], c);
      atomicAdd(&gh[i], v);
    }
  }
}

}  // namespace hadis

using namespace hadis;

extern "C" size_t hadis_records_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return sort_workspace_bytes(n);
}

extern "C" int hadis_records_sort(const double* h, const double* scores, int64_t n, int32_t n_rows,
                                  double* h_sorted, double* scores_sorted, uint32_t* perm,
                                  uint32_t* bad_records, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (!h || n <= 0 || n > 0xffffffffll || n_rows < 0 || (n_rows > 0 && (!scores || !scores_sorted))
      || !h_sorted || !bad_records || !workspace)
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_records_workspace_bytes(n)) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  HADIS_CUDA_TRY(cudaMemsetAsync(bad_records, 0, 4, st));
  const uint32_t* idx = nullptr;
  const int rc = sort_keys(h, nullptr, n, workspace, st, &idx, nullptr);
  if (rc != HADIS_OK) return rc;
  int64_t grid = ceil_div(n, 256);
  if (grid > kNumSMs * 8) grid = kNumSMs * 8;
  gather_kernel<<<(unsigned)grid, 256, 0, st>>>(h, scores, n, n_rows, idx, h_sorted, scores_sorted,
                                                perm, bad_records);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}

extern "C" size_t hadis_bin_hist_sorted_workspace_bytes(int32_t n_unique) {
  if (n_unique <= 0) return 0;
  return (size_t)8 * (2 * (size_t)n_unique + 4) + 2 * (kGuide + 1) + 256;
}

extern "C" int hadis_bin_hist_sorted(const double* h_sorted, const double* scores_sorted, int64_t n,
                                     int32_t n_light, const double* thr_unique, int32_t n_unique,
                                     int32_t hfix_shift, uint32_t* hist_cnt, uint64_t* hist_hsum,
                                     void* workspace, size_t workspace_bytes, void* stream) {
  if (!h_sorted || !scores_sorted || n <= 0 || n > 0xffffffffll || n_light <= 0 ||
      n_unique <= 0 || !thr_unique || !hist_cnt || !hist_hsum || !workspace || hfix_shift < 1 ||
      hfix_shift > 48 || n_light > 65535)
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_bin_hist_sorted_workspace_bytes(n_unique)) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t B1 = (int64_t)n_unique + 1;
  int64_t* rb = (int64_t*)workspace;
  int64_t* item_off = rb + (n_unique + 2);
  uint16_t* guide = (uint16_t*)(item_off + (n_unique + 2));
  const int64_t bins = B1 * B1 * n_light;
  HADIS_CUDA_TRY(cudaMemsetAsync(hist_cnt, 0, bins * sizeof(uint32_t), st));
  HADIS_CUDA_TRY(cudaMemsetAsync(hist_hsum, 0, bins * sizeof(uint64_t), st));
  row_plan_kernel<<<1, 1024, 0, st>>>(h_sorted, n, thr_unique, n_unique, rb, item_off, guide);
  HADIS_LAUNCH_CHECK();
  const size_t smem = (size_t)n_unique * 8 + (size_t)B1 * 16 + 2 * (kGuide + 1) + 16;
  if (smem > 227 * 1024) return HADIS_ERR_UNSUPPORTED;
  if (smem > 48 * 1024)
    HADIS_CUDA_TRY(cudaFuncSetAttribute(row_hist_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t max_items = ceil_div(n, kRowChunk) + B1;
  row_hist_kernel<<<dim3((unsigned)max_items, (unsigned)n_light), kK1Threads, smem, st>>>(
      h_sorted, scores_sorted, n, thr_unique, n_unique, guide, rb, item_off,
      ldexp(1.0, hfix_shift), hist_cnt, (unsigned long long*)hist_hsum);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(2);
  return HADIS_OK;
}
