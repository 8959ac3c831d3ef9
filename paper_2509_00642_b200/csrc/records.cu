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

constexpr int kK1Threads = 512;
constexpr int kRowChunk = 32768;      // records per CTA: 32768 * 2^16 = 2^31 per limb
constexpr int kGuide = 4096;          // score guide table buckets over [0, 1]

__global__ void gather_kernel(const double* __restrict__ h, const double* __restrict__ scores,
                              int64_t n, int n_rows, const uint32_t* __restrict__ idx,
                              double hscale, double* __restrict__ h_sorted,
                              unsigned long long* __restrict__ hfix_sorted,
                              double* __restrict__ s_sorted, uint32_t* __restrict__ perm,
                              uint32_t* __restrict__ bad) {
  uint32_t my_bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t q = idx[i];
    const double hq = h[q];
    const bool ok = hq >= 0.0 && hq <= 1.0;
    my_bad += !ok;
    h_sorted[i] = hq;
    hfix_sorted[i] = (unsigned long long)__dmul_rn(ok ? hq : 0.0, hscale);
    if (perm) perm[i] = q;
    int l = 0;
    for (; l + 8 <= n_rows; l += 8) {      // 8 random gathers in flight per thread
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = scores[(int64_t)(l + j) * n + q];
#pragma unroll
      for (int j = 0; j < 8; ++j) s_sorted[(int64_t)(l + j) * n + i] = v[j];
    }
    for (; l < n_rows; ++l) s_sorted[(int64_t)l * n + i] = scores[(int64_t)l * n + q];
  }
  if (my_bad) atomicAdd(bad, my_bad);
}

// row boundaries: rb[k] = #{h <= u[k-1]} (rb[0] = 0, rb[U+1] = n); rows with
// more than kRowChunk records are split into chunks; item_off = prefix of chunks
__global__ void __launch_bounds__(1024)
row_plan_kernel(const double* __restrict__ hs, int64_t n, const double* __restrict__ thr, int U,
                int64_t* __restrict__ rb, int64_t* __restrict__ item_off,
                uint32_t* __restrict__ guide) {
  __shared__ uint16_t s_g[kGuide + 1];
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
  // g(j) = #{u <= j / kGuide}; guide[j] packs (g(j), g(j+1)): for s in
  // [j/G, (j+1)/G), bs = #{u <= s} lies in [g(j), g(j+1)]
  for (int j = threadIdx.x; j <= kGuide; j += blockDim.x) {
    const double x = (double)j / kGuide;
    int lo = 0, hi = U;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (thr[mid] <= x) lo = mid + 1; else hi = mid; }
    s_g[j] = (uint16_t)lo;
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= kGuide; j += blockDim.x)
    guide[j] = (uint32_t)s_g[j] | ((uint32_t)s_g[j < kGuide ? j + 1 : kGuide] << 16);
  // item_off = exclusive prefix of per-row chunk counts (block-wide, chunked)
  __shared__ int64_t s_carry;
  __shared__ int64_t s_warp[32];
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base <= U; base += blockDim.x) {
    const int k = base + threadIdx.x;
    int64_t v = 0;
    if (k <= U) { const int64_t len = rb[k + 1] - rb[k]; v = len > 0 ? ceil_div(len, kRowChunk) : 0; }
    int64_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t o = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += o;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    const int64_t excl = s_carry + (warp > 0 ? s_warp[warp - 1] : 0) + incl - v;
    if (k <= U) item_off[k] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) item_off[U + 1] = s_carry;
}

// #{u <= s} via the guide table (s in [0, 1]) or binary search otherwise
__device__ __forceinline__ int score_bin(const double* u, int U, const uint32_t* guide, double s) {
  const int jg = __double2int_rz(s * kGuide);
  if ((unsigned)jg <= (unsigned)kGuide && s == s) {   // s in [0, 1] (clip output) and not NaN
    const uint32_t gj = guide[jg];
    int lo = (int)(gj & 0xffffu), hi = (int)(gj >> 16);
    if (hi - lo <= 4) {
      while (lo < hi && u[lo] <= s) ++lo;
      return lo;
    }
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (u[mid] <= s) lo = mid + 1; else hi = mid; }
    return lo;
  }
  return count_less_equal(u, U, s);
}

// grid: (light slots, item slots) -- the models of one chunk are adjacent CTAs,
// so the chunk's hardness is read from HBM once and from L2 by the others.
// Hardness (pre-scaled to fixed point at ingest) is accumulated relative to
// the chunk's smallest value: when the chunk's span fits 32 bits, two 16-bit
// limbs suffice (3 ATOMS per update), else three (4 ATOMS).  Bin arrays use a
// compile-time stride so the limb atomics share one address register.
constexpr int kBinStride = 2048;      // supports up to 2047 distinct thresholds here

template <bool kNarrow>
__global__ void __launch_bounds__(kK1Threads)
row_hist_kernel(const unsigned long long* __restrict__ hf, const double* __restrict__ ss, int64_t n,
                const double* __restrict__ thr, int U, const uint32_t* __restrict__ g_guide,
                const int64_t* __restrict__ rb, const int64_t* __restrict__ item_off,
                const uint8_t* __restrict__ item_narrow, uint32_t* __restrict__ g_cnt,
                unsigned long long* __restrict__ g_hsum, uint8_t* __restrict__ row_scanned) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B1 = U + 1;
  uint32_t* s_bin = reinterpret_cast<uint32_t*>(smem);          // [4][kBinStride]
  double* s_thr = reinterpret_cast<double*>(s_bin + 4 * kBinStride);
  uint32_t* s_guide = reinterpret_cast<uint32_t*>(s_thr + U);
  const int64_t items = item_off[U + 1];
  const int64_t item = blockIdx.y;
  if (item >= items || (item_narrow[item] != 0) != kNarrow) return;
  int lo = 0, hi = U + 1;
  while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (item_off[mid] <= item) lo = mid; else hi = mid - 1; }
  const int k = lo;
  const int64_t chunk = item - item_off[k];
  const int64_t r0 = rb[k] + chunk * kRowChunk;
  const int64_t r1 = min(rb[k + 1], r0 + kRowChunk);
  const bool whole_row = (r0 == rb[k]) && (r1 == rb[k + 1]);
  const int l = blockIdx.x;
  for (int i = threadIdx.x; i < U; i += blockDim.x) s_thr[i] = thr[i];
  for (int i = threadIdx.x; i < 4 * kBinStride; i += blockDim.x) s_bin[i] = 0;
  for (int i = threadIdx.x; i <= kGuide; i += blockDim.x) s_guide[i] = g_guide[i];
  __syncthreads();
  const double* srow = ss + (int64_t)l * n;
  const unsigned long long base = hf[r0];
  constexpr int kU = 4;
  int64_t q = r0 + threadIdx.x;
  for (; q + (kU - 1) * (int64_t)blockDim.x < r1; q += kU * (int64_t)blockDim.x) {
    unsigned long long hv[kU];
    double sv[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) { hv[j] = hf[q + j * blockDim.x]; sv[j] = srow[q + j * blockDim.x]; }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const unsigned long long d = hv[j] - base;
      uint32_t* a = s_bin + score_bin(s_thr, U, s_guide, sv[j]);
      atomicAdd(a, 1u);
      atomicAdd(a + kBinStride, (uint32_t)(d & 0xffffu));
      atomicAdd(a + 2 * kBinStride, (uint32_t)((d >> 16) & 0xffffu));
      if (!kNarrow) atomicAdd(a + 3 * kBinStride, (uint32_t)(d >> 32));
    }
  }
  for (; q < r1; q += blockDim.x) {
    const unsigned long long d = hf[q] - base;
    uint32_t* a = s_bin + score_bin(s_thr, U, s_guide, srow[q]);
    atomicAdd(a, 1u);
    atomicAdd(a + kBinStride, (uint32_t)(d & 0xffffu));
    atomicAdd(a + 2 * kBinStride, (uint32_t)((d >> 16) & 0xffffu));
    if (!kNarrow) atomicAdd(a + 3 * kBinStride, (uint32_t)(d >> 32));
  }
  __syncthreads();
  uint32_t* gc = g_cnt + ((int64_t)l * B1 + k) * B1;
  unsigned long long* gh = g_hsum + ((int64_t)l * B1 + k) * B1;
  auto bin_sum = [&](int i) {
    return (unsigned long long)s_bin[i] * base + (unsigned long long)s_bin[kBinStride + i] +
           ((unsigned long long)s_bin[2 * kBinStride + i] << 16) +
           ((unsigned long long)s_bin[3 * kBinStride + i] << 32);
  };
  if (!whole_row || !row_scanned) {
    for (int i = threadIdx.x; i < B1; i += blockDim.x) {
      const uint32_t c = s_bin[i];
      const unsigned long long v = bin_sum(i);
      if (whole_row) {
        gc[i] = c;
        gh[i] = v;
      } else if (c) {
        atomicAdd(&gc[i], c);
        atomicAdd(&gh[i], v);
      }
    }
    return;
  }
  // whole row: emit the K2 row prefix (along bs) directly -- thread-contiguous
  // segments, block scan of the segment totals, then the segment prefixes
  __shared__ uint32_t ws_c[kK1Threads / 32];
  __shared__ unsigned long long ws_h[kK1Threads / 32];
  const int per = (B1 + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(B1, i0 + per);
  uint32_t tc = 0;
  unsigned long long th = 0;
  for (int i = i0; i < i1; ++i) { tc += s_bin[i]; th += bin_sum(i); }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t ic = tc;
  unsigned long long ih = th;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t oc = __shfl_up_sync(0xffffffffu, ic, off);
    const unsigned long long oh = __shfl_up_sync(0xffffffffu, ih, off);
    if (lane >= off) { ic += oc; ih += oh; }
  }
  if (lane == 31) { ws_c[warp] = ic; ws_h[warp] = ih; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t wc = lane < nw ? ws_c[lane] : 0u;
    unsigned long long wh = lane < nw ? ws_h[lane] : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t oc = __shfl_up_sync(0xffffffffu, wc, off);
      const unsigned long long oh = __shfl_up_sync(0xffffffffu, wh, off);
      if (lane >= off) { wc += oc; wh += oh; }
    }
    if (lane < nw) { ws_c[lane] = wc; ws_h[lane] = wh; }
  }
  __syncthreads();
  uint32_t rc = (warp > 0 ? ws_c[warp - 1] : 0u) + ic - tc;
  unsigned long long rh = (warp > 0 ? ws_h[warp - 1] : 0ull) + ih - th;
  for (int i = i0; i < i1; ++i) {
    rc += s_bin[i];
    rh += bin_sum(i);
    gc[i] = rc;
    gh[i] = rh;
  }
  if (threadIdx.x == 0) row_scanned[(int64_t)l * B1 + k] = 1;
}

// per item: does its hardness span fit 32 bits (narrow) ?
__global__ void item_span_kernel(const unsigned long long* __restrict__ hf, int U,
                                 const int64_t* __restrict__ rb,
                                 const int64_t* __restrict__ item_off, int64_t max_items,
                                 uint8_t* __restrict__ item_narrow) {
  const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= max_items) return;
  if (item >= item_off[U + 1]) { item_narrow[item] = 0; return; }
  int lo = 0, hi = U + 1;
  while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (item_off[mid] <= item) lo = mid; else hi = mid - 1; }
  const int64_t r0 = rb[lo] + (item - item_off[lo]) * kRowChunk;
  const int64_t r1 = min(rb[lo + 1], r0 + kRowChunk);
  item_narrow[item] = hf[r1 - 1] - hf[r0] < (1ull << 32);
}

}  // namespace hadis

using namespace hadis;

extern "C" size_t hadis_records_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return sort_workspace_bytes(n);
}

extern "C" int hadis_records_sort(const double* h, const double* scores, int64_t n, int32_t n_rows,
                                  int32_t hfix_shift, double* h_sorted, uint64_t* hfix_sorted,
                                  double* scores_sorted, uint32_t* perm, uint32_t* bad_records,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  if (!h || n <= 0 || n > 0xffffffffll || n_rows < 0 || (n_rows > 0 && (!scores || !scores_sorted))
      || !h_sorted || !hfix_sorted || !bad_records || !workspace || hfix_shift < 1 ||
      hfix_shift > 48)
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_records_workspace_bytes(n)) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  HADIS_CUDA_TRY(cudaMemsetAsync(bad_records, 0, 4, st));
  const uint32_t* idx = nullptr;
  const int rc = sort_keys(h, nullptr, n, workspace, st, &idx, nullptr);
  if (rc != HADIS_OK) return rc;
  int64_t grid = ceil_div(n, 256);
  if (grid > kNumSMs * 8) grid = kNumSMs * 8;
  gather_kernel<<<(unsigned)grid, 256, 0, st>>>(h, scores, n, n_rows, idx, ldexp(1.0, hfix_shift),
                                                h_sorted, (unsigned long long*)hfix_sorted,
                                                scores_sorted, perm, bad_records);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}

static int64_t k1_max_items(int64_t n, int32_t n_unique) {
  return ceil_div(n, kRowChunk) + n_unique + 1;
}

extern "C" size_t hadis_bin_hist_sorted_workspace_bytes(int64_t n, int32_t n_unique) {
  if (n <= 0 || n_unique <= 0) return 0;
  return (size_t)8 * (2 * (size_t)n_unique + 4) + 4 * (kGuide + 1) +
         (size_t)k1_max_items(n, n_unique) + 256;
}

extern "C" int hadis_bin_hist_sorted(const double* h_sorted, const uint64_t* hfix_sorted,
                                     const double* scores_sorted, int64_t n, int32_t n_light,
                                     const double* thr_unique, int32_t n_unique,
                                     uint32_t* hist_cnt, uint64_t* hist_hsum, uint8_t* row_scanned,
                                     void* workspace, size_t workspace_bytes, void* stream) {
  if (!h_sorted || !hfix_sorted || !scores_sorted || n <= 0 || n > 0xffffffffll || n_light <= 0 ||
      n_unique <= 0 || !thr_unique || !hist_cnt || !hist_hsum || !workspace || n_light > 65535)
    return HADIS_ERR_ARG;
  if (n_unique + 1 > kBinStride) return HADIS_ERR_UNSUPPORTED;
  if (workspace_bytes < hadis_bin_hist_sorted_workspace_bytes(n, n_unique))
    return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t B1 = (int64_t)n_unique + 1;
  int64_t* rb = (int64_t*)workspace;
  int64_t* item_off = rb + (n_unique + 2);
  uint32_t* guide = (uint32_t*)(item_off + (n_unique + 2));
  uint8_t* item_narrow = (uint8_t*)(guide + (kGuide + 1));
  const int64_t bins = B1 * B1 * n_light;
  const int64_t max_items = k1_max_items(n, n_unique);
  if (max_items > 65535) return HADIS_ERR_UNSUPPORTED;
  HADIS_CUDA_TRY(cudaMemsetAsync(hist_cnt, 0, bins * sizeof(uint32_t), st));
  HADIS_CUDA_TRY(cudaMemsetAsync(hist_hsum, 0, bins * sizeof(uint64_t), st));
  if (row_scanned) HADIS_CUDA_TRY(cudaMemsetAsync(row_scanned, 0, (size_t)B1 * n_light, st));
  row_plan_kernel<<<1, 1024, 0, st>>>(h_sorted, n, thr_unique, n_unique, rb, item_off, guide);
  item_span_kernel<<<(unsigned)ceil_div(max_items, 256), 256, 0, st>>>(
      (const unsigned long long*)hfix_sorted, n_unique, rb, item_off, max_items, item_narrow);
  HADIS_LAUNCH_CHECK();
  const size_t smem = (size_t)4 * kBinStride * 4 + (size_t)n_unique * 8 + 4 * (kGuide + 1) + 16;
  if (smem > 227 * 1024) return HADIS_ERR_UNSUPPORTED;
  HADIS_CUDA_TRY(cudaFuncSetAttribute(row_hist_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  HADIS_CUDA_TRY(cudaFuncSetAttribute(row_hist_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid((unsigned)n_light, (unsigned)max_items);
  row_hist_kernel<true><<<grid, kK1Threads, smem, st>>>(
      (const unsigned long long*)hfix_sorted, scores_sorted, n, thr_unique, n_unique, guide, rb,
      item_off, item_narrow, hist_cnt, (unsigned long long*)hist_hsum, row_scanned);
  row_hist_kernel<false><<<grid, kK1Threads, smem, st>>>(
      (const unsigned long long*)hfix_sorted, scores_sorted, n, thr_unique, n_unique, guide, rb,
      item_off, item_narrow, hist_cnt, (unsigned long long*)hist_hsum, row_scanned);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(4);
  return HADIS_OK;
}
