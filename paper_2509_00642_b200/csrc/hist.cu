// K1 (bin + 2-D histogram) and K2 (2-D prefix scan) of the cascade profiler.
//
// Reference semantics (pkg/src/cascadesim/profiler.py):
//   bypass(q, theta) = h[q] > theta                       (:138)
//   reject(q, tau)   = not bypass and score_light[q] < tau (:149)
// With u = the sorted distinct threshold values (size U) we bin
//   bh(q) = #{u < h[q]}          -> bypass at theta = u[k]  <=>  bh > k
//   bs(q) = #{u <= s[q]}         -> s < tau = u[t]          <=>  bs <= t
// so every grid cell (k, t) is a union of histogram bins and all counts and
// hardness sums follow from 2-D prefix sums of an (U+1) x (U+1) histogram per
// light model.  Integer accumulation (counts u32, hardness in fixed point
// 2^-shift as u64) is exact and order independent, hence deterministic.
#include <algorithm>

#include "common.cuh"

namespace hadis {

constexpr int kHistThreads = 512;
constexpr int kMaxSmemThr = 8192;  // thresholds staged in shared memory up to this

// Shared-memory privatised variant: all light models' histograms fit on chip.
__global__ void __launch_bounds__(kHistThreads)
bin_hist_smem_kernel(const double* __restrict__ h, const double* __restrict__ scores, int64_t n,
                     int n_light, const double* __restrict__ thr, int U, double hscale,
                     uint32_t* __restrict__ g_cnt, unsigned long long* __restrict__ g_hsum,
                     uint32_t* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B1 = U + 1;
  const int bins = B1 * B1 * n_light;
  unsigned long long* s_hsum = reinterpret_cast<unsigned long long*>(smem);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_hsum + bins);
  double* s_thr = reinterpret_cast<double*>(s_cnt + ((bins + 1) & ~1));
  for (int i = threadIdx.x; i < bins; i += blockDim.x) { s_hsum[i] = 0; s_cnt[i] = 0; }
  for (int i = threadIdx.x; i < U; i += blockDim.x) s_thr[i] = thr[i];
  __syncthreads();

  uint32_t my_bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const double hq = h[q];
    const bool ok = hq >= 0.0 && hq <= 1.0;
    my_bad += !ok;
    const int bh = count_less(s_thr, U, hq);
    const unsigned long long hf = (unsigned long long)__dmul_rn(ok ? hq : 0.0, hscale);
    for (int l = 0; l < n_light; ++l) {
      const int bs = count_less_equal(s_thr, U, scores[(int64_t)l * n + q]);
      const int bin = (l * B1 + bh) * B1 + bs;
      atomicAdd(&s_cnt[bin], 1u);
      atomicAdd(&s_hsum[bin], hf);
    }
  }
  if (my_bad) atomicAdd(bad, my_bad);
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x) {
    if (s_cnt[i]) {
      atomicAdd(&g_cnt[i], s_cnt[i]);
      atomicAdd(&g_hsum[i], s_hsum[i]);
    }
  }
}

// Global-memory variant for large grids: L2-resident histograms, integer REDs.
__global__ void __launch_bounds__(kHistThreads)
bin_hist_global_kernel(const double* __restrict__ h, const double* __restrict__ scores, int64_t n,
                       int n_light, const double* __restrict__ thr, int U, double hscale,
                       uint32_t* __restrict__ g_cnt, unsigned long long* __restrict__ g_hsum,
                       uint32_t* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_thr = reinterpret_cast<double*>(smem);
  const bool staged = U <= kMaxSmemThr;
  if (staged) {
    for (int i = threadIdx.x; i < U; i += blockDim.x) s_thr[i] = thr[i];
    __syncthreads();
  }
  const double* u = staged ? s_thr : thr;
  const int64_t B1 = U + 1;
  uint32_t my_bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const double hq = h[q];
    const bool ok = hq >= 0.0 && hq <= 1.0;
    my_bad += !ok;
    const int bh = count_less(u, U, hq);
    const unsigned long long hf = (unsigned long long)__dmul_rn(ok ? hq : 0.0, hscale);
    for (int l = 0; l < n_light; ++l) {
      const int bs = count_less_equal(u, U, scores[(int64_t)l * n + q]);
      const int64_t bin = ((int64_t)l * B1 + bh) * B1 + bs;
      atomicAdd(&g_cnt[bin], 1u);
      atomicAdd(&g_hsum[bin], hf);
    }
  }
  if (my_bad) atomicAdd(bad, my_bad);
}

// K2a: inclusive prefix along bs (the contiguous axis): one warp per row.
__global__ void scan_rows_kernel(uint32_t* __restrict__ cnt, unsigned long long* __restrict__ hs,
                                 int64_t rows, int B1, const uint8_t* __restrict__ done) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= rows || (done && done[row])) return;
  uint32_t* c = cnt + row * B1;
  unsigned long long* s = hs + row * B1;
  uint32_t carry_c = 0;
  unsigned long long carry_s = 0;
  for (int base = 0; base < B1; base += 32) {
    const int i = base + lane;
    uint32_t vc = i < B1 ? c[i] : 0u;
    unsigned long long vs = i < B1 ? s[i] : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      uint32_t oc = __shfl_up_sync(0xffffffffu, vc, off);
      unsigned long long os = __shfl_up_sync(0xffffffffu, vs, off);
      if (lane >= off) { vc += oc; vs += os; }
    }
    vc += carry_c;
    vs += carry_s;
    if (i < B1) { c[i] = vc; s[i] = vs; }
    carry_c = __shfl_sync(0xffffffffu, vc, 31);
    carry_s = __shfl_sync(0xffffffffu, vs, 31);
  }
}

// K2b: inclusive prefix along bh.  Task = (32-column tile, light slot); each
// of the CTA's warps takes a contiguous band of rows (lanes = columns, so every
// access is a coalesced 128/256-byte row segment), sums its band, the bands'
// totals are scanned in shared memory, then each warp rewrites its band with
// the carried-in prefix.  Persistent CTAs walk the tasks in order, so the
// tables being scanned at any moment (CTAs x 1025 rows x 32 columns x 12 B,
// ~58 MB at c4) stay L2-resident and the second read of a band hits L2: the
// pass moves one read + one write of the tables from DRAM (a one-shot grid
// of all 495 tasks keeps the whole 189 MB alive and re-reads it from DRAM).
#ifndef HADIS_K2_WARPS
#define HADIS_K2_WARPS 32
#endif
#ifndef HADIS_K2_UNROLL
#define HADIS_K2_UNROLL 8
#endif
#ifndef HADIS_K2_CPS
#define HADIS_K2_CPS 1
#endif
constexpr int kColWarps = HADIS_K2_WARPS;
constexpr int kColU = HADIS_K2_UNROLL;

__global__ void __launch_bounds__(kColWarps * 32)
scan_cols_kernel(uint32_t* __restrict__ cnt, unsigned long long* __restrict__ hs, int n_light,
                 int B1) {
  __shared__ uint32_t s_c[kColWarps][32];
  __shared__ unsigned long long s_h[kColWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tiles = (B1 + 31) / 32;
  const int band = (B1 + kColWarps - 1) / kColWarps;
  const int k0 = min(B1, warp * band), k1 = min(B1, k0 + band);
  for (int task = blockIdx.x; task < tiles * n_light; task += gridDim.x) {
    const int t = (task % tiles) * 32 + lane;
    const int64_t l = task / tiles;
    uint32_t* c = cnt + l * B1 * (int64_t)B1 + t;
    unsigned long long* h = hs + l * B1 * (int64_t)B1 + t;
    const bool col = t < B1;
    uint32_t sc = 0;
    unsigned long long sh = 0;
    if (col) {
      int k = k0;
      for (; k + kColU <= k1; k += kColU) {
        uint32_t vc[kColU];
        unsigned long long vh[kColU];
#pragma unroll
        for (int j = 0; j < kColU; ++j) { vc[j] = c[(int64_t)(k + j) * B1]; vh[j] = h[(int64_t)(k + j) * B1]; }
#pragma unroll
        for (int j = 0; j < kColU; ++j) { sc += vc[j]; sh += vh[j]; }
      }
      for (; k < k1; ++k) { sc += c[(int64_t)k * B1]; sh += h[(int64_t)k * B1]; }
    }
    s_c[warp][lane] = sc;
    s_h[warp][lane] = sh;
    __syncthreads();
    uint32_t rc = 0;
    unsigned long long rh = 0;
    for (int w = 0; w < warp; ++w) { rc += s_c[w][lane]; rh += s_h[w][lane]; }
    if (col) {
      int k = k0;
      for (; k + kColU <= k1; k += kColU) {
        uint32_t vc[kColU];
        unsigned long long vh[kColU];
#pragma unroll
        for (int j = 0; j < kColU; ++j) { vc[j] = c[(int64_t)(k + j) * B1]; vh[j] = h[(int64_t)(k + j) * B1]; }
#pragma unroll
        for (int j = 0; j < kColU; ++j) {
          rc += vc[j];
          rh += vh[j];
          c[(int64_t)(k + j) * B1] = rc;
          h[(int64_t)(k + j) * B1] = rh;
        }
      }
      for (; k < k1; ++k) {
        rc += c[(int64_t)k * B1];
        rh += h[(int64_t)k * B1];
        c[(int64_t)k * B1] = rc;
        h[(int64_t)k * B1] = rh;
      }
    }
    __syncthreads();                                 // s_c / s_h reused by the next task
  }
}

}  // namespace hadis

using namespace hadis;

extern "C" int hadis_hfix_shift(int64_t n) {
  if (n <= 0) return 62;
  int bits = 0;
  while ((n >> bits) != 0) ++bits;
  int shift = 63 - bits;
  return shift > 48 ? 48 : shift;   // <= 48-bit hardness fixed point (3 x 16-bit K1 limbs)
}

extern "C" int hadis_bin_hist(const double* h, const double* scores, int64_t n, int32_t n_light,
                              const double* thr_unique, int32_t n_unique, int32_t hfix_shift,
                              uint32_t* hist_cnt, uint64_t* hist_hsum, uint32_t* bad_records,
                              void* stream) {
  if (n <= 0 || n > 0xffffffffll || n_light <= 0 || n_unique <= 0 || !h || !scores ||
      !thr_unique || !hist_cnt || !hist_hsum || !bad_records || hfix_shift < 1 || hfix_shift > 62)
    return HADIS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t B1 = (int64_t)n_unique + 1;
  const int64_t bins = B1 * B1 * n_light;
  HADIS_CUDA_TRY(cudaMemsetAsync(hist_cnt, 0, bins * sizeof(uint32_t), st));
  HADIS_CUDA_TRY(cudaMemsetAsync(hist_hsum, 0, bins * sizeof(uint64_t), st));
  HADIS_CUDA_TRY(cudaMemsetAsync(bad_records, 0, sizeof(uint32_t), st));
  const double hscale = ldexp(1.0, hfix_shift);
  const size_t smem_priv = (size_t)bins * 12 + 8 + (size_t)n_unique * 8;
  const int64_t blocks_needed = ceil_div(n, kHistThreads);
  if (smem_priv <= 160 * 1024) {
    HADIS_CUDA_TRY(hadis_ensure_smem((const void*)bin_hist_smem_kernel, (size_t)200 * 1024));
    const int per_sm = smem_priv <= 48 * 1024 ? 4 : (smem_priv <= 100 * 1024 ? 2 : 1);
    int64_t grid = (int64_t)kNumSMs * per_sm;
    if (grid > blocks_needed) grid = blocks_needed;
    bin_hist_smem_kernel<<<(unsigned)grid, kHistThreads, smem_priv, st>>>(
        h, scores, n, n_light, thr_unique, n_unique, hscale, hist_cnt,
        (unsigned long long*)hist_hsum, bad_records);
  } else {
    const size_t smem = n_unique <= kMaxSmemThr ? (size_t)n_unique * 8 : 0;
    // opt in unconditionally: static shared memory counts against the 48 KB default
    HADIS_CUDA_TRY(hadis_ensure_smem((const void*)bin_hist_global_kernel, (size_t)smem));
    int64_t grid = (int64_t)kNumSMs * 4;
    if (grid > blocks_needed) grid = blocks_needed;
    bin_hist_global_kernel<<<(unsigned)grid, kHistThreads, smem, st>>>(
        h, scores, n, n_light, thr_unique, n_unique, hscale, hist_cnt,
        (unsigned long long*)hist_hsum, bad_records);
  }
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}

extern "C" int hadis_hist_scan(uint32_t* hist_cnt, uint64_t* hist_hsum, int32_t n_light,
                               int32_t n_unique, const uint8_t* row_scanned, void* stream) {
  if (!hist_cnt || !hist_hsum || n_light <= 0 || n_unique <= 0) return HADIS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int B1 = n_unique + 1;
  const int64_t rows = (int64_t)n_light * B1;
  scan_rows_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0, st>>>(
      hist_cnt, (unsigned long long*)hist_hsum, rows, B1, row_scanned);
  HADIS_LAUNCH_CHECK();
  const int64_t tasks = ceil_div((int64_t)B1, 32) * n_light;
  const int64_t cgrid = std::min<int64_t>(tasks, (int64_t)kNumSMs * HADIS_K2_CPS);
  scan_cols_kernel<<<(unsigned)cgrid, kColWarps * 32, 0, st>>>(
      hist_cnt, (unsigned long long*)hist_hsum, n_light, B1);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(2);
  return HADIS_OK;
}
