// Row-bucketed record store + K1 (2-D histogram), per threshold grid.
//
// Reference semantics (pkg/src/cascadesim/profiler.py:138, 145-150):
//   bypass(q, theta) = h[q] > theta,  reject(q, tau) = not bypass and s[q] < tau
// With u = the sorted distinct thresholds (U values):
//   bh(q) = #{u < h[q]}   (the theta-row of record q)
//   bs(q) = #{u <= s[q]}  (its tau-bin for one light model)
//
// B0 setup    guide tables (h: #{u < x}, s: #{u <= x}) over [0, 1] in 4096
//             buckets, zeroed row counters.
// B1 count    records -> bh, CTA-private shared-memory row histogram, one
//             global atomic per non-empty row per CTA.  Validates h in [0, 1].
// B2 plan     row offsets (exclusive scan), per-row write cursors, K1 items
//             (row chunks of <= kRowChunk records), per-row fixed-point bounds.
// B3 scatter  the HBM-bound pass: every record array is read once (128-bit
//             loads); per tile, records are counting-sorted by bh in shared
//             memory (ATOMS ranks + one global cursor reservation per row),
//             then written row-bucketed and staged so consecutive threads
//             store consecutive addresses: hfix = floor(h * 2^shift) as u64
//             and the tau-bins bs (u16) of four light models per 8-byte
//             store (the scores themselves are never needed again).  Order
//             within a row is irrelevant: every K1 sum is an integer sum.
// K1 row_hist one CTA per (row chunk, model quad) accumulates the row's four
//             bs-histograms (count + 16-bit hardness limbs relative to the
//             row's fixed-point lower bound) with shared-memory ATOMS and
//             stores the rows, already prefix-summed along bs when it owns
//             the whole row (K2's row pass fused).
// The original-order arrays stay with the caller for the numpy-exact
// fidelity emulation, which depends on the reference's summation order.
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace hadis {

constexpr int kGuide = 4096;          // guide buckets over [0, 1]
constexpr int kMaxBins = 2048;        // U + 1 <= kMaxBins (u16 bins)
constexpr int kRowChunk = 32768;      // records per K1 CTA: 2^15 * 2^16 < 2^31 per limb
#ifndef HADIS_K1_THREADS
#define HADIS_K1_THREADS 384   // 3 CTAs per SM (56 registers): 300 vs 308 us at 512 x 2, 256: 321, 1024: 411
#endif
constexpr int kK1Threads = HADIS_K1_THREADS;
constexpr int kBkThreads = 1024;      // scatter CTA (512 x 2/SM and 4096-record tiles: slower;
constexpr int kBkTile = 8192;         // records per scatter tile   L2 bulk prefetch ahead: slower)
constexpr int kBkPer = kBkTile / kBkThreads;   // records per thread per tile (even)
constexpr int kCountThreads = 512;

// B3 (TMA path) geometry: 15 consumer warps + 1 producer warp (512 threads:
// 128 registers for 16 records per consumer), 7680-record tiles (~7.5
// records per row and tile at U = 1024: the write-out's row runs, and so its
// sector efficiency, grow with the tile), ring slots of 8 records per
// consumer (two per array tile).  Measured at c4 (us): 31 warps x 4 records
// 369, x 8 363; 15 x 16 359; 2-3 CTAs per SM with proportionally smaller
// tiles 465-576 (per-tile row costs); 4 ring slots or L2 bulk prefetch: no gain.
#ifndef HADIS_TMA_CWARPS
#define HADIS_TMA_CWARPS 15
#endif
#ifndef HADIS_TMA_PER
#define HADIS_TMA_PER 16
#endif
#ifndef HADIS_TMA_CHUNK_PER
#define HADIS_TMA_CHUNK_PER 8
#endif
#ifndef HADIS_TMA_SLOTS
#define HADIS_TMA_SLOTS 3
#endif
constexpr int kTmaConsumers = 32 * HADIS_TMA_CWARPS;
constexpr int kTmaThreads = kTmaConsumers + 32;        // + the producer warp
constexpr int kTmaPer = HADIS_TMA_PER;                 // records per consumer per tile
constexpr int kTmaChunkPer = HADIS_TMA_CHUNK_PER;      // records per consumer per ring slot (even)
constexpr int kTmaChunks = kTmaPer / kTmaChunkPer;     // ring slots per array tile
constexpr int kTmaChunk = kTmaChunkPer * kTmaConsumers;   // records per ring slot
constexpr int kTmaTile = kTmaPer * kTmaConsumers;      // records per tile (max)
constexpr int kTmaSlots = HADIS_TMA_SLOTS;
constexpr int kTmaBar = 1;                             // named barrier id (consumers)
static_assert(kTmaPer % kTmaChunkPer == 0 && kTmaChunkPer % 2 == 0, "pairs per chunk");
#ifndef HADIS_B3_WOBATCH
#define HADIS_B3_WOBATCH 2
#endif
constexpr int kTmaRowsPer = (kMaxBins + kTmaConsumers - 1) / kTmaConsumers;   // rows per consumer (max)

// Row plan (the `row_plan` buffer shared by B0..B3 and K1), offsets in bytes.
struct RowPlan {
  uint32_t* row_cnt;     // [kMaxBins]     B1 counts
  uint32_t* cursor;      // [kMaxBins]     B3 write cursors
  int64_t* row_off;      // [kMaxBins + 1] row start offsets (row_off[U+1] = n)
  int64_t* item_off;     // [kMaxBins + 1] first K1 item of each row
  uint64_t* row_base;    // [kMaxBins]     fixed-point lower bound of the row's hfix
  uint8_t* row_narrow;   // [kMaxBins]     hfix span of the row < 2^32
  uint32_t* guide_lt;    // [kGuide + 1]
  uint32_t* guide_le;    // [kGuide + 1]
  uint32_t* bad;         // [1]
  uint32_t* sparse;      // [1] nonzero: some guide bucket holds > 2 thresholds
  uint32_t* nonuniform;  // [1] nonzero: thresholds are not exactly i / (U - 1)
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// tau-bin store: light models in quads, bs[quad][record][4] (uint16), so one
// 8-byte store / load moves a record's bins of four models
constexpr int kQuad = 4;
__host__ __device__ inline int64_t n_quads(int n_light) { return (n_light + kQuad - 1) / kQuad; }
// records per quad row, rounded up to even: every quad row starts 16-byte
// aligned, so K1's two-record (uint4) loads stay aligned for odd n too
__host__ __device__ inline int64_t quad_stride(int64_t n) { return (n + 1) & ~(int64_t)1; }

__host__ __device__ inline RowPlan row_plan_at(void* base) {
  unsigned char* p = (unsigned char*)base;
  RowPlan r;
  size_t o = 0;
  r.row_cnt = (uint32_t*)(p + o);     o += align256(4 * kMaxBins);
  r.cursor = (uint32_t*)(p + o);      o += align256(4 * kMaxBins);
  r.row_off = (int64_t*)(p + o);      o += align256(8 * (kMaxBins + 1));
  r.item_off = (int64_t*)(p + o);     o += align256(8 * (kMaxBins + 1));
  r.row_base = (uint64_t*)(p + o);    o += align256(8 * kMaxBins);
  r.row_narrow = (uint8_t*)(p + o);   o += align256(kMaxBins);
  r.guide_lt = (uint32_t*)(p + o);    o += align256(4 * (kGuide + 1));
  r.guide_le = (uint32_t*)(p + o);    o += align256(4 * (kGuide + 1));
  r.bad = (uint32_t*)(p + o);         o += align256(4);
  r.sparse = (uint32_t*)(p + o);      o += align256(4);
  r.nonuniform = (uint32_t*)(p + o);  o += align256(4);
  return r;
}

static size_t row_plan_size() {
  return align256(4 * kMaxBins) * 2 + align256(8 * (kMaxBins + 1)) * 2 + align256(8 * kMaxBins) +
         align256(kMaxBins) + align256(4 * (kGuide + 1)) * 2 + align256(4) * 3;
}

// #{u < x} (kLE = false) or #{u <= x} (kLE = true) over sorted unique u, with
// a guide table g(j) = #{u op j/G} packed as (g(j), g(j+1)): for x in
// [j/G, (j+1)/G) the answer lies in [g(j), g(j+1)].  x*G is exact (G = 2^12).
template <bool kLE>
__device__ __forceinline__ int guided_bin(const double* u, int U, const uint32_t* guide, double x);

// Branch-free variant when every guide bucket holds at most two thresholds
// (rp.sparse == 0): u must be padded with two +inf entries (u[U], u[U+1]).
template <bool kLE>
__device__ __forceinline__ int guided_bin_dense(const double* u, int U, const uint32_t* guide,
                                                double x) {
  if (x >= 0.0 && x <= 1.0) {
    const int b = (int)(guide[__double2int_rz(x * kGuide)] & 0xffffu);
    const double u0 = u[b], u1 = u[b + 1];
    return b + (kLE ? (u0 <= x) + (u1 <= x) : (u0 < x) + (u1 < x));
  }
  return kLE ? count_less_equal(u, U, x) : count_less(u, U, x);
}

// Uniform grid u[i] = i / (U - 1) (rp.nonuniform == 0): g = trunc(x (U - 1)) is
// within one of the answer, so two independent compares finish it
// (u[g - 1] <= x always holds; u padded with +inf).
// Away from a grid point (fractional part of x (U - 1) in (1e-9, 1 - 1e-9),
// far beyond the ~1e-13 rounding of x (U - 1) and of u[g] = g / (U - 1)) the
// answer is g + 1 for both strict and non-strict counts, with no table read.
template <bool kLE>
__device__ __forceinline__ int uniform_bin(const double* u, int U, double x) {
  if (x >= 0.0 && x <= 1.0) {
    const double y = x * (double)(U - 1);
    const int g = min(__double2int_rz(y), U - 1);
    const double fr = y - (double)g;
    if (fr > 1e-9 && fr < 1.0 - 1e-9) return g + 1;
    const double u0 = u[g], u1 = u[g + 1];
    return g + (kLE ? (u0 <= x) + (u1 <= x) : (u0 < x) + (u1 < x));
  }
  return kLE ? count_less_equal(u, U, x) : count_less(u, U, x);
}

// the cheapest exact binning the plan allows: 0 uniform, 1 dense guide, 2 general
template <bool kLE>
__device__ __forceinline__ int plan_bin(int mode, const double* u, int U, const uint32_t* guide,
                                        double x) {
  return mode == 0 ? uniform_bin<kLE>(u, U, x)
                   : (mode == 1 ? guided_bin_dense<kLE>(u, U, guide, x) : guided_bin<kLE>(u, U, guide, x));
}

template <bool kLE>
__device__ __forceinline__ int guided_bin(const double* u, int U, const uint32_t* guide, double x) {
  if (x >= 0.0 && x <= 1.0) {
    const int jg = __double2int_rz(x * kGuide);
    const uint32_t gj = guide[jg];
    int lo = (int)(gj & 0xffffu), hi = (int)(gj >> 16);
    if (hi - lo <= 4) {
      while (lo < hi && (kLE ? u[lo] <= x : u[lo] < x)) ++lo;
      return lo;
    }
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (kLE ? u[mid] <= x : u[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
  }
  return kLE ? count_less_equal(u, U, x) : count_less(u, U, x);
}

// B0: guides (one thread per bucket) + zero the counters
__global__ void bucket_setup_kernel(const double* __restrict__ thr, int U, RowPlan rp) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < kMaxBins) rp.row_cnt[j] = 0;
  if (j < U && (U < 2 || thr[j] != (double)j / (double)(U - 1))) atomicOr(rp.nonuniform, 1u);
  if (j > kGuide + 1) return;
  auto cnt = [&](double x, bool le) {
    int lo = 0, hi = U;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (le ? thr[mid] <= x : thr[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  if (j <= kGuide) {
    const double x0 = (double)j / kGuide;
    const double x1 = (double)(j < kGuide ? j + 1 : kGuide) / kGuide;
    const int a0 = cnt(x0, false), a1 = cnt(x1, false), e0 = cnt(x0, true), e1 = cnt(x1, true);
    rp.guide_lt[j] = (uint32_t)a0 | ((uint32_t)a1 << 16);
    rp.guide_le[j] = (uint32_t)e0 | ((uint32_t)e1 << 16);
    if (a1 - a0 > 2 || e1 - e0 > 2) atomicOr(rp.sparse, 1u);
  }
}

// B1: row counts
__global__ void __launch_bounds__(kCountThreads)
bucket_count_kernel(const double* __restrict__ h, int64_t n, const double* __restrict__ thr, int U,
                    RowPlan rp) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem);             // [kMaxBins]
  uint32_t* s_guide = s_cnt + kMaxBins;                            // [kGuide + 1]
  double* s_thr = reinterpret_cast<double*>(s_guide + kGuide + 2); // [U]
  for (int i = threadIdx.x; i <= U; i += blockDim.x) s_cnt[i] = 0;
  for (int i = threadIdx.x; i <= kGuide; i += blockDim.x) s_guide[i] = rp.guide_lt[i];
  for (int i = threadIdx.x; i < U + 2; i += blockDim.x) s_thr[i] = i < U ? thr[i] : INFINITY;
  __syncthreads();
  const int mode = *rp.nonuniform == 0 ? 0 : (*rp.sparse == 0 ? 1 : 2);
  uint32_t my_bad = 0;
  const int64_t n2 = n >> 1;
  const double2* h2 = reinterpret_cast<const double2*>(h);
  const bool vec = (reinterpret_cast<uintptr_t>(h) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto one = [&](double x) {
    my_bad += !(x >= 0.0 && x <= 1.0);
    atomicAdd(&s_cnt[plan_bin<false>(mode, s_thr, U, s_guide, x)], 1u);
  };
  if (vec) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {    // four 16-byte loads in flight
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = h2[i + u * stride];
#pragma unroll
      for (int u = 0; u < 4; ++u) { one(v[u].x); one(v[u].y); }
    }
    for (; i < n2; i += stride) {
      const double2 v = h2[i];
      one(v.x);
      one(v.y);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) one(h[n - 1]);
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) one(h[i]);
  }
  if (my_bad) atomicAdd(rp.bad, my_bad);
  __syncthreads();
  for (int i = threadIdx.x; i <= U; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&rp.row_cnt[i], s_cnt[i]);
}

// block-wide exclusive scan of one int64 per thread (blockDim.x <= 1024)
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* s_warp, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
  const int64_t excl = (warp > 0 ? s_warp[warp - 1] : 0) + incl - v;
  *total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return excl;
}

// B2: row offsets, cursors, K1 items and fixed-point row bounds (one CTA of 1024)
__global__ void __launch_bounds__(1024)
bucket_plan_kernel(const double* __restrict__ thr, int U, double hscale, RowPlan rp) {
  __shared__ int64_t s_warp[32];
  __shared__ int64_t s_carry[2];
  if (threadIdx.x == 0) { s_carry[0] = 0; s_carry[1] = 0; }
  __syncthreads();
  for (int base = 0; base <= U; base += blockDim.x) {
    const int k = base + threadIdx.x;
    const int64_t c = k <= U ? (int64_t)rp.row_cnt[k] : 0;
    const int64_t items = c > 0 ? ceil_div(c, kRowChunk) : 0;
    int64_t tot_c, tot_i;
    const int64_t ec = block_excl_scan(c, s_warp, &tot_c);
    const int64_t ei = block_excl_scan(items, s_warp, &tot_i);
    if (k <= U) {
      const int64_t off = s_carry[0] + ec;
      rp.row_off[k] = off;
      rp.cursor[k] = (uint32_t)off;
      rp.item_off[k] = s_carry[1] + ei;
      // h in (u[k-1], u[k]] (row 0: [0, u[0]], row U: (u[U-1], 1]) -> hfix bounds
      const double lo_h = k == 0 ? 0.0 : fmin(fmax(thr[k - 1], 0.0), 1.0);
      const double hi_h = k == U ? 1.0 : fmin(fmax(thr[k], 0.0), 1.0);
      const uint64_t lo = (uint64_t)__dmul_rn(lo_h, hscale);
      const uint64_t hi = (uint64_t)__dmul_rn(fmax(hi_h, lo_h), hscale);
      rp.row_base[k] = lo;
      rp.row_narrow[k] = (hi - lo) < (1ull << 32);
    }
    __syncthreads();
    if (threadIdx.x == 0) { s_carry[0] += tot_c; s_carry[1] += tot_i; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { rp.row_off[U + 1] = s_carry[0]; rp.item_off[U + 1] = s_carry[1]; }
}

// Stage write-out: slot i -> its global position.  kBkPer slots per thread
// per pass, unrolled so the shared-memory reads of a pass are all in flight.
template <typename F>
__device__ __forceinline__ void write_out(int cnt, F&& store) {
  if (cnt == kBkTile) {
#pragma unroll
    for (int e = 0; e < kBkPer; ++e) store(e * kBkThreads + threadIdx.x);
  } else {
    for (int i = threadIdx.x; i < cnt; i += kBkThreads) store(i);
  }
}

// B3: scatter.  Tile t covers records [t*kBkTile, (t+1)*kBkTile); thread i
// owns records tile0 + 2*(j*kBkThreads + i) + {0, 1}, j < kBkPer/2, so each
// warp load is one 512-byte 128-bit-per-lane transaction.
struct ScatterSmem {
  unsigned long long* st64;   // [kBkTile] hfix staged in row order
  uint16_t* st16;             // [kQuad][kBkTile] tau-bins staged in row order (aliases st64)
  uint32_t* gpos;             // [kBkTile] sorted slot -> global position
  uint32_t* cnt;              // [kMaxBins] tile row counts, then local row offsets
  uint32_t* gbase;            // [kMaxBins] global base of the tile's run in each row
  uint32_t* guide_lt;
  uint32_t* guide_le;
  double* thr;                // [U + 2], +inf padded
  int64_t* warp;              // [32]
  uint32_t* tile_n;
};

// kFast: a full tile on a uniform grid (no bounds checks, no table search in
// the common case) -- the hot path; the general instantiation handles the
// last tile and guided grids.
template <bool kVec, bool kFast>
__device__ __forceinline__ void scatter_tile(const double* __restrict__ h,
                                             const double* __restrict__ scores, int64_t n,
                                             int n_light, int U, double hscale, int mode,
                                             const RowPlan& rp, uint64_t* __restrict__ hfix_rows,
                                             uint16_t* __restrict__ bs_rows, const ScatterSmem& sm,
                                             int64_t t0, int tn) {
  constexpr int kP = kBkPer / 2;
  const int B1 = U + 1;
  auto bin_h = [&](double x) {
    return kFast ? uniform_bin<false>(sm.thr, U, x) : plan_bin<false>(mode, sm.thr, U, sm.guide_lt, x);
  };
  auto bin_s = [&](double x) {
    return kFast ? uniform_bin<true>(sm.thr, U, x) : plan_bin<true>(mode, sm.thr, U, sm.guide_le, x);
  };
  for (int i = threadIdx.x; i < B1; i += blockDim.x) sm.cnt[i] = 0;
  __syncthreads();
  // 1. theta-row + local rank (ATOMS returns the rank within the tile's row)
  uint32_t key[kBkPer];          // (row << 16) | rank, 0xffffffff = no record
  uint64_t hf[kBkPer];
#pragma unroll
  for (int j = 0; j < kP; ++j) {
    const int r = 2 * (j * kBkThreads + threadIdx.x);
    double x0 = 0.0, x1 = 0.0;
    if (kVec && (kFast || r + 1 < tn)) {
      const double2 v = *reinterpret_cast<const double2*>(h + t0 + r);
      x0 = v.x; x1 = v.y;
    } else {
      if (r < tn) x0 = h[t0 + r];
      if (r + 1 < tn) x1 = h[t0 + r + 1];
    }
    const double xs[2] = {x0, x1};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (kFast || r + e < tn) {
        const double x = xs[e];
        const int b = bin_h(x);
        const uint32_t rank = atomicAdd(&sm.cnt[b], 1u);
        key[2 * j + e] = ((uint32_t)b << 16) | rank;
        hf[2 * j + e] = (uint64_t)__dmul_rn((x >= 0.0 && x <= 1.0) ? x : 0.0, hscale);
      } else {
        key[2 * j + e] = 0xffffffffu;
        hf[2 * j + e] = 0;
      }
    }
  }
  __syncthreads();
  // 2. local exclusive offsets + one global reservation per non-empty row
  {
    constexpr int kPer = (kMaxBins + kBkThreads - 1) / kBkThreads;
    const int per = (B1 + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per, i1 = min(B1, i0 + per);
    uint32_t cv[kPer], gv[kPer];              // counts first: the cursor atomics overlap
    int64_t tsum = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      cv[j] = i0 + j < i1 ? sm.cnt[i0 + j] : 0u;
      tsum += cv[j];
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) gv[j] = cv[j] ? atomicAdd(&rp.cursor[i0 + j], cv[j]) : 0u;
    int64_t total;
    int64_t run = block_excl_scan(tsum, sm.warp, &total);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (i0 + j < i1) {
        sm.gbase[i0 + j] = gv[j];
        sm.cnt[i0 + j] = (uint32_t)run;   // now the local row offsets
      }
      run += cv[j];
    }
    if (threadIdx.x == 0) *sm.tile_n = (uint32_t)total;
  }
  __syncthreads();
  // 3. sorted slot per record, its global position, hfix staged in row order
#pragma unroll
  for (int e = 0; e < kBkPer; ++e) {
    if (kFast || key[e] != 0xffffffffu) {
      const uint32_t b = key[e] >> 16, rank = key[e] & 0xffffu;
      const uint32_t slot = sm.cnt[b] + rank;
      sm.gpos[slot] = sm.gbase[b] + rank;
      sm.st64[slot] = hf[e];
      key[e] = slot;
    }
  }
  __syncthreads();
  const int cnt = kFast ? kBkTile : (int)*sm.tile_n;
  write_out(cnt, [&](int i) { hfix_rows[sm.gpos[i]] = sm.st64[i]; });
  // 4. per light model: tau-bins staged into row order, four models per
  //    write-out (one 8-byte store per record and quad).  Model l+1's
  //    scores are loaded while model l is binned (software pipelined).
  auto load_scores = [&](int l, double* sv) {
    const double* srow = scores + (int64_t)l * n + t0;
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      const int r = 2 * (j * kBkThreads + threadIdx.x);
      if (kVec && (kFast || r + 1 < tn)) {
        const double2 v = *reinterpret_cast<const double2*>(srow + r);
        sv[2 * j] = v.x; sv[2 * j + 1] = v.y;
      } else {
        sv[2 * j] = r < tn ? srow[r] : 0.0;
        sv[2 * j + 1] = r + 1 < tn ? srow[r + 1] : 0.0;
      }
    }
  };
  double sn[kBkPer];
  if (n_light > 0) load_scores(0, sn);
  for (int l = 0; l < n_light; ++l) {
    double sv[kBkPer];
#pragma unroll
    for (int e = 0; e < kBkPer; ++e) sv[e] = sn[e];
    if (l + 1 < n_light) load_scores(l + 1, sn);
    const int qm = l % kQuad;
    if (qm == 0) __syncthreads();      // previous quad (or hfix) fully written out
    uint16_t* st = sm.st16 + qm * kBkTile;
#pragma unroll
    for (int e = 0; e < kBkPer; ++e)
      if (kFast || key[e] != 0xffffffffu) st[key[e]] = (uint16_t)bin_s(sv[e]);
    if (qm == kQuad - 1 || l == n_light - 1) {
      __syncthreads();
      ushort4* orow = reinterpret_cast<ushort4*>(bs_rows) + (int64_t)(l / kQuad) * quad_stride(n);
      const uint16_t* s16 = sm.st16;
      write_out(cnt, [&](int i) {
        orow[sm.gpos[i]] = make_ushort4(s16[i], qm >= 1 ? s16[kBkTile + i] : 0,
                                        qm >= 2 ? s16[2 * kBkTile + i] : 0,
                                        qm >= 3 ? s16[3 * kBkTile + i] : 0);
      });
    }
  }
  __syncthreads();
}

template <bool kVec>
__device__ __noinline__ void scatter_tile_general(const double* __restrict__ h,
                                                  const double* __restrict__ scores, int64_t n,
                                                  int n_light, int U, double hscale, int mode,
                                                  const RowPlan& rp, uint64_t* __restrict__ hfix_rows,
                                                  uint16_t* __restrict__ bs_rows,
                                                  const ScatterSmem& sm, int64_t t0, int tn) {
  scatter_tile<kVec, false>(h, scores, n, n_light, U, hscale, mode, rp, hfix_rows, bs_rows, sm,
                            t0, tn);
}

template <bool kVec>
__global__ void __launch_bounds__(kBkThreads, 1)
bucket_scatter_kernel(const double* __restrict__ h, const double* __restrict__ scores, int64_t n,
                      int n_light, const double* __restrict__ thr, int U, double hscale,
                      RowPlan rp, uint64_t* __restrict__ hfix_rows, uint16_t* __restrict__ bs_rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t s_warp[32];
  __shared__ uint32_t s_tile_n;
  ScatterSmem sm;
  sm.st64 = reinterpret_cast<unsigned long long*>(smem);
  sm.st16 = reinterpret_cast<uint16_t*>(sm.st64);
  sm.gpos = reinterpret_cast<uint32_t*>(sm.st64 + kBkTile);
  sm.cnt = sm.gpos + kBkTile;
  sm.gbase = sm.cnt + kMaxBins;
  sm.guide_lt = sm.gbase + kMaxBins;
  sm.guide_le = sm.guide_lt + (kGuide + 2);
  sm.thr = reinterpret_cast<double*>(sm.guide_le + (kGuide + 2));
  sm.warp = s_warp;
  sm.tile_n = &s_tile_n;
  for (int i = threadIdx.x; i <= kGuide; i += blockDim.x) {
    sm.guide_lt[i] = rp.guide_lt[i];
    sm.guide_le[i] = rp.guide_le[i];
  }
  for (int i = threadIdx.x; i < U + 2; i += blockDim.x) sm.thr[i] = i < U ? thr[i] : INFINITY;
  const int mode = *rp.nonuniform == 0 ? 0 : (*rp.sparse == 0 ? 1 : 2);
  // one contiguous, even-sized record range per CTA (equal work per SM: 1221
  // round-robin tiles over 148 CTAs would leave a 9th partial wave at c4)
  const int64_t chunk = (ceil_div(n, (int64_t)gridDim.x) + 1) & ~(int64_t)1;
  const int64_t r0 = min(n, (int64_t)blockIdx.x * chunk), r1 = min(n, r0 + chunk);
  for (int64_t t0 = r0; t0 < r1; t0 += kBkTile) {
    const int tn = (int)min((int64_t)kBkTile, r1 - t0);
    if (mode == 0 && tn == kBkTile)
      scatter_tile<kVec, true>(h, scores, n, n_light, U, hscale, mode, rp, hfix_rows, bs_rows, sm,
                               t0, tn);
    else
      scatter_tile_general<kVec>(h, scores, n, n_light, U, hscale, mode, rp, hfix_rows, bs_rows,
                                 sm, t0, tn);
  }
}

// B3 (TMA-fed): the scatter with the record arrays streamed into a
// shared-memory ring by the bulk-copy engine.  One producer warp (one elected
// lane) issues cp.async.bulk copies of kTmaChunk-record chunks -- h, then each
// light model's scores, tile by tile -- into kTmaSlots ring slots, each
// completing on its "full" mbarrier; the 31 consumer warps wait on it, bin the
// chunk from shared memory and release the slot with one arrive per warp on
// its "empty" mbarrier, so loads stay in flight through every consumer-only
// phase.  Each CTA owns one contiguous record range (equal even-sized tiles).
// Per tile (<= kTmaTile records, kTmaPer per consumer):
//   H  theta-row bins + shared-memory ranks (ATOMS), hfix kept in registers
//   S  local row offsets (consumer scan) + one global cursor reservation per
//      non-empty row (all CTAs append at the same per-row cursor, so the
//      write frontier of the whole grid stays one dense run per row;
//      per-CTA precomputed row segments measured 2x slower: ~758K partial
//      lines alive in L2 instead of ~5K)
//   P  sorted slot -> global position + tile index; hfix staged in row order
//      and written out (consecutive threads, consecutive addresses)
//   Q  per model quad: every consumer bins its own records of the four
//      models into one 8-byte tau-bin word per record in registers, stores
//      them at their tile indices (16-byte, conflict-free) and the quad is
//      written out in sorted order.
// Uniform grids (the common case) bin with the branch-free uniform_bin_fast;
// measured (c4): the stores, not the loads, bound this kernel (streaming the
// records alone runs at 7.0 TB/s; all work without the stores at 5.5 TB/s).
struct TmaSmem {
  double* ring;               // [kTmaSlots][kTmaChunk]
  unsigned long long* st;     // [kTmaTile] hfix in row order, then one quad (tile order)
  uint32_t* gpos;             // [kTmaTile] sorted slot -> global position
  uint16_t* sidx;             // [kTmaTile] sorted slot -> tile index
  uint32_t* co;               // [B1] tile row counts, then local row offsets
  uint32_t* gb;               // [B1] global base of the tile's run in each row
  double* thr;                // [U + 2], +inf padded
};

__device__ __forceinline__ int64_t consumer_excl_scan(int64_t v, int64_t* s_warp, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kW = kTmaConsumers / 32;
  static_assert(kW <= 32, "one warp scans the warp totals");
  int64_t incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  named_sync(kTmaBar, kTmaConsumers);
  if (warp == 0) {
    int64_t w = lane < kW ? s_warp[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += o;
    }
    s_warp[lane] = w;
  }
  named_sync(kTmaBar, kTmaConsumers);
  const int64_t excl = (warp > 0 ? s_warp[warp - 1] : 0) + incl - v;
  *total = s_warp[kW - 1];
  named_sync(kTmaBar, kTmaConsumers);
  return excl;
}

// Uniform-grid bin without a table read, an XU convert or a branch:
// floor(x (U - 1)) is the low mantissa word of x (U - 1) + 2^52 (rounded
// toward zero); the answer is floor + 1 away from grid points (|frac - 1/2| <
// 1/2 - 1e-9, the margin of uniform_bin).  x = 0 and x = 1 (clipped scores)
// are exact grid points: floor + 1 for #{u <= x}, floor for #{u < x}.
// ok = false: the caller re-bins with uniform_bin.
template <bool kLE>
__device__ __forceinline__ int uniform_bin_fast(double x, double um1, bool* ok) {
  const double y = __dmul_rn(x, um1);
  const double t = __dadd_rz(y, 4503599627370496.0);                  // 2^52 + floor(y)
  const double d = __dadd_rn(y, -__dadd_rn(t, -4503599627370495.5));  // frac(y) - 1/2
  // x in [0, 1] up to the high word: hi <= 0x3ff00000 admits x in (1, 1 + 2^-20],
  // where floor(y) = U - 1 still gives the exact answer U (both counts)
  const uint32_t hi = (uint32_t)__double2hiint(x), lo = (uint32_t)__double2loint(x);
  const bool edge = (lo == 0u) & ((hi == 0u) | (hi == 0x3ff00000u));   // no short circuits:
  *ok = (hi <= 0x3ff00000u) & ((fabs(d) < 0.5 - 1e-9) | edge);           // keep it branch-free
  return __double2loint(t) + (kLE ? 1 : 1 - (int)edge);
}

// bins of a consumer's records of one ring chunk; kMode 0: uniform grid
// (fast bins, one warp vote, rare fix-up); 1: guide tables
template <int kMode, bool kLE>
__device__ __forceinline__ void bin_chunk(const double* thr, int U, double um1, int mode,
                                          const uint32_t* guide, const double (&x)[kTmaChunkPer],
                                          const bool (&valid)[kTmaChunkPer / 2],
                                          int (&b)[kTmaChunkPer]) {
  if (kMode == 0) {
    bool ok = true;
#pragma unroll
    for (int e = 0; e < kTmaChunkPer; ++e) {
      bool oke;
      b[e] = uniform_bin_fast<kLE>(x[e], um1, &oke);
      ok &= oke | !valid[e >> 1];
    }
    if (__any_sync(0xffffffffu, !ok)) {
      if (!ok) {
#pragma unroll
        for (int e = 0; e < kTmaChunkPer; ++e) b[e] = uniform_bin<kLE>(thr, U, x[e]);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < kTmaChunkPer; ++e) b[e] = plan_bin<kLE>(mode, thr, U, guide, x[e]);
  }
}

// tile index of a consumer's record e (chunk-major, two adjacent records per pair)
__device__ __forceinline__ int tma_rec(int e, int c) {
  return (e / kTmaChunkPer) * kTmaChunk + 2 * (((e % kTmaChunkPer) >> 1) * kTmaConsumers + c) +
         (e & 1);
}

template <int kMode>
__device__ __forceinline__ void scatter_consumers(const TmaSmem& sm, uint64_t* full,
                                                  uint64_t* empty, int64_t* s_warp, int64_t n,
                                                  int n_light, int U, double hscale,
                                                  const RowPlan& rp, int64_t r0, int64_t r1,
                                                  int64_t tile, uint64_t* __restrict__ hfix_rows,
                                                  uint16_t* __restrict__ bs_rows) {
  constexpr int kCP = kTmaChunkPer / 2;                // pairs per consumer and chunk
  const int c = threadIdx.x, lane = c & 31;
  const int B1 = U + 1;
  const double um1 = (double)(U - 1);
  const int mode = *rp.nonuniform == 0 ? 0 : (*rp.sparse == 0 ? 1 : 2);
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  int slot = 0;
  uint32_t ph = 0;
  // one ring chunk: the consumer's kTmaChunkPer records (pairs 16-byte loads)
  auto load_chunk = [&](const bool (&valid)[kCP], double (&x)[kTmaChunkPer]) {
    mbar_wait_u32(full0 + 8 * slot, ph);
    const double2* buf = reinterpret_cast<const double2*>(sm.ring + slot * kTmaChunk);
#pragma unroll
    for (int p = 0; p < kCP; ++p) {
      const double2 v = valid[p] ? buf[p * kTmaConsumers + c] : make_double2(0.0, 0.0);
      x[2 * p] = v.x;
      x[2 * p + 1] = v.y;
    }
    // order this thread's generic-proxy reads of the slot before the async-proxy
    // (bulk copy) writes the producer issues once the empty barrier completes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(empty0 + 8 * slot);
    if (++slot == kTmaSlots) { slot = 0; ph ^= 1u; }
  };
  // Pending write-out of the staged array (hfix or the last quad): consumer c
  // owns sorted slots c + k kTmaConsumers, k < kTmaPer; they are written a
  // few at a time between ring chunks of the next array, so the loads keep
  // streaming while the previous array drains.
  uint2* wo_quad = nullptr;           // null: hfix
  int wo_tn = 0, wo_done = kTmaPer;
#if HADIS_B3_WOBATCH > 1
  // kWB items at a time, every shared-memory read of the batch issued before
  // its global stores: the items' dependent read chains (gpos, sidx -> st)
  // overlap instead of running one item after the other through the
  // runtime-bounded loop (c4: 2 per batch -12 us, 4 -8 us, 8 +4 us)
  auto wo_items = [&](int upto) {
    constexpr int kWB = HADIS_B3_WOBATCH;
    while (wo_done < upto) {
      uint32_t gg[kWB];
      unsigned long long vv[kWB];
      bool ok[kWB];
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        const int i = c + (wo_done + u) * kTmaConsumers;
        ok[u] = wo_done + u < upto && i < wo_tn;
        gg[u] = ok[u] ? sm.gpos[i] : 0u;
        const int si = ok[u] ? (wo_quad ? (int)sm.sidx[i] : i) : 0;
        vv[u] = sm.st[si];
      }
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        if (ok[u]) {
          if (wo_quad) wo_quad[gg[u]] = reinterpret_cast<const uint2&>(vv[u]);
          else hfix_rows[gg[u]] = vv[u];
        }
      }
      wo_done = min(upto, wo_done + kWB);
    }
  };
#else
  auto wo_items = [&](int upto) {
    for (; wo_done < upto; ++wo_done) {
      const int i = c + wo_done * kTmaConsumers;
      if (i < wo_tn) {
        const uint32_t g = sm.gpos[i];
        if (wo_quad) wo_quad[g] = reinterpret_cast<const uint2*>(sm.st)[sm.sidx[i]];
        else hfix_rows[g] = sm.st[i];
      }
    }
  };
#endif
  // rows owned by this consumer (contiguous segment: scan order)
  const int per = (B1 + kTmaConsumers - 1) / kTmaConsumers;
  const int i0 = min(B1, c * per), i1 = min(B1, i0 + per);
  for (int i = i0; i < i1; ++i) sm.co[i] = 0;
  const int nq = (int)n_quads(n_light);
  uint2* const orow0 = reinterpret_cast<uint2*>(bs_rows);
  const int64_t qstride = quad_stride(n);
  named_sync(kTmaBar, kTmaConsumers);
  for (int64_t t0 = r0; t0 < r1; t0 += tile) {
    const int tn = (int)min(tile, r1 - t0);
    bool valid[kTmaChunks][kCP];                       // tn even: pairs are whole
#pragma unroll
    for (int k = 0; k < kTmaChunks; ++k)
#pragma unroll
      for (int p = 0; p < kCP; ++p) valid[k][p] = tma_rec(k * kTmaChunkPer + 2 * p, c) < tn;
    // H: theta-rows and ranks (the previous tile's last quad drains meanwhile)
    uint32_t key[kTmaPer];
    uint64_t hf[kTmaPer];
#pragma unroll
    for (int k = 0; k < kTmaChunks; ++k) {
      double x[kTmaChunkPer];
      int b[kTmaChunkPer];
      load_chunk(valid[k], x);
      bin_chunk<kMode, false>(sm.thr, U, um1, mode, rp.guide_lt, x, valid[k], b);
#pragma unroll
      for (int j = 0; j < kTmaChunkPer; ++j) {
        const int e = k * kTmaChunkPer + j;
        if (valid[k][j >> 1]) {
          const uint32_t rank = atomicAdd(&sm.co[b[j]], 1u);
          key[e] = ((uint32_t)b[j] << 16) | rank;
          hf[e] = (uint64_t)__dmul_rn((x[j] >= 0.0 && x[j] <= 1.0) ? x[j] : 0.0, hscale);
        } else {
          key[e] = 0xffffffffu;
          hf[e] = 0;
        }
      }
      wo_items((k + 1) * kTmaPer / kTmaChunks);
    }
    named_sync(kTmaBar, kTmaConsumers);
    // S: local row offsets + one global reservation per non-empty row (the
    // consumer's row counts are read into registers first, so its cursor
    // atomics are all in flight at once instead of one round trip per row)
    {
      uint32_t cv[kTmaRowsPer], gv[kTmaRowsPer];
      int64_t tsum = 0;
#pragma unroll
      for (int j = 0; j < kTmaRowsPer; ++j) {
        cv[j] = i0 + j < i1 ? sm.co[i0 + j] : 0u;
        tsum += cv[j];
      }
#pragma unroll
      for (int j = 0; j < kTmaRowsPer; ++j) gv[j] = cv[j] ? atomicAdd(&rp.cursor[i0 + j], cv[j]) : 0u;
      int64_t total;
      uint32_t run = (uint32_t)consumer_excl_scan(tsum, s_warp, &total);
#pragma unroll
      for (int j = 0; j < kTmaRowsPer; ++j) {
        if (i0 + j < i1) {
          sm.co[i0 + j] = run;
          sm.gb[i0 + j] = gv[j];
        }
        run += cv[j];
      }
    }
    named_sync(kTmaBar, kTmaConsumers);
    // P: sorted slots; hfix staged in row order
#pragma unroll
    for (int e = 0; e < kTmaPer; ++e) {
      if (key[e] != 0xffffffffu) {
        const uint32_t b = key[e] >> 16, rank = key[e] & 0xffffu;
        const uint32_t s = sm.co[b] + rank;
        sm.gpos[s] = sm.gb[b] + rank;
        sm.sidx[s] = (uint16_t)tma_rec(e, c);
        sm.st[s] = hf[e];
      }
    }
    named_sync(kTmaBar, kTmaConsumers);
    for (int i = i0; i < i1; ++i) sm.co[i] = 0;       // next tile's counters (offsets read)
    wo_quad = nullptr;                                 // hfix drains during quad 0
    wo_tn = tn;
    wo_done = 0;
    // Q: model quads, the four models' bins packed in registers
    for (int q = 0; q < nq; ++q) {
      uint32_t lo[kTmaPer], hi[kTmaPer];
      const int nm = min(kQuad, n_light - q * kQuad);
      const int steps = nm * kTmaChunks;
#pragma unroll
      for (int m = 0; m < kQuad; ++m) {
#pragma unroll
        for (int k = 0; k < kTmaChunks; ++k) {
          int b[kTmaChunkPer];
          if (m < nm) {
            double x[kTmaChunkPer];
            load_chunk(valid[k], x);
            bin_chunk<kMode, true>(sm.thr, U, um1, mode, rp.guide_le, x, valid[k], b);
            wo_items((m * kTmaChunks + k + 1) * kTmaPer / steps);
          } else {
#pragma unroll
            for (int j = 0; j < kTmaChunkPer; ++j) b[j] = 0;
          }
#pragma unroll
          for (int j = 0; j < kTmaChunkPer; ++j) {
            const int e = k * kTmaChunkPer + j;
            if (m == 0) lo[e] = (uint32_t)b[j];
            else if (m == 1) lo[e] |= (uint32_t)b[j] << 16;
            else if (m == 2) hi[e] = (uint32_t)b[j];
            else hi[e] |= (uint32_t)b[j] << 16;
          }
        }
      }
      wo_items(kTmaPer);
      named_sync(kTmaBar, kTmaConsumers);              // previous array drained from st
#pragma unroll
      for (int e = 0; e < kTmaPer; e += 2)
        if (valid[e / kTmaChunkPer][(e % kTmaChunkPer) >> 1])
          *reinterpret_cast<uint4*>(sm.st + tma_rec(e, c)) =
              make_uint4(lo[e], hi[e], lo[e + 1], hi[e + 1]);
      named_sync(kTmaBar, kTmaConsumers);
      wo_quad = orow0 + (int64_t)q * qstride;          // drains during the next quad / tile
      wo_done = 0;
    }
  }
  wo_items(kTmaPer);
}

__global__ void __launch_bounds__(kTmaThreads, 1)
bucket_scatter_tma_kernel(const double* __restrict__ h, const double* __restrict__ scores,
                          int64_t n, int n_light, const double* __restrict__ thr, int U,
                          double hscale, RowPlan rp, uint64_t* __restrict__ hfix_rows,
                          uint16_t* __restrict__ bs_rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kTmaSlots], empty[kTmaSlots];
  __shared__ int64_t s_warp[32];
  const int B1 = U + 1;
  TmaSmem sm;
  sm.ring = reinterpret_cast<double*>(smem);
  sm.st = reinterpret_cast<unsigned long long*>(sm.ring + kTmaSlots * kTmaChunk);
  sm.gpos = reinterpret_cast<uint32_t*>(sm.st + kTmaTile);
  sm.sidx = reinterpret_cast<uint16_t*>(sm.gpos + kTmaTile);
  sm.co = reinterpret_cast<uint32_t*>(sm.sidx + ((kTmaTile + 1) & ~1));
  sm.gb = sm.co + B1;
  sm.thr = reinterpret_cast<double*>(sm.gb + B1 + (((kTmaTile + 1) / 2) & 1));   // 8-byte aligned
  // one contiguous, even-sized record range per CTA (equal work per SM)
  const int64_t len = (ceil_div(n, (int64_t)gridDim.x) + 1) & ~(int64_t)1;
  const int64_t r0 = min(n, (int64_t)blockIdx.x * len), r1 = min(n, r0 + len);
  // equal even-sized tiles of at most kTmaTile records
  const int64_t ntiles = ceil_div(r1 - r0, (int64_t)kTmaTile);
  const int64_t tile = ntiles > 0 ? (ceil_div(r1 - r0, ntiles) + 1) & ~(int64_t)1 : kTmaTile;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTmaSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTmaConsumers / 32);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < U + 2; i += blockDim.x) sm.thr[i] = i < U ? thr[i] : INFINITY;
  __syncthreads();
  if (r0 >= r1) return;

  if (threadIdx.x >= kTmaConsumers) {                  // ---- producer warp
    if (threadIdx.x == kTmaConsumers) {
      const uint64_t pol = policy_evict_first();
      int slot = 0;
      uint32_t ph = 0;
      for (int64_t t0 = r0; t0 < r1; t0 += tile) {
        const int64_t tn = min(tile, r1 - t0);
        for (int a = 0; a <= n_light; ++a) {
          const double* src = (a == 0 ? h : scores + (int64_t)(a - 1) * n) + t0;
          for (int k = 0; k < kTmaChunks; ++k) {
            const int64_t m = min((int64_t)kTmaChunk, tn - (int64_t)k * kTmaChunk);
            mbar_wait(&empty[slot], ph ^ 1u);          // slot released by every consumer warp
            if (m > 0) {
              mbar_arrive_expect_tx(&full[slot], (uint32_t)(m * 8));
              bulk_load(sm.ring + (int64_t)slot * kTmaChunk, src + (int64_t)k * kTmaChunk,
                        (uint32_t)(m * 8), &full[slot], pol);
            } else {
              mbar_arrive(&full[slot]);                // empty chunk: complete the phase
            }
            if (++slot == kTmaSlots) { slot = 0; ph ^= 1u; }
          }
        }
      }
    }
    return;
  }
  const int mode = *rp.nonuniform == 0 ? 0 : 1;
  if (mode == 0)
    scatter_consumers<0>(sm, full, empty, s_warp, n, n_light, U, hscale, rp, r0, r1, tile,
                         hfix_rows, bs_rows);
  else
    scatter_consumers<1>(sm, full, empty, s_warp, n, n_light, U, hscale, rp, r0, r1, tile,
                         hfix_rows, bs_rows);
}

// dynamic shared memory limit of the TMA scatter (227 KB minus its static part)
constexpr size_t kTmaSmemMax = 227 * 1024 - 2 * 8 * kTmaSlots - 8 * 32 - 64;

static size_t scatter_tma_smem(int U) {
  const size_t B1 = (size_t)U + 1;
  const size_t T = kTmaTile, T2 = (T + 1) & ~(size_t)1;
  return (size_t)8 * kTmaSlots * kTmaChunk + 8 * T + 4 * T + 2 * T2 +
         4 * (2 * B1 + ((T2 / 2) & 1)) + (size_t)8 * (U + 2);
}

// K1: one CTA per (row chunk, model quad).  Each record's hfix (8 B) and its
// four tau-bins (one 8-byte load) feed the four models' shared-memory row
// histograms: count + 16-bit hardness limbs relative to the row's fixed-point
// lower bound (<= kRowChunk = 2^15 records per CTA, so no 32-bit limb can
// overflow); wide rows (span >= 2^32) add a third limb.
template <bool kNarrow>
__device__ __forceinline__ void row_accumulate(const uint64_t* __restrict__ hf,
                                               const ushort4* __restrict__ bq, int64_t r0,
                                               int64_t r1, unsigned long long base, int nm,
                                               uint32_t* s_bin, int B1s) {
  auto add1 = [&](uint32_t* sb, unsigned long long d, int b) {
    uint32_t* a = sb + b;
    atomicAdd(a, 1u);
    atomicAdd(a + B1s, (uint32_t)(d & 0xffffu));
    atomicAdd(a + 2 * B1s, (uint32_t)((d >> 16) & 0xffffu));
    if (!kNarrow) atomicAdd(a + 3 * B1s, (uint32_t)(d >> 32));
  };
  auto add = [&](unsigned long long hv, ushort4 b) {
    const unsigned long long d = hv - base;
    add1(s_bin, d, b.x);
    if (nm > 1) add1(s_bin + 4 * B1s, d, b.y);
    if (nm > 2) add1(s_bin + 8 * B1s, d, b.z);
    if (nm > 3) add1(s_bin + 12 * B1s, d, b.w);
  };
  const int64_t a0 = min(r1, (r0 + 1) & ~(int64_t)1);   // even: 16-byte aligned pairs
  const int64_t a1 = a0 + ((r1 - a0) & ~(int64_t)1);
  if (threadIdx.x == 0 && r0 < a0) add(hf[r0], bq[r0]);
  if (threadIdx.x == 1 && a1 < r1) add(hf[a1], bq[a1]);
  const ulonglong2* h2 = reinterpret_cast<const ulonglong2*>(hf);
  const uint4* b2 = reinterpret_cast<const uint4*>(bq);   // two records' quads
  const int64_t g0 = a0 >> 1, g1 = a1 >> 1;
  auto q4 = [](unsigned lo, unsigned hi) {
    return make_ushort4((unsigned short)(lo & 0xffffu), (unsigned short)(lo >> 16),
                        (unsigned short)(hi & 0xffffu), (unsigned short)(hi >> 16));
  };
  int64_t g = g0 + threadIdx.x;
  for (; g + blockDim.x < g1; g += 2 * blockDim.x) {
    const ulonglong2 hA = h2[g], hB = h2[g + blockDim.x];
    const uint4 bA = b2[g], bB = b2[g + blockDim.x];
    add(hA.x, q4(bA.x, bA.y));
    add(hA.y, q4(bA.z, bA.w));
    add(hB.x, q4(bB.x, bB.y));
    add(hB.y, q4(bB.z, bB.w));
  }
  for (; g < g1; g += blockDim.x) {
    const ulonglong2 hA = h2[g];
    const uint4 bA = b2[g];
    add(hA.x, q4(bA.x, bA.y));
    add(hA.y, q4(bA.z, bA.w));
  }
}

__global__ void __launch_bounds__(kK1Threads)
row_hist_kernel(const uint64_t* __restrict__ hf, const uint16_t* __restrict__ bs, int64_t n, int U,
                int n_light, RowPlan rp, uint32_t* __restrict__ g_cnt,
                unsigned long long* __restrict__ g_hsum, uint8_t* __restrict__ row_scanned) {
  extern __shared__ __align__(16) uint32_t s_bin[];    // [kQuad][4][B1s]
  const int B1 = U + 1;
  const int B1s = B1 | 1;                               // odd stride between limb arrays
  const int64_t items = rp.item_off[U + 1];
  const int64_t item = blockIdx.y;
  if (item >= items) return;
  int lo = 0, hi = U + 1;
  while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (rp.item_off[mid] <= item) lo = mid; else hi = mid - 1; }
  const int k = lo;
  const bool narrow = rp.row_narrow[k] != 0;
  const int64_t chunk = item - rp.item_off[k];
  const int64_t r0 = rp.row_off[k] + chunk * kRowChunk;
  const int64_t r1 = min(rp.row_off[k + 1], r0 + kRowChunk);
  const bool whole_row = (r0 == rp.row_off[k]) && (r1 == rp.row_off[k + 1]);
  const int quad = blockIdx.x;
  const int nm = min(kQuad, n_light - quad * kQuad);
  for (int i = threadIdx.x; i < nm * 4 * B1s; i += blockDim.x) s_bin[i] = 0;
  __syncthreads();
  const unsigned long long base = rp.row_base[k];
  const ushort4* bq = reinterpret_cast<const ushort4*>(bs) + (int64_t)quad * quad_stride(n);
  if (narrow) row_accumulate<true>(hf, bq, r0, r1, base, nm, s_bin, B1s);
  else row_accumulate<false>(hf, bq, r0, r1, base, nm, s_bin, B1s);
  __syncthreads();
  auto bin_sum = [&](const uint32_t* sb, int i) {
    return (unsigned long long)sb[i] * base + (unsigned long long)sb[B1s + i] +
           ((unsigned long long)sb[2 * B1s + i] << 16) +
           (narrow ? 0ull : (unsigned long long)sb[3 * B1s + i] << 32);
  };
  if (!whole_row || !row_scanned) {
    for (int m = 0; m < nm; ++m) {
      const int l = quad * kQuad + m;
      const uint32_t* sb = s_bin + m * 4 * B1s;
      uint32_t* gc = g_cnt + ((int64_t)l * B1 + k) * B1;
      unsigned long long* gh = g_hsum + ((int64_t)l * B1 + k) * B1;
      for (int i = threadIdx.x; i < B1; i += blockDim.x) {
        const uint32_t c = sb[i];
        const unsigned long long v = bin_sum(sb, i);
        if (whole_row) {
          gc[i] = c;
          gh[i] = v;
        } else if (c) {
          atomicAdd(&gc[i], c);
          atomicAdd(&gh[i], v);
        }
      }
    }
    return;
  }
  // whole row: emit the K2 row prefix (along bs) of all nm models at once --
  // thread-contiguous segments, one block scan of the segment totals (per
  // model, carried together), then the segment prefixes
  const int per = (B1 + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(B1, i0 + per);
  uint32_t tc[kQuad];
  unsigned long long th[kQuad];
#pragma unroll
  for (int m = 0; m < kQuad; ++m) {
    tc[m] = 0;
    th[m] = 0;
    if (m < nm)
      for (int i = i0; i < i1; ++i) { tc[m] += s_bin[m * 4 * B1s + i]; th[m] += bin_sum(s_bin + m * 4 * B1s, i); }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t ic[kQuad];
  unsigned long long ih[kQuad];
#pragma unroll
  for (int m = 0; m < kQuad; ++m) { ic[m] = tc[m]; ih[m] = th[m]; }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int m = 0; m < kQuad; ++m) {
      const uint32_t oc = __shfl_up_sync(0xffffffffu, ic[m], off);
      const unsigned long long oh = __shfl_up_sync(0xffffffffu, ih[m], off);
      if (lane >= off) { ic[m] += oc; ih[m] += oh; }
    }
  }
  __shared__ uint32_t ws_cq[kQuad][kK1Threads / 32];
  __shared__ unsigned long long ws_hq[kQuad][kK1Threads / 32];
  if (lane == 31)
#pragma unroll
    for (int m = 0; m < kQuad; ++m) { ws_cq[m][warp] = ic[m]; ws_hq[m][warp] = ih[m]; }
  __syncthreads();
  if (warp < kQuad) {
    const int m = warp, nw = blockDim.x >> 5;
    uint32_t wc = lane < nw ? ws_cq[m][lane] : 0u;
    unsigned long long wh = lane < nw ? ws_hq[m][lane] : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t oc = __shfl_up_sync(0xffffffffu, wc, off);
      const unsigned long long oh = __shfl_up_sync(0xffffffffu, wh, off);
      if (lane >= off) { wc += oc; wh += oh; }
    }
    if (lane < nw) { ws_cq[m][lane] = wc; ws_hq[m][lane] = wh; }
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < kQuad; ++m) {
    if (m >= nm) break;
    const int l = quad * kQuad + m;
    const uint32_t* sb = s_bin + m * 4 * B1s;
    uint32_t* gc = g_cnt + ((int64_t)l * B1 + k) * B1;
    unsigned long long* gh = g_hsum + ((int64_t)l * B1 + k) * B1;
    uint32_t rc = (warp > 0 ? ws_cq[m][warp - 1] : 0u) + ic[m] - tc[m];
    unsigned long long rh = (warp > 0 ? ws_hq[m][warp - 1] : 0ull) + ih[m] - th[m];
    for (int i = i0; i < i1; ++i) {
      rc += sb[i];
      rh += bin_sum(sb, i);
      gc[i] = rc;
      gh[i] = rh;
    }
    if (threadIdx.x == 0) row_scanned[(int64_t)l * B1 + k] = 1;
  }
}

// Before K1 (row_scanned path): one warp per (light model, row).  Empty rows
// are written as zeros -- already their own prefix -- and flagged scanned;
// rows split across K1 CTAs (atomics) are zeroed and left for K2's row pass;
// every other row is written whole by one K1 CTA.
__global__ void prep_rows_kernel(RowPlan rp, int n_light, int U, uint32_t* __restrict__ g_cnt,
                                 unsigned long long* __restrict__ g_hsum,
                                 uint8_t* __restrict__ row_scanned) {
  const int B1 = U + 1;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= (int64_t)n_light * B1) return;
  const int k = (int)(row % B1);
  const uint32_t c = rp.row_cnt[k];
  const bool zero = c == 0 || c > (uint32_t)kRowChunk;
  if (zero) {
    uint32_t* gc = g_cnt + row * B1;
    unsigned long long* gh = g_hsum + row * B1;
    for (int i = lane; i < B1; i += 32) { gc[i] = 0u; gh[i] = 0ull; }
  }
  if (lane == 0) row_scanned[row] = c == 0;
}

static size_t scatter_smem(int U) {
  return (size_t)8 * kBkTile + (size_t)4 * (kBkTile + 2 * kMaxBins + 2 * (kGuide + 2)) +
         (size_t)8 * (U + 2);
}

}  // namespace hadis

using namespace hadis;

extern "C" int64_t hadis_bs_store_elems(int64_t n, int32_t n_light) {
  return n <= 0 || n_light <= 0 ? 0 : n_quads(n_light) * kQuad * quad_stride(n);
}

extern "C" size_t hadis_row_plan_bytes(int32_t n_unique) {
  if (n_unique <= 0 || n_unique + 1 > kMaxBins) return 0;
  return row_plan_size();
}

static int records_args_ok(const double* h, const double* scores, int64_t n, int32_t n_light,
                           const double* thr_unique, int32_t n_unique, int32_t hfix_shift,
                           const void* row_plan, size_t row_plan_bytes) {
  if (!h || n <= 0 || n > 0xffffffffll || n_light < 0 || (n_light > 0 && !scores) ||
      !thr_unique || n_unique <= 0 || !row_plan || hfix_shift < 1 || hfix_shift > 48)
    return HADIS_ERR_ARG;
  if (n_unique + 1 > kMaxBins) return HADIS_ERR_UNSUPPORTED;
  if (row_plan_bytes < row_plan_size()) return HADIS_ERR_CAPACITY;
  return HADIS_OK;
}

// B0..B2: guides, row counts, row offsets / K1 items (reads h only)
extern "C" int hadis_records_plan(const double* h, int64_t n, const double* thr_unique,
                                  int32_t n_unique, int32_t hfix_shift, uint32_t* bad_records,
                                  void* row_plan, size_t row_plan_bytes, void* stream) {
  const int rc = records_args_ok(h, h, n, 0, thr_unique, n_unique, hfix_shift, row_plan,
                                 row_plan_bytes);
  if (rc != HADIS_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const RowPlan rp = row_plan_at(row_plan);
  const double hscale = ldexp(1.0, hfix_shift);
  HADIS_CUDA_TRY(cudaMemsetAsync(rp.bad, 0, 256 * 3, st));      // bad, sparse, nonuniform
  bucket_setup_kernel<<<(unsigned)ceil_div(kGuide + 2, 256), 256, 0, st>>>(thr_unique, n_unique, rp);
  HADIS_LAUNCH_CHECK();
  const size_t csmem = (size_t)4 * (kMaxBins + kGuide + 2) + (size_t)8 * (n_unique + 2);
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)bucket_count_kernel, (size_t)csmem));
  int64_t cgrid = ceil_div(n, 2 * kCountThreads * 8);
  if (cgrid > kNumSMs * 2) cgrid = kNumSMs * 2;
  bucket_count_kernel<<<(unsigned)cgrid, kCountThreads, csmem, st>>>(h, n, thr_unique, n_unique, rp);
  HADIS_LAUNCH_CHECK();
  bucket_plan_kernel<<<1, 1024, 0, st>>>(thr_unique, n_unique, hscale, rp);
  HADIS_LAUNCH_CHECK();
  if (bad_records)
    HADIS_CUDA_TRY(cudaMemcpyAsync(bad_records, rp.bad, 4, cudaMemcpyDeviceToDevice, st));
  hadis_count_launches(3);
  return HADIS_OK;
}

// B3: the HBM-bound scatter into the row-bucketed store (needs the plan)
extern "C" int hadis_records_scatter(const double* h, const double* scores, int64_t n,
                                     int32_t n_light, const double* thr_unique, int32_t n_unique,
                                     int32_t hfix_shift, uint64_t* hfix_rows, uint16_t* bs_rows,
                                     void* row_plan, size_t row_plan_bytes, void* stream) {
  const int rc = records_args_ok(h, scores, n, n_light, thr_unique, n_unique, hfix_shift,
                                 row_plan, row_plan_bytes);
  if (rc != HADIS_OK) return rc;
  if (!hfix_rows || (n_light > 0 && !bs_rows)) return HADIS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const RowPlan rp = row_plan_at(row_plan);
  const double hscale = ldexp(1.0, hfix_shift);
  bool vec = (reinterpret_cast<uintptr_t>(h) & 15) == 0 && (n & 1) == 0 &&
             (n_light == 0 || (reinterpret_cast<uintptr_t>(scores) & 15) == 0);
  int64_t sgrid = ceil_div(n, kBkTile);
  if (sgrid > kNumSMs) sgrid = kNumSMs;
  const char* legacy = getenv("HADIS_B3_REGISTER_PATH");   // A/B switch for measurements
  const size_t tsmem = scatter_tma_smem(n_unique);
  if (vec && tsmem <= kTmaSmemMax && !(legacy && legacy[0] == '1')) {
    // aligned record arrays: the TMA-fed scatter over the plan's record ranges
    // (binning mode read on the device)
    HADIS_CUDA_TRY(hadis_ensure_smem((const void*)bucket_scatter_tma_kernel, (size_t)tsmem));
    int64_t tgrid = ceil_div(n, kTmaTile);
    if (tgrid > kNumSMs) tgrid = kNumSMs;
    bucket_scatter_tma_kernel<<<(unsigned)tgrid, kTmaThreads, tsmem, st>>>(
        h, scores, n, n_light, thr_unique, n_unique, hscale, rp, hfix_rows, bs_rows);
    HADIS_LAUNCH_CHECK();
    hadis_count_launches(1);
    return HADIS_OK;
  }
  const size_t ssmem = scatter_smem(n_unique);
  auto kern = vec ? bucket_scatter_kernel<true> : bucket_scatter_kernel<false>;
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)kern, (size_t)ssmem));
  kern<<<(unsigned)sgrid, kBkThreads, ssmem, st>>>(h, scores, n, n_light, thr_unique, n_unique,
                                                   hscale, rp, hfix_rows, bs_rows);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}

extern "C" int hadis_records_bucket(const double* h, const double* scores, int64_t n,
                                    int32_t n_light, const double* thr_unique, int32_t n_unique,
                                    int32_t hfix_shift, uint64_t* hfix_rows, uint16_t* bs_rows,
                                    uint32_t* bad_records, void* row_plan, size_t row_plan_bytes,
                                    void* stream) {
  const int rc = hadis_records_plan(h, n, thr_unique, n_unique, hfix_shift, bad_records, row_plan,
                                    row_plan_bytes, stream);
  if (rc != HADIS_OK) return rc;
  return hadis_records_scatter(h, scores, n, n_light, thr_unique, n_unique, hfix_shift, hfix_rows,
                               bs_rows, row_plan, row_plan_bytes, stream);
}

extern "C" int hadis_bin_hist_rows(const uint64_t* hfix_rows, const uint16_t* bs_rows, int64_t n,
                                   int32_t n_light, int32_t n_unique, const void* row_plan,
                                   uint32_t* hist_cnt, uint64_t* hist_hsum, uint8_t* row_scanned,
                                   void* stream) {
  if (!hfix_rows || !bs_rows || n <= 0 || n > 0xffffffffll || n_light <= 0 || n_unique <= 0 ||
      !row_plan || !hist_cnt || !hist_hsum || n_light > 65535)
    return HADIS_ERR_ARG;
  if (n_unique + 1 > kMaxBins) return HADIS_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const RowPlan rp = row_plan_at(const_cast<void*>(row_plan));
  const int64_t B1 = (int64_t)n_unique + 1;
  const int64_t bins = B1 * B1 * n_light;
  const int64_t max_items = ceil_div(n, kRowChunk) + n_unique + 1;
  if (max_items > 65535) return HADIS_ERR_UNSUPPORTED;
  if (row_scanned) {
    const int64_t rows = B1 * n_light;
    prep_rows_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0, st>>>(
        rp, n_light, n_unique, hist_cnt, (unsigned long long*)hist_hsum, row_scanned);
    HADIS_LAUNCH_CHECK();
    hadis_count_launches(1);
  } else {
    HADIS_CUDA_TRY(cudaMemsetAsync(hist_cnt, 0, bins * sizeof(uint32_t), st));
    HADIS_CUDA_TRY(cudaMemsetAsync(hist_hsum, 0, bins * sizeof(uint64_t), st));
  }
  const int B1s = (n_unique + 1) | 1;
  const size_t ksmem = (size_t)kQuad * 4 * B1s * 4;
  // opt in unconditionally: static shared memory counts against the 48 KB default
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)row_hist_kernel, (size_t)ksmem));
  const dim3 grid((unsigned)n_quads(n_light), (unsigned)max_items);
  row_hist_kernel<<<grid, kK1Threads, ksmem, st>>>(hfix_rows, bs_rows, n, n_unique, n_light, rp,
                                                  hist_cnt, (unsigned long long*)hist_hsum,
                                                  row_scanned);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}
