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
constexpr int kK1Threads = 512;
constexpr int kBkThreads = 1024;      // scatter CTA (512 x 2/SM and 4096-record tiles: slower;
constexpr int kBkTile = 8192;         // records per scatter tile   L2 bulk prefetch ahead: slower)
constexpr int kBkPer = kBkTile / kBkThreads;   // records per thread per tile (even)
constexpr int kCountThreads = 512;

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
    const int per = (B1 + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per, i1 = min(B1, i0 + per);
    int64_t tsum = 0;
    for (int i = i0; i < i1; ++i) tsum += sm.cnt[i];
    int64_t total;
    int64_t run = block_excl_scan(tsum, sm.warp, &total);
    for (int i = i0; i < i1; ++i) {
      const uint32_t c = sm.cnt[i];
      sm.gbase[i] = c ? atomicAdd(&rp.cursor[i], c) : 0u;
      sm.cnt[i] = (uint32_t)run;          // now the local row offsets
      run += c;
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

// B3 (TMA-fed): the same scatter with the record arrays streamed into a
// shared-memory ring by the bulk-copy engine instead of register prefetch.
// One producer warp (one elected lane) issues cp.async.bulk copies of
// kTmaChunk-record chunks -- h, then each light model's scores, tile by tile
// -- into kTmaSlots ring slots, each completing on its "full" mbarrier; the
// kTmaConsumers consumer threads (16 warps) wait on it, bin the chunk from
// shared memory and release the slot with one arrive per warp on its "empty"
// mbarrier.  Loads therefore stay in flight through the tile prologue
// (ranks, block scan, cursor reservations) and every write-out, and no
// record data is held in registers across phases.  Consumer-only phases
// synchronise with a named barrier; the producer never joins them.
#ifndef HADIS_TMA_CONSUMER_WARPS
#define HADIS_TMA_CONSUMER_WARPS 31
#endif
#ifndef HADIS_TMA_PER_CHUNK
#define HADIS_TMA_PER_CHUNK 4
#endif
#ifndef HADIS_TMA_SLOTS
#define HADIS_TMA_SLOTS 3
#endif
constexpr int kTmaConsumers = 32 * HADIS_TMA_CONSUMER_WARPS;   // consumer threads
constexpr int kTmaThreads = kTmaConsumers + 32;        // + the producer warp
#ifndef HADIS_TMA_PER
#define HADIS_TMA_PER 8
#endif
constexpr int kTmaPer = HADIS_TMA_PER;                 // records per consumer per tile
constexpr int kTmaPerChunk = HADIS_TMA_PER_CHUNK;      // records per consumer per ring chunk
constexpr int kTmaChunks = kTmaPer / kTmaPerChunk;     // chunks per record array and tile
constexpr int kTmaChunk = kTmaPerChunk * kTmaConsumers;   // records per ring slot
constexpr int kTmaTile = kTmaPer * kTmaConsumers;      // records per tile
constexpr int kTmaSlots = HADIS_TMA_SLOTS;
constexpr int kTmaBar = 1;                             // named barrier id (consumers)

struct TmaSmem {
  double* ring;               // [kTmaSlots][kTmaChunk]
  unsigned long long* st64;   // [kTmaTile] hfix staged in row order
  ushort4* st4;               // [kTmaTile] tau-bins of a model quad per slot (aliases st64)
  uint32_t* gpos;             // [kTmaTile]
  uint32_t* cnt;              // [kMaxBins]
  uint32_t* gbase;            // [kMaxBins]
  double* thr;                // [U + 2]
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

__global__ void __launch_bounds__(kTmaThreads, 1)
bucket_scatter_tma_kernel(const double* __restrict__ h, const double* __restrict__ scores,
                          int64_t n, int n_light, const double* __restrict__ thr, int U,
                          double hscale, RowPlan rp, uint64_t* __restrict__ hfix_rows,
                          uint16_t* __restrict__ bs_rows) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kTmaSlots], empty[kTmaSlots];
  __shared__ int64_t s_warp[32];
  __shared__ uint32_t s_tile_n;
  TmaSmem sm;
  sm.ring = reinterpret_cast<double*>(smem);
  sm.st64 = reinterpret_cast<unsigned long long*>(sm.ring + kTmaSlots * kTmaChunk);
  sm.st4 = reinterpret_cast<ushort4*>(sm.st64);
  sm.gpos = reinterpret_cast<uint32_t*>(sm.st64 + kTmaTile);
  sm.cnt = sm.gpos + kTmaTile;
  sm.gbase = sm.cnt + kMaxBins;
  sm.thr = reinterpret_cast<double*>(sm.gbase + kMaxBins);
  const int B1 = U + 1;
  const int64_t chunk = (ceil_div(n, (int64_t)gridDim.x) + 1) & ~(int64_t)1;
  const int64_t r0 = min(n, (int64_t)blockIdx.x * chunk), r1 = min(n, r0 + chunk);
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
      for (int64_t t0 = r0; t0 < r1; t0 += kTmaTile) {
        const int64_t tn = min((int64_t)kTmaTile, r1 - t0);
        for (int a = 0; a <= n_light; ++a) {
          const double* src = (a == 0 ? h : scores + (int64_t)(a - 1) * n) + t0;
          for (int c = 0; c < kTmaChunks; ++c) {
            const int64_t m = min((int64_t)kTmaChunk, tn - (int64_t)c * kTmaChunk);
            mbar_wait(&empty[slot], ph ^ 1u);          // slot released by every consumer warp
            if (m > 0) {
              mbar_arrive_expect_tx(&full[slot], (uint32_t)(m * 8));
              bulk_load(sm.ring + slot * kTmaChunk, src + (int64_t)c * kTmaChunk,
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

  // ---- consumers (threads 0 .. kTmaConsumers-1)
  const int lane = threadIdx.x & 31;
  int slot = 0;
  uint32_t ph = 0;
  // record e of this consumer: chunk e / kTmaPerChunk, two adjacent records
  // per 16-byte load
  auto rec = [](int e) { return 2 * ((e >> 1) * kTmaConsumers + (int)threadIdx.x) + (e & 1); };
  auto acquire = [&]() { mbar_wait(&full[slot], ph); return sm.ring + slot * kTmaChunk; };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == kTmaSlots) { slot = 0; ph ^= 1u; }
  };
  // uniform grids (the common case) bin with two compares; others search
  // with the guide tables (read through L1 from the row plan)
  const int mode = *rp.nonuniform == 0 ? 0 : (*rp.sparse == 0 ? 1 : 2);
  auto bin_h = [&](double x) {
    return mode == 0 ? uniform_bin<false>(sm.thr, U, x)
                     : plan_bin<false>(mode, sm.thr, U, rp.guide_lt, x);
  };
  auto bin_s = [&](double x) {
    return mode == 0 ? uniform_bin<true>(sm.thr, U, x)
                     : plan_bin<true>(mode, sm.thr, U, rp.guide_le, x);
  };
  for (int64_t t0 = r0; t0 < r1; t0 += kTmaTile) {
    const int tn = (int)min((int64_t)kTmaTile, r1 - t0);
    for (int i = threadIdx.x; i < B1; i += kTmaConsumers) sm.cnt[i] = 0;
    named_sync(kTmaBar, kTmaConsumers);
    // 1. theta-row + local rank from the two h chunks; hfix kept in registers
    uint32_t key[kTmaPer];
    uint64_t hf[kTmaPer];
#pragma unroll
    for (int c = 0; c < kTmaChunks; ++c) {
      const double* buf = acquire();
      double xs[kTmaPerChunk];                      // 16-byte shared loads, two records each
#pragma unroll
      for (int e2 = 0; e2 < kTmaPerChunk; e2 += 2) {
        const double2 v = reinterpret_cast<const double2*>(buf)[(rec(c * kTmaPerChunk + e2) - c * kTmaChunk) >> 1];
        xs[e2] = v.x; xs[e2 + 1] = v.y;
      }
#pragma unroll
      for (int e = c * kTmaPerChunk; e < (c + 1) * kTmaPerChunk; ++e) {
        const int r = rec(e);
        if (r < tn) {
          const double x = xs[e - c * kTmaPerChunk];
          const int b = bin_h(x);
          const uint32_t rank = atomicAdd(&sm.cnt[b], 1u);
          key[e] = ((uint32_t)b << 16) | rank;
          hf[e] = (uint64_t)__dmul_rn((x >= 0.0 && x <= 1.0) ? x : 0.0, hscale);
        } else {
          key[e] = 0xffffffffu;
          hf[e] = 0;
        }
      }
      release();
    }
    named_sync(kTmaBar, kTmaConsumers);
    // 2. local exclusive offsets + one global reservation per non-empty row
    {
      const int per = (B1 + kTmaConsumers - 1) / kTmaConsumers;
      const int i0 = threadIdx.x * per, i1 = min(B1, i0 + per);
      int64_t tsum = 0;
      for (int i = i0; i < i1; ++i) tsum += sm.cnt[i];
      int64_t total;
      int64_t run = consumer_excl_scan(tsum, s_warp, &total);
      for (int i = i0; i < i1; ++i) {
        const uint32_t c = sm.cnt[i];
        sm.gbase[i] = c ? atomicAdd(&rp.cursor[i], c) : 0u;
        sm.cnt[i] = (uint32_t)run;
        run += c;
      }
      if (threadIdx.x == 0) s_tile_n = (uint32_t)total;
    }
    named_sync(kTmaBar, kTmaConsumers);
    // 3. sorted slot, global position, hfix staged in row order
#pragma unroll
    for (int e = 0; e < kTmaPer; ++e) {
      if (key[e] != 0xffffffffu) {
        const uint32_t b = key[e] >> 16, rank = key[e] & 0xffffu;
        const uint32_t s = sm.cnt[b] + rank;
        sm.gpos[s] = sm.gbase[b] + rank;
        sm.st64[s] = hf[e];
        key[e] = s;
      }
    }
    named_sync(kTmaBar, kTmaConsumers);
    const int cnt = (int)s_tile_n;
    for (int i = threadIdx.x; i < cnt; i += kTmaConsumers) hfix_rows[sm.gpos[i]] = sm.st64[i];
    // 4. per light model: two chunks binned into the quad staging, four
    //    models per write-out (one 8-byte store per record and quad)
    for (int l = 0; l < n_light; ++l) {
      const int qm = l % kQuad;
      if (qm == 0) named_sync(kTmaBar, kTmaConsumers);   // previous write-out done
      uint16_t* st = reinterpret_cast<uint16_t*>(sm.st4) + qm;    // lane qm of each slot
#pragma unroll
      for (int c = 0; c < kTmaChunks; ++c) {
        const double* buf = acquire();
        double xs[kTmaPerChunk];
#pragma unroll
        for (int e2 = 0; e2 < kTmaPerChunk; e2 += 2) {
          const double2 v = reinterpret_cast<const double2*>(buf)[(rec(c * kTmaPerChunk + e2) - c * kTmaChunk) >> 1];
          xs[e2] = v.x; xs[e2 + 1] = v.y;
        }
#pragma unroll
        for (int e = c * kTmaPerChunk; e < (c + 1) * kTmaPerChunk; ++e)
          if (key[e] != 0xffffffffu)
            st[4 * key[e]] = (uint16_t)bin_s(xs[e - c * kTmaPerChunk]);
        release();
      }
      if (qm == kQuad - 1 || l == n_light - 1) {
        named_sync(kTmaBar, kTmaConsumers);
        ushort4* orow = reinterpret_cast<ushort4*>(bs_rows) + (int64_t)(l / kQuad) * quad_stride(n);
        // lanes past the last model of a partial quad carry stale bins; K1
        // reads only the quad's n_light % 4 models
        for (int i = threadIdx.x; i < cnt; i += kTmaConsumers) orow[sm.gpos[i]] = sm.st4[i];
      }
    }
    named_sync(kTmaBar, kTmaConsumers);
  }
}

static size_t scatter_tma_smem(int U) {
  return (size_t)8 * kTmaSlots * kTmaChunk + (size_t)8 * kTmaTile + (size_t)4 * kTmaTile +
         (size_t)4 * 2 * kMaxBins + (size_t)8 * (U + 2);
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
  HADIS_CUDA_TRY(cudaFuncSetAttribute(bucket_count_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
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
  if (vec && !(legacy && legacy[0] == '1')) {
    // aligned record arrays: the TMA-fed scatter (binning mode read on the device)
    const size_t tsmem = scatter_tma_smem(n_unique);
    HADIS_CUDA_TRY(cudaFuncSetAttribute(bucket_scatter_tma_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));
    bucket_scatter_tma_kernel<<<(unsigned)sgrid, kTmaThreads, tsmem, st>>>(
        h, scores, n, n_light, thr_unique, n_unique, hscale, rp, hfix_rows, bs_rows);
    HADIS_LAUNCH_CHECK();
    hadis_count_launches(1);
    return HADIS_OK;
  }
  const size_t ssmem = scatter_smem(n_unique);
  auto kern = vec ? bucket_scatter_kernel<true> : bucket_scatter_kernel<false>;
  HADIS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
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
  HADIS_CUDA_TRY(cudaFuncSetAttribute(row_hist_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksmem));
  const dim3 grid((unsigned)n_quads(n_light), (unsigned)max_items);
  row_hist_kernel<<<grid, kK1Threads, ksmem, st>>>(hfix_rows, bs_rows, n, n_unique, n_light, rp,
                                                  hist_cnt, (unsigned long long*)hist_hsum,
                                                  row_scanned);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}
