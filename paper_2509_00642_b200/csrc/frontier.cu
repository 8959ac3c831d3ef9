// K3 + K4: grid-cell evaluation, Pareto extraction and row emission.
//
// Reference: pkg/src/cascadesim/profiler.py:140-174 and catalog.py:171-192.
// For each pair (light i, heavy j) and each distinct-threshold cell (k, t):
//   nb = n - R[k]            (R[k] = #{bh <= k}: records not bypassed)
//   nr = C_i[k][t]           (non-bypassed and s_i < tau)
//   lat = ((n-nb)*L_i + (nb+nr)*L_j) / n          -- bit-exact, no FMA
//   r_light = (n-nb)/n, r_heavy = (nb+nr)/n          -- bit-exact
//   fid* = (b_j*nH + b_i*nL + (p_j*SH + p_i*SL)*2^-shift) / n
// where SH/SL are exact fixed-point hardness sums.  fid* differs from numpy's
// pairwise mean by at most delta (a rigorous per-pair bound), so a Pareto
// decision is "certain" unless two cells' fid* lie within 2*delta and their
// heavy sets differ (equal heavy sets give bitwise-equal fidelities in both
// numpy and here).  Uncertain decisions are re-decided on numpy-exact values
// from the pairwise emulation (pairwise.cuh).
//
// Pipeline (all stream-ordered, no host synchronisation):
//   F1 bucket minima   per pair, latency buckets -> min fid*          (atomicMin)
//   F2 prefix minima   exclusive prefix-min over buckets
//   F3 filter          keep cells with fid* <= prefix-min + 2 delta (candidates)
//   F4/F5 group        counting sort of candidates by (pair, bucket)
//   F6 decide          kill / keep / uncertain per candidate (in-bucket compare,
//                      heavy-set twin test, prefix-min margin)
//   F7 no-bypass row   theta = max(thresholds) sub-frontier (profiler.py:168-170)
//   F8-F11             partners of uncertain cells -> numpy-exact fid -> decide
//   F12 emit           kept-cell bitmap -> rows in (theta, tau) order
//   F13/F14            exact fidelity patch for emitted rows
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cfloat>
#include <cmath>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"
#include "pairwise.cuh"

namespace hadis {

enum : uint32_t { kKept = 1u, kUncertain = 2u };

struct PairConst {
  double Ll, Lh, bl, pl, bh, ph;
  double delta2;       // 2 * delta (fidelity space)
  double delta2_S;     // the same margin in numerator space (fid* * n), padded
  double off_x, scale_x;  // latency-numerator bucket map: b = floor(fma(x, scale_x, off_x))
  int slot;
};

struct Grid {
  const uint32_t* cnt;      // K2 prefix counts [slot][B1][B1]
  const uint64_t* hs;       // K2 prefix hardness sums
  int64_t n;
  int U, B1;
  double inv_scale;         // 2^-shift
  int nbuckets;
  int K;
  const int32_t* first_pos;
  int64_t bm_stride;        // bits per pair in the kept bitmap (words_per_pair * 32)
  const int32_t* pk;        // twin row: largest k' < k with R[k'] < R[k], else -1
  const int32_t* row_rep;   // rank with the smallest first_pos in k's row class
  const uint8_t* row_start; // 1 if k starts its row class (R[k-1] < R[k])
  const int32_t* sorted;    // *sorted != 0: first_pos increases with rank (sorted list)
  double rn;                // RN(1 / n): divisions by n through div_n
};

// a / n correctly rounded, for the fixed divisor n (record count, < 2^32) and
// rn = RN(1/n): q0 = RN(a rn) is within one ulp of a/n, the residual a - n q0
// is exact with one FMA, and RN(q0 + r rn) is then the correctly rounded
// quotient (Markstein's theorem; no over/underflow for |a| < 2^64) -- three
// FP64 ops instead of __ddiv_rn's reciprocal refinement and slow-path checks.
// Checked against IEEE division on 6e8 random and near-midpoint cases (n up to
// 2^33) and by every bit-exact table test.
__device__ __forceinline__ double div_n(double a, double dn, double rn) {
  const double q0 = __dmul_rn(a, rn);
  return __fma_rn(__fma_rn(-q0, dn, a), rn, q0);
}

struct CellVal {
  double lat, fid;
  uint32_t n_keep_light;    // R[k]  (= n - nb)
  uint32_t n_heavy;         // nb + nr
};

__device__ __forceinline__ const uint32_t* slot_cnt(const Grid& g, int slot) {
  return g.cnt + (int64_t)slot * g.B1 * g.B1;
}
__device__ __forceinline__ const uint64_t* slot_hs(const Grid& g, int slot) {
  return g.hs + (int64_t)slot * g.B1 * g.B1;
}

// fid* numerator, the one formula every stage uses (so equal heavy sets give
// bitwise-equal values):  S = p_h SH 2^-s + (b_h nH + (p_l SL 2^-s + b_l nL)),
// each + a fused multiply-add (two FP64 pipe ops per heavy partner).
// The light part depends on the light model only, so row passes stage it
// once per cell for all heavy partners.  SH 2^-s is exact (power of two).
__device__ __forceinline__ double light_part(double bl, double pl, double dnL, double dSLs) {
  return __fma_rn(pl, dSLs, __dmul_rn(bl, dnL));
}
__device__ __forceinline__ double fid_num(double bh, double ph, double dnH, double dSHs, double lp) {
  return __fma_rn(ph, dSHs, __fma_rn(bh, dnH, lp));
}

__device__ __forceinline__ CellVal eval_cell(const Grid& g, const PairConst& pc, int k, int t) {
  const uint32_t* C = slot_cnt(g, pc.slot);
  const uint64_t* S = slot_hs(g, pc.slot);
  const int64_t rk = (int64_t)k * g.B1;
  const uint32_t Rk = C[rk + g.U];
  const uint64_t Rhk = S[rk + g.U];
  const uint64_t Htot = S[(int64_t)g.U * g.B1 + g.U];
  const uint32_t nr = C[rk + t];
  const uint64_t sh_rej = S[rk + t];
  const uint32_t n = (uint32_t)g.n;
  const uint32_t nH = (n - Rk) + nr;
  const uint64_t SH = (Htot - Rhk) + sh_rej;
  const uint64_t SL = Htot - SH;
  CellVal v;
  v.n_keep_light = Rk;
  v.n_heavy = nH;
  const double dn = (double)g.n;
  v.lat = div_n(__dadd_rn(__dmul_rn((double)Rk, pc.Ll), __dmul_rn((double)nH, pc.Lh)), dn, g.rn);
  const double lp = light_part(pc.bl, pc.pl, (double)(n - nH), __dmul_rn((double)SL, g.inv_scale));
  v.fid = div_n(fid_num(pc.bh, pc.ph, (double)nH, __dmul_rn((double)SH, g.inv_scale), lp), dn, g.rn);
  return v;
}

// Division-free numerators: x = (n-nb) L_i + (nb+nr) L_j  (lat = x / n) and
// S = fid* * n.  Both are monotone images of lat / fid*, enough to bucket and filter.
__device__ __forceinline__ void cell_numerators(const Grid& g, const PairConst& pc, int k, int t,
                                                double* x, double* S) {
  const uint32_t* C = slot_cnt(g, pc.slot);
  const uint64_t* Sh = slot_hs(g, pc.slot);
  const int64_t rk = (int64_t)k * g.B1;
  const uint32_t Rk = C[rk + g.U];
  const uint64_t Htot = Sh[(int64_t)g.U * g.B1 + g.U];
  const uint32_t n = (uint32_t)g.n;
  const uint32_t nH = (n - Rk) + C[rk + t];
  const uint64_t SH = (Htot - Sh[rk + g.U]) + Sh[rk + t];
  const uint64_t SL = Htot - SH;
  *x = __dadd_rn(__dmul_rn((double)Rk, pc.Ll), __dmul_rn((double)nH, pc.Lh));
  const double lp = light_part(pc.bl, pc.pl, (double)(n - nH), __dmul_rn((double)SL, g.inv_scale));
  *S = fid_num(pc.bh, pc.ph, (double)nH, __dmul_rn((double)SH, g.inv_scale), lp);
}

// Per-(light slot, k, t) integer statistics, shared by every heavy partner.
struct CellInts {
  uint32_t Rk, nH;       // records kept by the light stage; heavy-served records
  uint64_t SH, SL;       // fixed-point hardness sums of heavy / light-served records
  double dRk, dnH, dnL, dSH, dSL;   // the same, converted once for every partner
};

__device__ __forceinline__ CellInts cell_ints(const Grid& g, const uint32_t* C, const uint64_t* Sh,
                                             int k, int t) {
  const int64_t rk = (int64_t)k * g.B1;
  CellInts c;
  c.Rk = C[rk + g.U];
  const uint64_t Htot = Sh[(int64_t)g.U * g.B1 + g.U];
  c.nH = ((uint32_t)g.n - c.Rk) + C[rk + t];
  c.SH = (Htot - Sh[rk + g.U]) + Sh[rk + t];
  c.SL = Htot - c.SH;
  c.dRk = (double)c.Rk;
  c.dnH = (double)c.nH;
  c.dnL = (double)((uint32_t)g.n - c.nH);
  c.dSH = (double)c.SH;
  c.dSL = (double)c.SL;
  return c;
}

__device__ __forceinline__ void numerators_of(const Grid& g, const PairConst& pc, const CellInts& c,
                                              double* x, double* S) {
  *x = __dadd_rn(__dmul_rn(c.dRk, pc.Ll), __dmul_rn(c.dnH, pc.Lh));
  const double lp = light_part(pc.bl, pc.pl, c.dnL, __dmul_rn(c.dSL, g.inv_scale));
  *S = fid_num(pc.bh, pc.ph, c.dnH, __dmul_rn(c.dSH, g.inv_scale), lp);
}

// bucket of a latency numerator; monotone non-decreasing in x (hence in lat)
__device__ __forceinline__ int bucket_of_x(const PairConst& pc, int nbuckets, double x) {
  // floor without the XU convert: adding 1.5 * 2^52 rounding down leaves
  // floor(y) in the low mantissa word (|y| < 2^51; y < 0 gives -1 -> bucket 0)
  const int b = __double2loint(__dadd_rd(__fma_rn(x, pc.scale_x, pc.off_x), 6755399441055744.0));
  return min(max(b, 0), nbuckets - 1);
}

// exact u32 -> f64 on the FP64 pipe (I2F runs on the 4x slower XU pipe)
__device__ __forceinline__ double u32_to_double(uint32_t v) {
  return __dadd_rn(__hiloint2double(0x43300000, (int)v), -4503599627370496.0);
}

// min of two non-NaN doubles: one FP64-pipe compare + two selects
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// order_key without branches and without folding -0.0 into +0.0: row passes
// only use these keys for minima / value compares, where -0 < +0 is harmless
__device__ __forceinline__ unsigned long long order_key_fast(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return b ^ ((unsigned long long)((long long)b >> 63) | 0x8000000000000000ull);
}

__device__ __forceinline__ int bucket_of(const Grid& g, const PairConst& pc, int k, int t) {
  double x, S;
  cell_numerators(g, pc, k, t, &x, &S);
  return bucket_of_x(pc, g.nbuckets, x);
}

// Is (k, t) the first cell of its exact-duplicate class?  Classes are
// rectangles {row class of k} x {run of equal reject counts along tau}.
__device__ __forceinline__ bool class_start(const Grid& g, const uint32_t* C, int k, int t) {
  if (!g.row_start[k]) return false;
  const int64_t rk = (int64_t)k * g.B1;
  return t == 0 || C[rk + t] != C[rk + t - 1];
}

// Rank with the smallest first position in the tau-run of row k containing t.
__device__ __noinline__ int rep_tau_search(const Grid& g, const uint32_t* C, int k, int t);

__device__ __forceinline__ int rep_tau(const Grid& g, const uint32_t* C, int k, int t,
                                       bool run_start = false) {
  if (run_start && *g.sorted) return t;       // smallest rank == smallest position
  return rep_tau_search(g, C, k, t);
}

// first_pos-smallest rank of t's duplicate run (binary searches along the row)
__device__ __noinline__ int rep_tau_search(const Grid& g, const uint32_t* C, int k, int t) {
  const uint32_t* row = C + (int64_t)k * g.B1;
  const uint32_t v = row[t];
  int lo = 0, hi = t;                         // first index with row[idx] == v
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (row[mid] < v) lo = mid + 1; else hi = mid; }
  const int start = lo;
  if (*g.sorted) return start;
  lo = t + 1; hi = g.U;                       // first index with row[idx] > v
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (row[mid] <= v) lo = mid + 1; else hi = mid; }
  int best = start;
  for (int i = start + 1; i < lo; ++i)
    if (g.first_pos[i] < g.first_pos[best]) best = i;
  return best;
}

// representative (smallest grid index) cell of (k, t)'s duplicate class
__device__ __forceinline__ uint32_t rep_cell(const Grid& g, const uint32_t* C, int k, int t,
                                             bool run_start = false) {
  return (uint32_t)(g.row_rep[k] * g.U + rep_tau(g, C, k, t, run_start));
}

__device__ __forceinline__ int64_t grid_index(const Grid& g, int k, int t) {
  return (int64_t)g.first_pos[k] * g.K + g.first_pos[t];
}

// equal heavy sets H(k1,t1) == H(k2,t2) from prefix counts (exact)
__device__ bool same_heavy(const Grid& g, int slot, int k1, int t1, int k2, int t2) {
  if (k1 > k2) { int x = k1; k1 = k2; k2 = x; x = t1; t1 = t2; t2 = x; }
  const uint32_t* C = slot_cnt(g, slot);
  const uint32_t n = (uint32_t)g.n;
  const int64_t r1 = (int64_t)k1 * g.B1, r2 = (int64_t)k2 * g.B1;
  const uint32_t h1 = (n - C[r1 + g.U]) + C[r1 + t1];
  const uint32_t h2 = (n - C[r2 + g.U]) + C[r2 + t2];
  if (h1 != h2) return false;
  const int tm = t1 < t2 ? t1 : t2;
  const uint32_t inter = (n - C[r2 + g.U]) + (C[r2 + t2] - C[r1 + t2]) + C[r1 + tm];
  return inter == h1;
}

// ---------------------------------------------------------------- F0: setup

__global__ void pair_const_kernel(int n_pairs, const int32_t* __restrict__ pair_slot,
                                  const double* __restrict__ params, int64_t n, int shift,
                                  int nbuckets, PairConst* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const double* q = params + (int64_t)p * HADIS_PAIR_PARAMS;
  PairConst c;
  c.Ll = q[0]; c.Lh = q[1]; c.bl = q[2]; c.pl = q[3]; c.bh = q[4]; c.ph = q[5];
  c.slot = pair_slot[p];
  // |numpy pairwise mean - fid*| <= (D + 16) u Fmax + maxpen * n * 2^-shift / n,
  // D <= 96 covers numpy's recursion for any n < 2^64; doubled for margin.
  const double u = ldexp(1.0, -53);
  const double fbig = fmax(fabs(c.bl) + fabs(c.pl), fabs(c.bh) + fabs(c.ph));
  const double pmax = fmax(fabs(c.pl), fabs(c.ph));
  const double delta = 2.0 * (128.0 * u * fbig + pmax * ldexp(1.0, -shift)) + DBL_MIN;
  c.delta2 = 2.0 * delta;
  const double dn = (double)n;
  c.delta2_S = c.delta2 * dn * 1.001;
  const double lo = fmin(c.Ll, c.Lh) * dn * (1.0 - 1e-12);
  const double hi = (c.Ll + c.Lh) * dn * (1.0 + 1e-12);
  c.scale_x = (double)nbuckets / (hi - lo);
  c.off_x = -lo * c.scale_x;
  out[p] = c;
}

// Row classes (ranks with equal R[k] = #{bh <= k}; light-model independent):
//   pk[k]        largest k' < k with R[k'] < R[k] (else -1): canonical heavy-set twin row
//   row_start[k] k starts its class;  row_rep[k] class member with the smallest first_pos
__global__ void __launch_bounds__(1024)
row_classes_kernel(const uint32_t* __restrict__ cnt, int U, int B1,
                   const int32_t* __restrict__ first_pos, int32_t* pk, int32_t* row_rep,
                   uint8_t* row_start, int32_t* sorted) {
  // Classes are runs of equal R.  Each thread owns a contiguous segment of ranks;
  // three block scans give every rank its run start a (max-scan of starts), its
  // run end b (reverse min-scan of starts) and the run's first_pos-smallest rank
  // (segmented min-scan of (first_pos, rank) keys, read at the run's last rank).
  // (One walk per rank to its run's ends was O(run^2): 13 us at c4.)
  extern __shared__ __align__(8) unsigned char rc_smem[];
  long long* s_runmin = reinterpret_cast<long long*>(rc_smem);   // [U] min key over [a(k), k]
  uint32_t* s_R = reinterpret_cast<uint32_t*>(s_runmin + U);      // [U]
  __shared__ int s_unsorted;
  __shared__ long long s_w[32];
  const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (U + T - 1) / T, k0 = min(U, tid * per), k1 = min(U, k0 + per);
  if (tid == 0) s_unsorted = 0;
  __syncthreads();
  for (int k = tid; k < U; k += T) {
    s_R[k] = cnt[(int64_t)k * B1 + U];
    if (k > 0 && first_pos[k] < first_pos[k - 1]) s_unsorted = 1;
  }
  __syncthreads();
  if (tid == 0) *sorted = !s_unsorted;
  auto is_start = [&](int k) { return k == 0 || s_R[k - 1] != s_R[k]; };
  // generic exclusive block scan over the thread totals (op: associative, id: identity)
  auto block_excl = [&](long long v, long long id, auto op) {
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = op(x, y);
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
      long long w = lane < (T >> 5) ? s_w[lane] : id;
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w = op(w, y);
      }
      s_w[lane] = w;
    }
    __syncthreads();
    long long e = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) e = id;
    const long long pre = wid > 0 ? s_w[wid - 1] : id;
    const long long r = op(pre, e);
    __syncthreads();
    return r;
  };
  auto mx = [](long long x, long long y) { return x > y ? x : y; };
  auto mn = [](long long x, long long y) { return x < y ? x : y; };
  // 1. run start a(k): last start <= k
  long long t = -1;
  for (int k = k0; k < k1; ++k) if (is_start(k)) t = k;
  long long run_a = block_excl(t, -1, mx);
  // 2. run end b(k): first start > k (reverse scan: threads in reverse order)
  long long u = U;
  for (int k = k1 - 1; k >= k0; --k) if (is_start(k)) u = k;
  // exclusive min over higher threads = reverse exclusive scan: scan the mirrored thread ids
  // (implemented as a min over all threads > tid through shared memory)
  __shared__ int s_first_start[1024];
  s_first_start[tid] = (int)u;
  __syncthreads();
  for (int o = 1; o < T; o <<= 1) {                 // suffix min across threads (log steps)
    const int v = tid + o < T ? s_first_start[tid + o] : U;
    __syncthreads();
    if (v < s_first_start[tid]) s_first_start[tid] = v;
    __syncthreads();
  }
  int run_b = tid + 1 < T ? s_first_start[tid + 1] : U;
  // 3. segmented min of (first_pos << 32 | rank), restarted at run starts
  const long long kInf = 0x7fffffffffffffffll;
  long long seg = kInf;
  bool has_start = false;
  for (int k = k0; k < k1; ++k) {
    const long long key = ((long long)first_pos[k] << 32) | (unsigned)k;
    if (is_start(k)) { seg = key; has_start = true; } else seg = mn(seg, key);
  }
  // carry across threads: (has_start, seg) pairs combine as a segmented min
  // encoded as "reset" flag in the top bit handled by two scans: the carry into a
  // thread is the min over the preceding threads back to the last one with a start
  __shared__ long long s_seg[1024];
  __shared__ int s_has[1024];
  s_seg[tid] = seg;
  s_has[tid] = has_start;
  __syncthreads();
  long long carry = kInf;
  for (int j = tid - 1; j >= 0; --j) {              // runs span few threads: short walk
    carry = mn(carry, s_seg[j]);
    if (s_has[j]) break;
  }
  // final pass: every rank's a, b and the run minimum
  long long cur_a = run_a, cur = carry;
  for (int k = k0; k < k1; ++k) {
    const long long key = ((long long)first_pos[k] << 32) | (unsigned)k;
    if (is_start(k)) { cur_a = k; cur = key; } else cur = mn(cur, key);
    s_runmin[k] = cur;                              // min over [a(k), k]
    pk[k] = (int32_t)cur_a - 1;
    row_start[k] = is_start(k);
  }
  __syncthreads();
  long long nb = run_b;
  for (int k = k1 - 1; k >= k0; --k) {
    if (k + 1 < U && is_start(k + 1)) nb = k + 1;
    row_rep[k] = (int32_t)(s_runmin[nb - 1] & 0xffffffffll);
  }
}

// ---------------------------------------------------------- F1: bucket minima


// Pairs sharing a light slot are contiguous ("groups"); a thread loads one
// (slot, k, t) cell's integer statistics once and evaluates every heavy
// partner of the group.  grid: (cell tiles, group upper bound), x fastest, so
// one light model's prefix table stays L2-resident while its pairs run.
__global__ void group_kernel(const int32_t* __restrict__ pair_slot, int n_pairs,
                             int32_t* __restrict__ group_p0, int32_t* __restrict__ n_groups,
                             unsigned long long* counters, int max_group) {
  // one warp: group starts by ballot, 32 pairs per step (was one thread: 10 us)
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int ng = 0;
  for (int p0 = 0; p0 < n_pairs; p0 += 32) {
    const int p = p0 + lane;
    const bool start = p < n_pairs && (p == 0 || pair_slot[p] != pair_slot[p - 1]);
    const unsigned m = __ballot_sync(0xffffffffu, start);
    if (start) group_p0[ng + __popc(m & ((1u << lane) - 1u))] = p;
    ng += __popc(m);
  }
  if (lane == 0) group_p0[ng] = n_pairs;
  __syncwarp();
  bool too_big = false;
  for (int i = lane; i < ng; i += 32) too_big |= group_p0[i + 1] - group_p0[i] > max_group;
  if (__any_sync(0xffffffffu, too_big)) {            // > 65 pool models: unsupported
    if (lane == 0) counters[4] |= 128ull;
    ng = 0;
  }
  if (lane == 0) *n_groups = ng;
}

struct __align__(16) Cand {
  uint32_t pair, cell, bucket, pad;   // cell = k * U + t (representative)
  double lat, fid;
};
struct Cands {
  Cand* c;
};

// F3's unordered candidate list: 16 bytes (x and the bucket are recomputed
// from the cell in F5, bit-identically: same prefix-table counts, same ops)
struct __align__(16) ListCand {
  uint32_t pair, cell;   // cell = k * U + t (representative)
  double S;              // fid* numerator
};

// Row passes F1 / F3.  One warp per (light slot, theta rank k); a CTA holds
// kRowWarps rows of one slot group.  Along a row the latency numerator x is
// non-decreasing in t (the reject count is), so a cell whose S exceeds the
// exclusive prefix-min of S over the earlier cells of its row is dominated by
// one of them (lat <=, fid* <).  The row is walked in windows of kRowWin
// cells: the warp stages the window's statistics in shared memory (nH as u32,
// the hardness terms as doubles; shared by every heavy partner of the slot);
// per partner, lane l evaluates
// its kRowT contiguous cells, one warp scan of the lane minima gives each
// lane its carry-in, and the per-cell test is one compare.  The [j][33]
// layout keeps staging stores and per-lane reads conflict-free.  Rows that
// repeat an earlier row's R[k] (same row class) are exact duplicates and are
// skipped.
#ifndef HADIS_ROW_FSCAN
#define HADIS_ROW_FSCAN 1      // float upper-bound row scan (c4: -18 us, same candidates)
#endif
constexpr int kRowWarps = 8;         // rows per CTA (4: no gain)
constexpr int kCoarseShift = 4;      // F1/F3 latency buckets: the fine ones >> 4
                                     // (3 and 5 measured: F1 vs candidate trade-off, no gain)
constexpr int kMaxGroup = 64;        // heavy partners per light slot (pool <= 65 models)
constexpr int kRowT = 4;             // cells per lane per window (8: F3 +40 us; 2: slower)
constexpr int kRowWin = 32 * kRowT;  // cells per window
constexpr int kRowPad = 33;

struct RowSmem {
  uint32_t nH[kRowWarps][kRowT * kRowPad];  // heavy-served records (u32: 4 CTAs/SM fit)
  double2 hl[kRowWarps][kRowT * kRowPad];   // (hardness sum * 2^-shift, light part of S)
  double carry[kRowWarps][kMaxGroup];
  PairConst pc[kMaxGroup];
};

__device__ __forceinline__ bool row_task(const Grid& g, const PairConst* __restrict__ pcs,
                                         const int32_t* __restrict__ group_p0,
                                         const int32_t* __restrict__ n_groups, RowSmem& sm,
                                         int* p0, int* p1, int* k, int kstride = 1,
                                         int pchunks = 1) {
  const int grp = blockIdx.y / pchunks;
  if (grp >= *n_groups) return false;
  *p0 = group_p0[grp];
  *p1 = group_p0[grp + 1];
  if (pchunks > 1) {                               // this CTA's share of the partners
    const int cs = (*p1 - *p0 + pchunks - 1) / pchunks;
    *p0 += (blockIdx.y % pchunks) * cs;
    *p1 = min(*p1, *p0 + cs);
    if (*p0 >= *p1) return false;
  }
  const int np = *p1 - *p0;                      // <= kMaxGroup (checked on the host)
  for (int i = threadIdx.x; i < np * (int)(sizeof(PairConst) / 8); i += blockDim.x)
    reinterpret_cast<double*>(sm.pc)[i] = reinterpret_cast<const double*>(pcs + *p0)[i];
  __syncthreads();
  *k = (blockIdx.x * kRowWarps + (threadIdx.x >> 5)) * kstride;
  return *k < g.U && g.row_start[*k];
}

// visit(p, pc, w0, sv[kRowT], take) once per (window, partner), all lanes:
// lane l owns cells t = w0 + l*kRowT + j; sv[j] = S (+inf past the row end;
// minima and compares run on the FP64 pipe, which has the slack -- u64 keys
// cost four ALU ops per min); bit j of take = the cell passes the row test -- strict
// prefix-min (F1) or class start within 2 delta of the prefix-min (F3).
template <bool kFilter, typename F, typename W, typename P>
__device__ __forceinline__ void row_traverse(const Grid& g, RowSmem& sm, int p0, int p1, int k,
                                             F&& visit, W&& window_done, P&& pre) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* C = slot_cnt(g, sm.pc[0].slot);
  const uint64_t* Sh = slot_hs(g, sm.pc[0].slot);
  const int64_t rk = (int64_t)k * g.B1;
  const uint32_t n = (uint32_t)g.n;
  const uint32_t Rk = C[rk + g.U];
  const uint64_t Htot = Sh[(int64_t)g.U * g.B1 + g.U];
  const uint64_t Hnb = Htot - Sh[rk + g.U];        // hardness of bypassed records
  const double bl = sm.pc[0].bl, pl = sm.pc[0].pl, inv = g.inv_scale;
  uint32_t* s_nH = sm.nH[warp];
  double2* s_hl = sm.hl[warp];
  {
    const int q0 = p0, q1 = p1;
    for (int p = q0 + lane; p < q1; p += 32) sm.carry[warp][p - q0] = INFINITY;
    for (int w0 = 0; w0 < g.U; w0 += kRowWin) {
      __syncwarp();
      // stage: all kRowT coalesced loads of the window in flight, then convert
      uint32_t nrv[kRowT];
      uint64_t shv[kRowT];
#pragma unroll
      for (int r = 0; r < kRowT; ++r) {
        const int t = w0 + r * 32 + lane;
        nrv[r] = t < g.U ? C[rk + t] : 0u;
        shv[r] = t < g.U ? Sh[rk + t] : 0ull;
      }
      uint32_t prev = w0 > 0 ? C[rk + w0 - 1] : 0u;  // C at the cell before the window
      uint32_t cls_m[kRowT];                       // bit l of cls_m[r]: cell r*32+l starts its class
#pragma unroll
      for (int r = 0; r < kRowT; ++r) {
        const int i = r * 32 + lane, t = w0 + i;
        const int at = (i % kRowT) * kRowPad + i / kRowT;
        uint32_t left = __shfl_up_sync(0xffffffffu, nrv[r], 1);
        if (lane == 0) left = prev;
        prev = __shfl_sync(0xffffffffu, nrv[r], 31);
        if (t < g.U) {
          const uint32_t nr = nrv[r];
          const uint64_t SH = Hnb + shv[r];
          const uint32_t nH = (n - Rk) + nr;
          s_nH[at] = nH;
          s_hl[at] = make_double2(__dmul_rn((double)SH, inv),
                                  light_part(bl, pl, (double)(n - nH),
                                             __dmul_rn((double)(Htot - SH), inv)));
        } else {                                         // past the row end: S = +inf
          s_nH[at] = 0u;
          s_hl[at] = make_double2(0.0, INFINITY);
        }
        cls_m[r] = __ballot_sync(0xffffffffu, t < g.U && (t == 0 || nrv[r] != left));
      }
      // this lane's cells are w0 + 4 lane + j: bits 4 (lane % 8) + j of cls_m[lane / 8]
      const int qr = lane >> 3;
      const uint32_t cls4 =
          ((qr == 0 ? cls_m[0] : qr == 1 ? cls_m[1] : qr == 2 ? cls_m[2] : cls_m[3]) >>
           (4 * (lane & 7))) & 15u;
      static_assert(kRowT == 4, "class-start bits: 4 cells per lane");
      __syncwarp();
      // the lane's cells, read from the staged window once for all partners
      // (c4: -18 us against shared-memory reads per partner)
      double2 r_hl[kRowT];
      uint32_t r_nH[kRowT];
#pragma unroll
      for (int j = 0; j < kRowT; ++j) {
        r_hl[j] = s_hl[j * kRowPad + lane];
        r_nH[j] = s_nH[j * kRowPad + lane];
      }
      // one partner: S of the lane's cells, warp scan of the lane minima (the
      // row carry enters through lane 0, so only lane 0 touches it), row test
      auto scan = [&](int p, double (&sv)[kRowT]) -> unsigned {
        const PairConst& pc = sm.pc[p - p0];
        const double ph = pc.ph, bh = pc.bh;
        double lmin = INFINITY;
#pragma unroll
        for (int j = 0; j < kRowT; ++j) {
          const double2 v = r_hl[j];
          sv[j] = fid_num(bh, ph, u32_to_double(r_nH[j]), v.x, v.y);
          lmin = dmin(lmin, sv[j]);
        }
        double* const carry = &sm.carry[warp][p - q0];
        const double c0 = lane == 0 ? *carry : INFINITY;
#if HADIS_ROW_FSCAN
        // scan of upper bounds in float (rounded up): run / carry may exceed
        // the exact prefix minima, so the row tests only keep MORE cells
        float fincl = __double2float_ru(dmin(lmin, c0));
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float o = __shfl_up_sync(0xffffffffu, fincl, off);
          if (lane >= off) fincl = fminf(fincl, o);
        }
        double run = (double)__shfl_up_sync(0xffffffffu, fincl, 1);
        const double tot = (double)__shfl_sync(0xffffffffu, fincl, 31);
#else
        double incl = dmin(lmin, c0);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double o = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl = dmin(incl, o);
        }
        double run = __shfl_up_sync(0xffffffffu, incl, 1);
        const double tot = __shfl_sync(0xffffffffu, incl, 31);
#endif
        if (lane == 0) {
          run = c0;
          *carry = tot;
        }
        unsigned take = 0;
        const double dpc = pc.delta2_S;
#pragma unroll
        for (int j = 0; j < kRowT; ++j) {
          bool t_ok;
          if (kFilter) {
            t_ok = ((cls4 >> j) & 1u) && sv[j] <= run + dpc;
          } else {
            t_ok = sv[j] < run;
          }
          take |= (unsigned)t_ok << j;
          run = dmin(run, sv[j]);
        }
        return take;
      };
      for (int p = q0; p < q1; ++p) {
        double sv[kRowT];
        pre(p, sm.pc[p - p0], r_nH);                     // loads that need no scan result
        const unsigned take = scan(p, sv);
        visit(p, sm.pc[p - p0], w0, sv, take);
      }
      window_done(w0);                             // staged window still valid here
    }
    __syncwarp();
  }
}

// F1: per (pair, latency bucket) minimum of S over the row-frontier cells --
// enough for the EXCLUSIVE bucket prefix minima (a cell dropped here is
// dominated by an earlier cell of its row, which sits in the same or a lower
// bucket).  Reads the current minima first (all in flight): most cells do
// not lower them.
// Sampled: F1 walks every kstride-th theta-row only.  Every minimum is still
// a real cell's S, so the prefix minima G' >= G remain valid domination
// certificates for F3; they are only weaker (c4, measured: stride 4 -> F1
// 314 -> ~115 us, candidates 12.4M -> 13.9M, step -145 us; strides 2 / 3 /
// 5 / 6 / 8 / 16 and 1 / 4 / 8 partner chunks per row: slower).  Skipping
// windows above a sampled snapshot in a second full F1 pass, or whole F3
// windows above G at their first cell, measured no gain: the row walk
// itself, not the per-cell bucket work, is F1/F3's cost.
__global__ void __launch_bounds__(kRowWarps * 32, 32 / kRowWarps)   // 4 CTAs/SM at 8 warps
bucket_min_kernel(Grid g, const PairConst* __restrict__ pcs, const int32_t* __restrict__ group_p0,
                  const int32_t* __restrict__ n_groups, unsigned long long* __restrict__ bmin,
                  int kstride, int pchunks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  int p0, p1, k;
  if (!row_task(g, pcs, group_p0, n_groups, sm, &p0, &p1, &k, kstride, pchunks)) return;
  const double dRk = (double)slot_cnt(g, sm.pc[0].slot)[(int64_t)k * g.B1 + g.U];
  int bk[kRowT];
  unsigned long long cur[kRowT];
  row_traverse<false>(g, sm, p0, p1, k, [&](int p, const PairConst&, int,
                                            const double* sv, unsigned take) {
    unsigned long long* const bp = bmin + (int64_t)p * (g.nbuckets >> kCoarseShift);
    // row-frontier keys strictly decrease along the walk: of consecutive taken
    // cells in one coarse bucket only the last can lower its minimum
#pragma unroll
    for (int j = 0; j + 1 < kRowT; ++j)
      if ((take >> (j + 1) & 1u) && bk[j + 1] == bk[j]) take &= ~(1u << j);
#pragma unroll
    for (int j = 0; j < kRowT; ++j) {
      const unsigned long long key = order_key_fast(sv[j]);
      if ((take >> j & 1u) && key < cur[j]) atomicMin(bp + bk[j], key);
    }
  }, [](int) {}, [&](int p, const PairConst& pc, const uint32_t (&nHr)[kRowT]) {
    // every cell's coarse bucket and current minimum, loaded before the row
    // scan so their latency overlaps it (past the row end: bucket of nH = 0)
    const unsigned long long* const bp = bmin + (int64_t)p * (g.nbuckets >> kCoarseShift);
    const double xr = __dmul_rn(dRk, pc.Ll);
#pragma unroll
    for (int j = 0; j < kRowT; ++j) {
      bk[j] = bucket_of_x(pc, g.nbuckets, __dadd_rn(xr, __dmul_rn(u32_to_double(nHr[j]), pc.Lh))) >>
              kCoarseShift;
      cur[j] = bp[bk[j]];
    }
  });
}

// ------------------------------------------------- F2: exclusive prefix minima

constexpr int kScanThreads = 1024;

__device__ __forceinline__ unsigned long long block_exclusive_min(unsigned long long v,
                                                                  unsigned long long* total) {
  __shared__ unsigned long long warp_min[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl = min(incl, o);
  }
  unsigned long long excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = ~0ull;
  if (lane == 31) warp_min[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    unsigned long long w = lane < nw ? warp_min[lane] : ~0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w = min(w, o);
    }
    if (lane < nw) warp_min[lane] = w;
  }
  __syncthreads();
  const unsigned long long before = warp > 0 ? min(warp_min[warp - 1], excl) : excl;
  *total = warp_min[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

// per pair: exclusive prefix-min over bucket minima, in three grid-wide phases
// (tile minima -> per-pair scan of tile minima -> in-tile scan with carry)
constexpr int kPrefTile = 4 * kScanThreads;

__global__ void __launch_bounds__(kScanThreads)
prefix_tile_min_kernel(const unsigned long long* __restrict__ bmin, int nbuckets,
                       unsigned long long* __restrict__ tmin) {
  const int p = blockIdx.y, tile = blockIdx.x;
  const int i0 = tile * kPrefTile + 4 * threadIdx.x;
  const unsigned long long* src = bmin + (int64_t)p * nbuckets;
  unsigned long long m = ~0ull;
  if ((nbuckets & 3) == 0 && i0 + 3 < nbuckets) {          // two 16-byte loads
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(src + i0);
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(src + i0 + 2);
    m = min(min(a.x, a.y), min(b.x, b.y));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) if (i0 + j < nbuckets) m = min(m, src[i0 + j]);
  }
  unsigned long long total;
  block_exclusive_min(m, &total);
  if (threadIdx.x == 0) tmin[(int64_t)p * gridDim.x + tile] = total;
}

__global__ void prefix_carry_kernel(unsigned long long* __restrict__ tmin, int tiles, int n_pairs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  unsigned long long run = ~0ull;
  for (int t = 0; t < tiles; ++t) {
    const unsigned long long v = tmin[(int64_t)p * tiles + t];
    tmin[(int64_t)p * tiles + t] = run;          // exclusive
    run = min(run, v);
  }
}

__global__ void __launch_bounds__(kScanThreads)
prefix_apply_kernel(const unsigned long long* __restrict__ bmin, int nbuckets,
                    const unsigned long long* __restrict__ tcarry, double* __restrict__ gpre) {
  const int p = blockIdx.y, tile = blockIdx.x;
  const int i0 = tile * kPrefTile + 4 * threadIdx.x;
  const unsigned long long* src = bmin + (int64_t)p * nbuckets;
  double* dst = gpre + (int64_t)p * nbuckets;
  unsigned long long v[4];
  unsigned long long m = ~0ull;
  const bool vec = (nbuckets & 3) == 0 && i0 + 3 < nbuckets;   // 16-byte loads / stores
  if (vec) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(src + i0);
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(src + i0 + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = i0 + j < nbuckets ? src[i0 + j] : ~0ull;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) m = min(m, v[j]);
  unsigned long long total;
  unsigned long long run = min(tcarry[(int64_t)p * gridDim.x + tile], block_exclusive_min(m, &total));
  double o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    o[j] = run == ~0ull ? INFINITY : from_order_key(run);
    run = min(run, v[j]);
  }
  if (vec) {
    *reinterpret_cast<double2*>(dst + i0) = make_double2(o[0], o[1]);
    *reinterpret_cast<double2*>(dst + i0 + 2) = make_double2(o[2], o[3]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) if (i0 + j < nbuckets) dst[i0 + j] = o[j];
  }
}

// ------------------------------------------------------------- F3: filter

// ---------------------------------------------- F4: offsets (exclusive scan)

// (the bucket and chunk offsets are CUB scans, see count_offsets; the block
// scan below serves emit)

__device__ __forceinline__ unsigned long long block_exclusive_sum(unsigned long long v,
                                                                  unsigned long long* total) {
  __shared__ unsigned long long warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    unsigned long long ws = lane < nw ? warp_sums[lane] : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, ws, off);
      if (lane >= off) ws += o;
    }
    if (lane < nw) warp_sums[lane] = ws;
  }
  __syncthreads();
  const unsigned long long before = (warp > 0 ? warp_sums[warp - 1] : 0ull) + incl - v;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}


// --------------------------------------------------------------- F6: decide

struct Uncertain {
  uint32_t* universe;
  uint32_t* pair;
  uint32_t* cell;
};

__device__ __forceinline__ void set_bit(uint32_t* bm, int64_t bit) {
  atomicOr(&bm[bit >> 5], 1u << (bit & 31));
}
__device__ __forceinline__ bool get_bit(const uint32_t* bm, int64_t bit) {
  return (bm[bit >> 5] >> (bit & 31)) & 1u;
}

// Request numpy-exact fidelity for a cell (deduplicated through a bitmap).
__device__ void request_exact(int64_t cells, int p, uint32_t cell, uint32_t* req_bm,
                              uint32_t* req_pair, uint32_t* req_cell, int64_t cap,
                              unsigned long long* counters) {
  const int64_t bit = (int64_t)p * cells + cell;
  const uint32_t m = 1u << (bit & 31);
  const uint32_t old = atomicOr(&req_bm[bit >> 5], m);
  if (old & m) return;
  const unsigned long long at = atomicAdd(&counters[2], 1ull);
  if ((int64_t)at < cap) { req_pair[at] = (uint32_t)p; req_cell[at] = cell; }
}

__device__ void push_uncertain(int universe, int p, uint32_t cell, Uncertain un, int64_t cap,
                               unsigned long long* counters) {
  const unsigned long long at = atomicAdd(&counters[1], 1ull);
  if ((int64_t)at < cap) { un.universe[at] = universe; un.pair[at] = p; un.cell[at] = cell; }
}

// kill(d, c) for d with lat_d <= lat_c, given fidelities known to be comparable
__device__ __forceinline__ bool kills(double fd, double fc, double lat_d, double lat_c,
                                      int64_t idx_d, int64_t idx_c) {
  return fd < fc || (fd == fc && (lat_d < lat_c || idx_d < idx_c));
}

struct DecideOut {
  uint32_t* kept_bm;
  Uncertain un;
  int64_t ucap;
  uint32_t* req_bm;
  uint32_t* req_pair;
  uint32_t* req_cell;
  int64_t rcap;
  unsigned long long* counters;
};

// Certified main-universe decision for candidate `self` (pair p, representative
// cell, bucket-mates grp[s0, s1)); G_S = exclusive prefix-min numerator of its
// bucket.  Keeps, drops or queues the cell for the exact-fidelity resolution.
template <typename Mate>
__device__ void decide_one(const Grid& g, const PairConst& pc, int p, uint32_t cell, double lat,
                           double fid, double G_S, const Cands& grp, int64_t s0, int64_t s1,
                           int64_t self, const DecideOut& o, Mate&& mate) {
  const int k = (int)(cell / g.U), t = (int)(cell % g.U);
  const int64_t idx = grid_index(g, k, t);
  bool killed = false, unsure = false;
  // fl(S / n) is exactly the lower buckets' min fid*
  const double G = div_n(G_S, (double)g.n, g.rn);
  if (G < fid - pc.delta2) {
    killed = true;
  } else if (G <= fid + pc.delta2) {
    // a lower-bucket cell is close: certain only if it is this cell's
    // heavy-set twin with more bypass (equal fidelity, strictly lower latency)
    unsure = true;
    const int kp = g.pk[k];
    if (kp >= 0) {
      const uint32_t* C = slot_cnt(g, pc.slot);
      const int64_t rk = (int64_t)k * g.B1, rp = (int64_t)kp * g.B1;
      if (C[rk + t] - C[rp + t] == C[rk + g.U] - C[rp + g.U]) {
        const CellVal tw = eval_cell(g, pc, kp, t);
        if (tw.lat < lat) {
          killed = true;
        } else if (tw.lat == lat) {
          const uint32_t tc = rep_cell(g, C, kp, t);
          if (grid_index(g, (int)(tc / g.U), (int)(tc % g.U)) < idx) killed = true;
        }
      }
    }
  }
  for (int64_t j = s0; j < s1 && !killed; ++j) {
    if (j == self) continue;
    const double2 lf = mate(j);               // (lat, fid) of bucket-mate j
    const double ld = lf.x;
    if (ld > lat) continue;
    const double fd = lf.y;
    if (fabs(fd - fid) > pc.delta2) {
      if (fd < fid) killed = true;
      continue;
    }
    const uint32_t dc = grp.c[j].cell;
    const int kd = (int)(dc / g.U), td = (int)(dc % g.U);
    if (same_heavy(g, pc.slot, kd, td, k, t)) {
      if (ld < lat || grid_index(g, kd, td) < idx) killed = true;
    } else {
      unsure = true;
    }
  }
  if (killed) return;
  const int64_t cells = (int64_t)g.U * g.U;
  if (!unsure) {
    set_bit(o.kept_bm, (int64_t)p * g.bm_stride + cell);
  } else {
    push_uncertain(0, p, cell, o.un, o.ucap, o.counters);
    request_exact(cells, p, cell, o.req_bm, o.req_pair, o.req_cell, o.rcap, o.counters);
  }
}

// F3: candidates = class-start cells within 2 delta (numerator space) of both
// their row's prefix minimum and their bucket's exclusive prefix minimum.
// Per window the partners' pass masks go to shared memory; one list
// reservation per (warp, window) for all partners (the reservation atomic's
// round trip was the kernel's largest stall), then the candidates are
// re-evaluated from the staged window (same formulas, bit-identical values),
// counted per (pair, fine bucket) and appended; F5 groups them by bucket.
__global__ void __launch_bounds__(kRowWarps * 32, 32 / kRowWarps)   // 4 CTAs/SM (3, 5, 6: slower)
filter_kernel(Grid g, const PairConst* __restrict__ pcs, const int32_t* __restrict__ group_p0,
              const int32_t* __restrict__ n_groups, const double* __restrict__ gpre,
              uint32_t* __restrict__ bcnt, ListCand* __restrict__ lst, int64_t cap,
              unsigned long long* __restrict__ n_list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  int p0, p1, k;
  if (!row_task(g, pcs, group_p0, n_groups, sm, &p0, &p1, &k)) return;
  const uint32_t* C = slot_cnt(g, sm.pc[0].slot);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* const s_take = smem_raw + sizeof(RowSmem) + warp * (kMaxGroup * 32);
  const uint32_t krep = (uint32_t)g.row_rep[k] * (uint32_t)g.U;
  const bool sorted_thr = *g.sorted != 0;          // first_pos increasing: rep = own rank
  const double dRk = (double)C[(int64_t)k * g.B1 + g.U];
  const uint32_t* s_nH = sm.nH[warp];
  const double2* s_hl = sm.hl[warp];
  int cnt = 0;                                     // this lane's candidates in the window
  double gv[kRowT];
  row_traverse<true>(g, sm, p0, p1, k, [&](int p, const PairConst& pc, int,
                                           const double* sv, unsigned take) {
#pragma unroll
    for (int j = 0; j < kRowT; ++j)
      if (!(sv[j] <= gv[j] + pc.delta2_S)) take &= ~(1u << j);
    s_take[(p - p0) * 32 + lane] = (uint8_t)take;
    cnt += __popc(take);
  }, [&](int w0) {
    const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
    cnt = 0;
    if (total == 0) return;
    unsigned long long at0 = 0;
    if (lane == 0) at0 = atomicAdd(n_list, (unsigned long long)total);
    int64_t base = (int64_t)__shfl_sync(0xffffffffu, at0, 0);
    for (int p = p0; p < p1; ++p) {                // partner-major, lane-contiguous runs
      const unsigned tk = s_take[(p - p0) * 32 + lane];
      const int c = __popc(tk);
      int incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (tot == 0) continue;
      int64_t at = base + incl - c;
      base += tot;
      const PairConst& pc = sm.pc[p - p0];
      const double xr = __dmul_rn(dRk, pc.Ll);
#pragma unroll
      for (int j = 0; j < kRowT; ++j) {
        if (!(tk >> j & 1u)) continue;
        const int a = j * kRowPad + lane;
        const double dnH = u32_to_double(s_nH[a]);
        const double x = __dadd_rn(xr, __dmul_rn(dnH, pc.Lh));
        const int b = bucket_of_x(pc, g.nbuckets, x);
        atomicAdd(&bcnt[(int64_t)p * g.nbuckets + b], 1u);
        if (at < cap) {
          // raw numerators; F5 divides (lat = x / n, fid* = S / n)
          const int t = w0 + lane * kRowT + j;
          lst[at] = ListCand{(uint32_t)p,
                             krep + (uint32_t)(sorted_thr ? t : rep_tau(g, C, k, t, true)),
                             fid_num(pc.bh, pc.ph, dnH, s_hl[a].x, s_hl[a].y)};
        }
        ++at;
      }
    }
  }, [&](int p, const PairConst& pc, const uint32_t (&nHr)[kRowT]) {
    // every cell's bucket prefix minimum, loaded before the row scan so the
    // latency overlaps it
    const double* const gp = gpre + (int64_t)p * (g.nbuckets >> kCoarseShift);
    const double xr = __dmul_rn(dRk, pc.Ll);
#pragma unroll
    for (int j = 0; j < kRowT; ++j)
      gv[j] = gp[bucket_of_x(pc, g.nbuckets, __dadd_rn(xr, __dmul_rn(u32_to_double(nHr[j]), pc.Lh))) >>
                 kCoarseShift];
  });
}

// F5: group the candidate list by (pair, bucket) with the scanned counts
__global__ void group_cands_kernel(Grid g, const PairConst* __restrict__ pcs,
                                   const ListCand* __restrict__ lst,
                                   const unsigned long long* __restrict__ n_list,
                                   int64_t cap, int nbuckets, double dn,
                                   const unsigned long long* __restrict__ boff,
                                   uint32_t* __restrict__ bcur, Cands grp,
                                   unsigned long long* __restrict__ fmin) {
  if ((int64_t)*n_list > cap) return;
  const int64_t m = (int64_t)*n_list;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t n = (uint32_t)g.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const ListCand lc = lst[i];
    const PairConst& pc = pcs[lc.pair];
    // x exactly as F3 formed it: the representative cell has the same (R_k, nr)
    const uint32_t* C = slot_cnt(g, pc.slot);
    const uint32_t k = lc.cell / (uint32_t)g.U, t = lc.cell - k * (uint32_t)g.U;
    const uint32_t Rk = C[(int64_t)k * g.B1 + g.U];
    const uint32_t nH = (n - Rk) + C[(int64_t)k * g.B1 + t];
    const double x = __dadd_rn(__dmul_rn((double)Rk, pc.Ll), __dmul_rn((double)nH, pc.Lh));
    Cand cd{lc.pair, lc.cell, (uint32_t)bucket_of_x(pc, nbuckets, x), 0u, x, lc.S};
    const int64_t key = (int64_t)cd.pair * nbuckets + cd.bucket;
    // fine-bucket minima over the candidates: every cell F1/F3 pruned is
    // beaten by a candidate at lower-or-equal latency, so the exclusive
    // prefix of these minima is the exact fine G
    atomicMin(&fmin[key], (unsigned long long)order_key(cd.fid));
    cd.lat = div_n(cd.lat, dn, g.rn);     // the list holds raw numerators
    cd.fid = div_n(cd.fid, dn, g.rn);
    // in-bucket slot: the bucket's count, consumed downwards (no cursor array to zero)
    grp.c[(int64_t)boff[key] + atomicSub(&bcur[key], 1u) - 1u] = cd;
  }
}

__global__ void candidates_total_kernel(const unsigned long long* __restrict__ total,
                                        unsigned long long* __restrict__ counters) {
  if (blockIdx.x == 0 && threadIdx.x == 0) counters[0] = *total;
}

// One thread per candidate (grid-stride over the bucket-grouped list); its
// bucket-mates are the candidates of its segment, read straight from global
// memory (neighbouring threads share segments, so they stay L1-resident).
constexpr int kDecThreads = 256;
#ifndef HADIS_DEC_CPS
#define HADIS_DEC_CPS 32
#endif
#ifndef HADIS_GROUP_CPS
#define HADIS_GROUP_CPS 4
#endif

__global__ void __launch_bounds__(kDecThreads)   // 6 / 8 CTAs per SM forced: same / worse
decide_kernel(Grid g, const PairConst* __restrict__ pcs,
              const unsigned long long* __restrict__ counters_ro, int64_t cap,
              const unsigned long long* __restrict__ boff, const uint32_t* __restrict__ bcnt,
              const double* __restrict__ gpre, Cands grp, DecideOut o) {
  if ((int64_t)counters_ro[0] > cap) return;
  const int64_t m = (int64_t)counters_ro[0];
  const double dn = (double)g.n;
  // one thread per candidate; its bucket-mates are the neighbouring candidates
  // of the same segment (L1-resident for the warp): a branch-free certified
  // pass, the full decide_one logic only on near-ties
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Cand cd = grp.c[i];
    const int p = (int)cd.pair;
    const int64_t key = (int64_t)p * g.nbuckets + cd.bucket;
    const int64_t s0 = (int64_t)boff[key];
    const int64_t s1 = min((int64_t)boff[key + 1], m);   // exclusive scan: next start
    const double GS = gpre[key];
    const double d2 = pcs[p].delta2;
    const double G = div_n(GS, dn, g.rn);
    const double lo = cd.fid - d2, hi = cd.fid + d2;
    bool kill = G < lo, close = G <= hi && !kill;
    if (!kill) {                // (killed by G: no mates needed; kU mates' loads in flight per step)
      constexpr int kU = 8;                          // (c4: -12 us vs one at a time)
      int64_t j = s0;
      for (; j + kU <= s1; j += kU) {
        double2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = *reinterpret_cast<const double2*>(&grp.c[j + u].lat);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const bool le = v[u].x <= cd.lat;
          kill |= le & (v[u].y < lo);
          close |= le & (v[u].y <= hi) & (j + u != i);
        }
      }
      for (; j < s1; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(&grp.c[j].lat);
        const bool le = v.x <= cd.lat;
        kill |= le & (v.y < lo);
        close |= le & (v.y <= hi) & (j != i);
      }
    }
    if (kill) continue;
    if (!close) {
      set_bit(o.kept_bm, (int64_t)p * g.bm_stride + cd.cell);
      continue;
    }
    decide_one(g, pcs[p], p, cd.cell, cd.lat, cd.fid, GS, grp, s0, s1, i, o,
               [&](int64_t q) { return make_double2(grp.c[q].lat, grp.c[q].fid); });
  }
}

// measurement aid (HADIS_DEBUG_BUCKETS): candidates the exact fine prefix G
// alone kills (c4: 2.82M of 13.94M -- nearly every candidate that is not a row)
__global__ void debug_kills_kernel(Grid g, const PairConst* __restrict__ pcs,
                                   const unsigned long long* __restrict__ counters_ro, int64_t cap,
                                   const double* __restrict__ gpre, Cands grp,
                                   unsigned long long* __restrict__ out) {
  if ((int64_t)counters_ro[0] > cap) return;
  const int64_t m = (int64_t)counters_ro[0];
  unsigned long long kills = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Cand cd = grp.c[i];
    const int64_t key = (int64_t)cd.pair * g.nbuckets + cd.bucket;
    const double G = div_n(gpre[key], (double)g.n, g.rn);
    kills += G < cd.fid - pcs[cd.pair].delta2;
  }
  atomicAdd(out, kills);
}

// ------------------------------------------------- F7: no-bypass sub-frontier

constexpr int kRowThreads = 1024;
constexpr int kMaxRowU = 8192;

// theta = max(thresholds) row (rank U-1): cells sorted by tau have
// non-decreasing latency; equal nr means identical cells (keep smallest index).
__global__ void __launch_bounds__(kRowThreads)
nobypass_kernel(Grid g, const PairConst* __restrict__ pcs, uint32_t* kept_bm, Uncertain un,
                int64_t ucap, uint32_t* req_bm, uint32_t* req_pair, uint32_t* req_cell,
                int64_t rcap, unsigned long long* counters) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_fid = reinterpret_cast<double*>(smem);            // per group (by start t)
  double* s_pre = s_fid + g.U;                                 // exclusive prefix-min per t
  int32_t* s_rep = reinterpret_cast<int32_t*>(s_pre + g.U);    // group representative t
  int32_t* s_start = s_rep + g.U;                              // group start t for each t
  const int p = blockIdx.x;
  const PairConst pc = pcs[p];
  const uint32_t* C = slot_cnt(g, pc.slot);
  const int k = g.U - 1;
  const int64_t rk = (int64_t)k * g.B1;
  const int64_t cells = (int64_t)g.U * g.U;
  // group starts: t == 0 or nr changes
  for (int t = threadIdx.x; t < g.U; t += blockDim.x) {
    const bool start = (t == 0) || (C[rk + t] != C[rk + t - 1]);
    s_start[t] = start ? t : -1;
    s_fid[t] = start ? eval_cell(g, pc, k, t).fid : INFINITY;
  }
  __syncthreads();
  // block scans over t (each thread owns a contiguous chunk): exclusive
  // prefix-min of the group fidelities, inclusive max of the group starts
  {
    __shared__ double w_min[kRowThreads / 32];
    __shared__ int w_max[kRowThreads / 32];
    const int per = (g.U + blockDim.x - 1) / blockDim.x;
    const int t0 = threadIdx.x * per, t1 = min(g.U, t0 + per);
    double cmin = INFINITY;
    int cmax = -1;
    for (int t = t0; t < t1; ++t) { cmin = fmin(cmin, s_fid[t]); cmax = max(cmax, s_start[t]); }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double imin = cmin;
    int imax = cmax;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double om = __shfl_up_sync(0xffffffffu, imin, off);
      const int ox = __shfl_up_sync(0xffffffffu, imax, off);
      if (lane >= off) { imin = fmin(imin, om); imax = max(imax, ox); }
    }
    if (lane == 31) { w_min[warp] = imin; w_max[warp] = imax; }
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      double wm = lane < nw ? w_min[lane] : INFINITY;
      int wx = lane < nw ? w_max[lane] : -1;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double om = __shfl_up_sync(0xffffffffu, wm, off);
        const int ox = __shfl_up_sync(0xffffffffu, wx, off);
        if (lane >= off) { wm = fmin(wm, om); wx = max(wx, ox); }
      }
      if (lane < nw) { w_min[lane] = wm; w_max[lane] = wx; }
    }
    __syncthreads();
    // carry-in = everything before this thread's chunk
    const double prev_min = __shfl_up_sync(0xffffffffu, imin, 1);
    const int prev_max = __shfl_up_sync(0xffffffffu, imax, 1);
    double run = lane > 0 ? prev_min : INFINITY;
    int cur = lane > 0 ? prev_max : -1;
    if (warp > 0) { run = fmin(run, w_min[warp - 1]); cur = max(cur, w_max[warp - 1]); }
    __syncthreads();
    for (int t = t0; t < t1; ++t) {
      const double f = s_fid[t];
      const int st = s_start[t];
      if (st >= 0) { s_pre[t] = run; cur = st; }
      run = fmin(run, f);
      s_start[t] = cur;                           // now: the start of t's group
    }
  }
  __syncthreads();
  // group representative: the member with the smallest caller position
  for (int t = threadIdx.x; t < g.U; t += blockDim.x)
    if (s_start[t] == t) s_rep[t] = t;
  __syncthreads();
  if (!*g.sorted) {                               // unsorted caller grid (rare): sequential
    if (threadIdx.x == 0) {
      for (int t = 0; t < g.U; ++t) {
        const int st = s_start[t];
        if (g.first_pos[t] < g.first_pos[s_rep[st]]) s_rep[st] = t;
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < g.U; t += blockDim.x) {
    if (s_start[t] != t) continue;
    const double f = s_fid[t], m = s_pre[t];
    const uint32_t cell = (uint32_t)(k * g.U + s_rep[t]);
    if (m < f - pc.delta2) continue;                   // certainly dominated
    if (m > f + pc.delta2) {                           // certainly a new minimum
      set_bit(kept_bm, (int64_t)p * g.bm_stride + cell);
    } else {
      push_uncertain(1, p, cell, un, ucap, counters);
      request_exact(cells, p, cell, req_bm, req_pair, req_cell, rcap, counters);
    }
  }
}

// --------------------------------------- F8: partners of uncertain decisions

__global__ void partners_kernel(Grid g, const PairConst* __restrict__ pcs,
                                const unsigned long long* __restrict__ counters_ro, int64_t cap,
                                int64_t ucap, Uncertain un, Cands grp,
                                const unsigned long long* __restrict__ boff, uint32_t* req_bm,
                                uint32_t* req_pair, uint32_t* req_cell, int64_t rcap,
                                unsigned long long* counters) {
  if ((int64_t)counters_ro[0] > cap) return;
  const int64_t nu = (int64_t)min((unsigned long long)ucap, counters_ro[1]);
  const int64_t m = (int64_t)counters_ro[0];
  const int64_t cells = (int64_t)g.U * g.U;
  for (int64_t e = blockIdx.x; e < nu; e += gridDim.x) {
    const int p = (int)un.pair[e];
    const uint32_t cell = un.cell[e];
    const int k = (int)(cell / g.U), t = (int)(cell % g.U);
    const PairConst pc = pcs[p];
    const CellVal v = eval_cell(g, pc, k, t);
    if (un.universe[e] == 0) {
      const int b = bucket_of(g, pc, k, t);
      const int64_t s0 = (int64_t)boff[(int64_t)p * g.nbuckets];
      const int64_t s1 = min((int64_t)boff[(int64_t)p * g.nbuckets + b + 1], m);
      for (int64_t j = s0 + threadIdx.x; j < s1; j += blockDim.x) {
        if (grp.c[j].lat > v.lat || fabs(grp.c[j].fid - v.fid) > pc.delta2) continue;
        request_exact(cells, p, grp.c[j].cell, req_bm, req_pair, req_cell, rcap, counters);
      }
    } else {
      const uint32_t* C = slot_cnt(g, pc.slot);
      const int64_t rk = (int64_t)(g.U - 1) * g.B1;
      for (int td = threadIdx.x; td < t; td += blockDim.x) {
        if (td > 0 && C[rk + td] == C[rk + td - 1]) continue;   // group starts only
        if (C[rk + td] == C[rk + t]) continue;                  // same group as t
        const CellVal d = eval_cell(g, pc, g.U - 1, td);
        if (fabs(d.fid - v.fid) > pc.delta2) continue;
        request_exact(cells, p, (uint32_t)((g.U - 1) * g.U + td), req_bm, req_pair, req_cell,
                      rcap, counters);
      }
    }
  }
}

// ------------------------------------------------ F9: numpy-exact fidelities

// Cells to emulate are (pair, cell) lists of length *count (capped by cap).
struct CellList {
  const uint32_t* pair;
  const uint32_t* cell;
  const unsigned long long* count;   // device count (requests) ...
  const unsigned long long* count2;  // ... or pair_off[n_pairs] (emitted rows)
  int64_t cap;
};

__device__ __forceinline__ int64_t cell_list_len(const CellList& cl) {
  const unsigned long long c = cl.count ? *cl.count : *cl.count2;
  return (int64_t)min((unsigned long long)cl.cap, c);
}

constexpr int kPwRootThreads = 128;
constexpr int kPwCellsPerLaunch = 16384;
constexpr int64_t kPwRootGridY = 4 * kNumSMs;   // cells in flight per pw_roots launch

// grid: (roots / kPwRootThreads, cells in this batch)
__global__ void __launch_bounds__(kPwRootThreads)
pw_roots_kernel(Grid g, const PairConst* __restrict__ pcs, const double* __restrict__ thr,
                const double* __restrict__ h, const double* __restrict__ scores, CellList cl,
                int64_t first, int64_t batch, const PwPlan* __restrict__ plan,
                double* __restrict__ vals) {
  // grid-stride over the batch's cells: the grid stays small when few (or no)
  // cells need exact values -- the common case
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= plan->n_roots) return;
  const int64_t len = cell_list_len(cl);
  const int node = plan->root[r];
  for (int64_t j = blockIdx.y; j < batch && first + j < len; j += gridDim.y) {
    const int64_t c = first + j;
    const int p = (int)cl.pair[c];
    const uint32_t cell = cl.cell[c];
    const PairConst pc = pcs[p];
    const CellCost cc{thr[cell / g.U], thr[cell % g.U], pc.bl, pc.pl, pc.bh, pc.ph};
    vals[j * kPwPlanNodes + node] =
        pw_subtree(h, scores + (int64_t)pc.slot * g.n, plan->off[node], plan->len[node], cc);
  }
}

__global__ void pw_combine_kernel(CellList cl, int64_t first, const PwPlan* __restrict__ plan,
                                  double* __restrict__ vals, double dn,
                                  double* __restrict__ out_fid) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = first + j;
  if (j >= kPwCellsPerLaunch || c >= cell_list_len(cl)) return;
  double* v = vals + j * kPwPlanNodes;
  for (int i = plan->n_nodes - 1; i >= 0; --i) {
    const int ch = plan->child[i];
    if (ch >= 0) v[i] = __dadd_rn(v[ch], v[ch + 1]);
  }
  out_fid[c] = __ddiv_rn(v[0], dn);
}


// ------------------------------------------- F10: sort requests by (pair, cell)

constexpr int kSortMax = 2048;

__global__ void __launch_bounds__(1024)
sort_requests_kernel(const unsigned long long* __restrict__ counters_ro, int64_t rcap,
                     int64_t cells, uint32_t* req_pair, uint32_t* req_cell, double* req_fid) {
  __shared__ unsigned long long key[kSortMax];
  __shared__ double val[kSortMax];
  const int64_t nr = (int64_t)min((unsigned long long)rcap, counters_ro[2]);
  if (nr <= 1 || nr > kSortMax) return;
  int npow = 1;
  while (npow < nr) npow <<= 1;
  for (int i = threadIdx.x; i < npow; i += blockDim.x) {
    key[i] = i < nr ? (unsigned long long)req_pair[i] * cells + req_cell[i] : ~0ull;
    val[i] = i < nr ? req_fid[i] : 0.0;
  }
  __syncthreads();
  for (int size = 2; size <= npow; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npow; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          if ((key[i] > key[j]) == up) {
            unsigned long long tk = key[i]; key[i] = key[j]; key[j] = tk;
            double tv = val[i]; val[i] = val[j]; val[j] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    req_pair[i] = (uint32_t)(key[i] / cells);
    req_cell[i] = (uint32_t)(key[i] % cells);
    req_fid[i] = val[i];
  }
}

// Request sets larger than one CTA's bitonic sort (exact_cap > kSortMax):
// (pair, cell) keys padded with ~0 past the request count, CUB radix sort
// over the whole capacity (graph-capturable: the size is the capacity).
__global__ void pack_requests_kernel(const unsigned long long* __restrict__ counters_ro,
                                     int64_t rcap, int64_t cells,
                                     const uint32_t* __restrict__ req_pair,
                                     const uint32_t* __restrict__ req_cell,
                                     const double* __restrict__ req_fid,
                                     unsigned long long* __restrict__ kin,
                                     double* __restrict__ vin) {
  const int64_t nr = (int64_t)min((unsigned long long)rcap, counters_ro[2]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rcap;
       i += (int64_t)gridDim.x * blockDim.x) {
    kin[i] = i < nr ? (unsigned long long)req_pair[i] * cells + req_cell[i] : ~0ull;
    vin[i] = i < nr ? req_fid[i] : 0.0;
  }
}

__global__ void unpack_requests_kernel(const unsigned long long* __restrict__ counters_ro,
                                       int64_t rcap, int64_t cells,
                                       const unsigned long long* __restrict__ kout,
                                       const double* __restrict__ vout, uint32_t* req_pair,
                                       uint32_t* req_cell, double* req_fid) {
  const int64_t nr = (int64_t)min((unsigned long long)rcap, counters_ro[2]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr;
       i += (int64_t)gridDim.x * blockDim.x) {
    req_pair[i] = (uint32_t)(kout[i] / cells);
    req_cell[i] = (uint32_t)(kout[i] % cells);
    req_fid[i] = vout[i];
  }
}

static size_t request_sort_temp_bytes(int64_t ecap) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const double*)nullptr,
                                  (double*)nullptr, ecap, 0, 64);
  return bytes;
}

__device__ bool lookup_exact(int64_t nr, int64_t cells, const uint32_t* req_pair,
                             const uint32_t* req_cell, const double* req_fid, int p,
                             uint32_t cell, double* out) {
  const unsigned long long want = (unsigned long long)p * cells + cell;
  int64_t lo = 0, hi = nr;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const unsigned long long k = (unsigned long long)req_pair[mid] * cells + req_cell[mid];
    if (k < want) lo = mid + 1; else hi = mid;
  }
  if (lo < nr && (unsigned long long)req_pair[lo] * cells + req_cell[lo] == want) {
    *out = req_fid[lo];
    return true;
  }
  return false;
}

// ------------------------------------------- F11: re-decide uncertain cells

__global__ void resolve_kernel(Grid g, const PairConst* __restrict__ pcs,
                               const unsigned long long* __restrict__ counters_ro, int64_t cap,
                               int64_t ucap, int64_t rcap, int64_t sort_max, Uncertain un,
                               Cands grp,
                               const unsigned long long* __restrict__ boff,
                               const uint32_t* __restrict__ req_pair,
                               const uint32_t* __restrict__ req_cell,
                               const double* __restrict__ req_fid, uint32_t* kept_bm,
                               unsigned long long* counters) {
  __shared__ int s_kill;
  if ((int64_t)counters_ro[0] > cap) return;
  const int64_t nu = (int64_t)min((unsigned long long)ucap, counters_ro[1]);
  const int64_t m = (int64_t)min((unsigned long long)cap, counters_ro[0]);
  const int64_t nr = (int64_t)min((unsigned long long)rcap, counters_ro[2]);
  const int64_t cells = (int64_t)g.U * g.U;
  if (nr > sort_max) {  // requests were not sorted: report, decide nothing
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&counters[4], 2ull);
    return;
  }
  for (int64_t e = blockIdx.x; e < nu; e += gridDim.x) {
    const int p = (int)un.pair[e];
    const uint32_t cell = un.cell[e];
    const int k = (int)(cell / g.U), t = (int)(cell % g.U);
    const PairConst pc = pcs[p];
    const CellVal v = eval_cell(g, pc, k, t);
    const int64_t idx = grid_index(g, k, t);
    double fc = 0.0;
    const bool have_c = lookup_exact(nr, cells, req_pair, req_cell, req_fid, p, cell, &fc);
    if (threadIdx.x == 0) s_kill = have_c ? 0 : 2;
    __syncthreads();
    if (un.universe[e] == 0) {
      const int b = bucket_of(g, pc, k, t);
      const int64_t s0 = (int64_t)boff[(int64_t)p * g.nbuckets];
      const int64_t s1 = min((int64_t)boff[(int64_t)p * g.nbuckets + b + 1], m);
      for (int64_t j = s0 + threadIdx.x; j < s1 && have_c; j += blockDim.x) {
        const uint32_t dc = grp.c[j].cell;
        if (dc == cell) continue;
        const double ld = grp.c[j].lat;
        if (ld > v.lat) continue;
        double fd = grp.c[j].fid;
        double fcc = v.fid;
        if (fabs(fd - v.fid) <= pc.delta2) {
          if (!lookup_exact(nr, cells, req_pair, req_cell, req_fid, p, dc, &fd)) { atomicMax(&s_kill, 2); continue; }
          fcc = fc;
        }
        if (kills(fd, fcc, ld, v.lat, grid_index(g, (int)(dc / g.U), (int)(dc % g.U)), idx))
          atomicMax(&s_kill, 1);
      }
    } else {
      const uint32_t* C = slot_cnt(g, pc.slot);
      const int64_t rk = (int64_t)(g.U - 1) * g.B1;
      for (int td = threadIdx.x; td < t && have_c; td += blockDim.x) {
        if (td > 0 && C[rk + td] == C[rk + td - 1]) continue;
        if (C[rk + td] == C[rk + t]) continue;
        const CellVal d = eval_cell(g, pc, g.U - 1, td);
        double fd = d.fid, fcc = v.fid;
        if (fabs(d.fid - v.fid) <= pc.delta2) {
          if (!lookup_exact(nr, cells, req_pair, req_cell, req_fid, p,
                            (uint32_t)((g.U - 1) * g.U + td), &fd)) { atomicMax(&s_kill, 2); continue; }
          fcc = fc;
        }
        if (fd <= fcc) atomicMax(&s_kill, 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_kill == 0) set_bit(kept_bm, (int64_t)p * g.bm_stride + cell);
      if (s_kill == 2) atomicOr(&counters[4], 4ull);   // missing exact value: overflow
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- F12: emit

// The kept bitmap is cut into chunks of kEmitWords words (per pair); chunk
// popcounts -> device-wide scan -> one CTA per chunk writes its rows, so rows
// come out pair-major and, within a pair, in (theta rank, tau rank) order.
constexpr int kEmitWords = 256;   // = emit CTA size (64 / 128 / 512 measured: no gain)

// one warp per chunk (kEmitWords words, 8 per lane as two 16-byte loads), 8
// chunks per CTA (one CTA per chunk and thread per word: 16 us at c4)
constexpr int kCountWarps = 8;
__global__ void __launch_bounds__(kCountWarps * 32)
count_chunks_kernel(const uint32_t* __restrict__ kept_bm, int64_t words_per_pair, int n_chunks,
                    uint32_t* __restrict__ chunk_rows) {
  static_assert(kEmitWords == 32 * 8, "8 words per lane");
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kCountWarps + (threadIdx.x >> 5), p = blockIdx.y;
  if (c >= n_chunks) return;
  const uint32_t* w = kept_bm + (int64_t)p * words_per_pair;
  const int64_t w0 = (int64_t)c * kEmitWords + 4 * lane;
  uint32_t v = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t wi = w0 + h * 128;
    if (wi + 3 < words_per_pair && ((words_per_pair & 3) == 0)) {
      const uint4 q = *reinterpret_cast<const uint4*>(w + wi);
      v += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    } else {
      for (int j = 0; j < 4; ++j) if (wi + j < words_per_pair) v += __popc(w[wi + j]);
    }
  }
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) chunk_rows[(int64_t)p * n_chunks + c] = v;
}

__global__ void pair_offsets_kernel(const unsigned long long* __restrict__ chunk_off, int n_chunks,
                                    int n_pairs, unsigned long long* __restrict__ pair_off,
                                    int64_t* stats, int64_t out_cap, unsigned long long* counters) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n_pairs) {
    const unsigned long long a = chunk_off[(int64_t)p * n_chunks];
    const unsigned long long b = chunk_off[(int64_t)(p + 1) * n_chunks];
    pair_off[p] = a;
    stats[HADIS_ST_PAIR0 + p] = (int64_t)(b - a);
  }
  if (p == 0) {
    const unsigned long long run = chunk_off[(int64_t)n_pairs * n_chunks];
    pair_off[n_pairs] = run;
    stats[HADIS_ST_ROWS] = (int64_t)run;
    stats[HADIS_ST_CANDIDATES] = (int64_t)counters[0];
    stats[HADIS_ST_UNCERTAIN] = (int64_t)counters[1];
    stats[HADIS_ST_EXACT_CELLS] = (int64_t)counters[2];
    if ((int64_t)run > out_cap) counters[4] |= 8ull;
  }
}

struct Rows {
  int32_t* pair;
  int32_t* theta_pos;
  int32_t* tau_pos;
  double* r_light;  // null in the compact form (multi-GPU slab): rebuilt from
  double* r_heavy;  // n_light / n_heavy by the merge, bit for bit
  double* fid;
  double* lat;
  uint32_t* cell;   // workspace: k * U + t, for exact patches
  uint32_t* n_light;   // compact form only: R_k (records the light stage serves)
  uint32_t* n_heavy;   // compact form only: nb + nr (records the heavy stage serves)
};

// bits -> cell list in shared memory -> one row per thread (coalesced stores)
// 6 CTAs/SM: latency bound like decide (-60 us at c4; group_cands the opposite)
__global__ void __launch_bounds__(kEmitWords, 6)
emit_rows_kernel(Grid g, const PairConst* __restrict__ pcs, const uint32_t* __restrict__ kept_bm,
                 int64_t words_per_pair, int n_chunks,
                 const unsigned long long* __restrict__ chunk_off, int64_t out_cap, Rows out,
                 const unsigned long long* __restrict__ counters, int exact_fid) {
  __shared__ uint32_t s_cell[kEmitWords * 32];
  // the row -> cell map is read only by the exact-fidelity passes: skip it when
  // none will run (no exact requests, exact_fid off: 45 MB of stores at c4)
  const bool keep_cell = exact_fid || counters[2] != 0;
  const int p = blockIdx.y, ch = blockIdx.x;
  const int64_t wi = (int64_t)ch * kEmitWords + threadIdx.x;
  const uint32_t word = wi < words_per_pair ? kept_bm[(int64_t)p * words_per_pair + wi] : 0u;
  const int64_t cells = (int64_t)g.U * g.U;
  unsigned long long total;
  int at = (int)block_exclusive_sum((unsigned long long)__popc(word), &total);
  uint32_t bits = word;
  while (bits) {
    const int b = __ffs(bits) - 1;
    bits &= bits - 1;
    s_cell[at++] = (uint32_t)(wi * 32 + b);
  }
  __syncthreads();
  const PairConst pc = pcs[p];
  const double dn = (double)g.n;
  const unsigned long long base = chunk_off[(int64_t)p * n_chunks + ch];
  for (int i = threadIdx.x; i < (int)total; i += blockDim.x) {
    const int64_t c = s_cell[i];
    const int64_t r = (int64_t)base + i;
    if (c >= cells || r >= out_cap) continue;
    const int k = (int)((uint32_t)c / (uint32_t)g.U), t = (int)((uint32_t)c - (uint32_t)k * g.U);
    const CellVal v = eval_cell(g, pc, k, t);
    if (keep_cell || out.n_light == nullptr) out.pair[r] = p;   // compact: workspace only
    out.theta_pos[r] = g.first_pos[k];
    out.tau_pos[r] = g.first_pos[t];
    out.fid[r] = v.fid;
    if (keep_cell) out.cell[r] = (uint32_t)c;
    if (out.n_light != nullptr) {                  // compact rows (uniform branch)
      out.n_light[r] = v.n_keep_light;
      out.n_heavy[r] = v.n_heavy;
    } else {
      out.r_light[r] = div_n((double)v.n_keep_light, dn, g.rn);
      out.r_heavy[r] = div_n((double)v.n_heavy, dn, g.rn);
      out.lat[r] = v.lat;
    }
  }
}

// F13: patch rows whose fidelity was computed exactly during resolution
__global__ void patch_rows_kernel(const unsigned long long* __restrict__ counters_ro, int64_t rcap,
                                  const uint32_t* __restrict__ req_pair,
                                  const uint32_t* __restrict__ req_cell,
                                  const double* __restrict__ req_fid,
                                  const unsigned long long* __restrict__ pair_off, int64_t out_cap,
                                  Rows out) {
  const int64_t nr = (int64_t)min((unsigned long long)rcap, counters_ro[2]);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr) return;
  const int p = (int)req_pair[i];
  const uint32_t cell = req_cell[i];
  int64_t lo = (int64_t)pair_off[p], hi = (int64_t)pair_off[p + 1];
  if (hi > out_cap) hi = out_cap;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (out.cell[mid] < cell) lo = mid + 1; else hi = mid;
  }
  if (lo < (int64_t)pair_off[p + 1] && lo < out_cap && out.cell[lo] == cell) out.fid[lo] = req_fid[i];
}

__global__ void finish_stats_kernel(const unsigned long long* counters, int64_t cap, int64_t ucap,
                                    int64_t rcap, int64_t* stats) {
  unsigned long long of = counters[4];
  if ((int64_t)counters[0] > cap) of |= 16ull;
  if ((int64_t)counters[1] > ucap) of |= 32ull;
  if ((int64_t)counters[2] > rcap) of |= 64ull;
  stats[HADIS_ST_OVERFLOW] = (int64_t)of;
}

// ------------------------------------------------ explicit-cell exact means

__global__ void __launch_bounds__(kPwThreads)
fid_exact_kernel(const double* __restrict__ h, const double* __restrict__ scores, int64_t n,
                 int n_cells, const int32_t* __restrict__ slot, const double* __restrict__ theta,
                 const double* __restrict__ tau, const double* __restrict__ params,
                 double* __restrict__ out) {
  __shared__ PwShared sh;
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    const double* q = params + (int64_t)c * 4;
    CellCost cc{theta[c], tau[c], q[0], q[1], q[2], q[3]};
    const double sum = pw_block_sum(h, scores + (int64_t)slot[c] * n, n, cc, sh);
    if (threadIdx.x == 0) out[c] = __ddiv_rn(sum, (double)n);
  }
}

// ------------------------------------------------- single-pass scan (CUB)
// The bucket offsets (exclusive sum of the per-bucket candidate counts) run as
// a CUB decoupled-look-back scan: one read and one write per bucket (the
// three-launch tile scan read twice: c4 53 -> 32 us).  The per-pair prefix
// minima stay on the tile kernels: a CUB segmented-min scan over (min, head)
// pairs measured 5x slower (non-word tile state, per-element modulo).

struct CountIn {        // bucket counts widened to 64 bits, 0 past the end
  const uint32_t* cnt;
  int64_t n;
  __host__ __device__ unsigned long long operator()(int64_t i) const {
    return i < n ? (unsigned long long)cnt[i] : 0ull;
  }
};

static cudaError_t count_offsets(void* temp, size_t& temp_bytes, const uint32_t* cnt, int64_t n,
                                 unsigned long long* off, cudaStream_t st) {
  auto in = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), CountIn{cnt, n});
  return cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, off, n + 1, st);   // off[n] = total
}

static size_t scan_temp_bytes(int64_t items) {   // enough for any scan of <= items
  size_t c = 0;
  count_offsets(nullptr, c, nullptr, items, nullptr, 0);
  return c;
}

// ------------------------------------------------------------ workspace

struct Layout {
  size_t pcs, pk, row_rep, row_start, sorted, bmin, gpre, cmin, cpre, ctmin, bcnt, boff, grp, lst, kept, reqbm, un[3], req[3],
      counters, groups, tmin, pwplan, pwvals, pair_rows, chunk_off, pair_off, row_cell,
      row_pair, scan_temp, scan_temp_bytes, rsort[5], rsort_bytes, total;
};

static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static Layout make_layout(int n_pairs, int U, int nbuckets, int64_t cap, int64_t ecap,
                          int64_t out_cap) {
  Layout L{};
  size_t at = 0;
  auto take = [&](size_t bytes) { size_t r = at; at = align_up(at + bytes); return r; };
  const int64_t pb = (int64_t)n_pairs * nbuckets;
  const int64_t cells = (int64_t)U * U;
  const int64_t words = (cells + 31) / 32 * n_pairs;
  L.pcs = take(sizeof(PairConst) * n_pairs);
  L.pk = take(sizeof(int32_t) * U);
  L.row_rep = take(sizeof(int32_t) * U);
  L.row_start = take(U);
  L.sorted = take(4);
  L.bmin = take(8 * pb);
  L.gpre = take(8 * pb);
  L.cmin = take(8 * (pb >> kCoarseShift));
  L.cpre = take(8 * (pb >> kCoarseShift));
  L.ctmin = take(8 * (ceil_div(nbuckets >> kCoarseShift, 4096) * n_pairs + 1));
  L.bcnt = take(4 * pb);
  L.boff = take(8 * (pb + 1));
  L.grp = take(sizeof(Cand) * cap);
  L.lst = take(sizeof(ListCand) * cap);
  L.kept = take(4 * words);
  L.reqbm = take(4 * words);
  L.un[0] = take(4 * ecap); L.un[1] = take(4 * ecap); L.un[2] = take(4 * ecap);
  L.req[0] = take(4 * ecap); L.req[1] = take(4 * ecap); L.req[2] = take(8 * ecap);
  L.counters = take(8 * 8);
  L.groups = take(4 * (n_pairs + 2));
  L.tmin = take(8 * (ceil_div(nbuckets, 4096) * n_pairs + 1));
  L.pwplan = take(sizeof(PwPlan));
  const int64_t pw_batch = std::min<int64_t>(std::max(ecap, out_cap), kPwCellsPerLaunch);
  L.pwvals = take(8 * (int64_t)kPwPlanNodes * pw_batch);
  const int64_t n_cw = ceil_div((cells + 31) / 32, kEmitWords) * n_pairs;   // emit chunks
  L.pair_rows = take(4 * n_cw);
  L.chunk_off = take(8 * (n_cw + 1));
  L.pair_off = take(8 * (n_pairs + 1));
  L.row_cell = take(4 * out_cap);
  L.row_pair = take(4 * out_cap);                  // compact outputs: pair ids of the rows
  L.scan_temp_bytes = scan_temp_bytes(std::max<int64_t>(pb, n_cw));
  L.scan_temp = take(L.scan_temp_bytes ? L.scan_temp_bytes : 1);
  if (ecap > kSortMax) {                           // CUB request sort (see pack_requests_kernel)
    L.rsort[0] = take(8 * ecap); L.rsort[1] = take(8 * ecap);     // keys in / out
    L.rsort[2] = take(8 * ecap); L.rsort[3] = take(8 * ecap);     // fid in / out
    L.rsort_bytes = request_sort_temp_bytes(ecap);
    L.rsort[4] = take(L.rsort_bytes ? L.rsort_bytes : 1);
  }
  L.total = at;
  return L;
}

// Latency buckets per pair: coarse enough that the bucket minima stay
// L2-resident (2^16 x 8 B per pair); candidates are pre-thinned by the row
// prefix-min, so coarse buckets admit few extra candidates.
static int buckets_for(int U) {
  const int64_t cells = (int64_t)U * U;
  int64_t b = 1024;
  while (b < cells / 16 && b < (1 << 16)) b <<= 1;
  return (int)b;
}

}  // namespace hadis

using namespace hadis;

extern "C" size_t hadis_frontier_workspace_bytes(int32_t n_pairs, int32_t n_unique,
                                                 int64_t cand_cap, int64_t exact_cap,
                                                 int64_t out_cap) {
  if (n_pairs <= 0 || n_unique <= 0 || cand_cap <= 0 || exact_cap <= 0 || out_cap <= 0) return 0;
  return make_layout(n_pairs, n_unique, buckets_for(n_unique), cand_cap, exact_cap, out_cap).total;
}

// Shared body of hadis_pair_frontiers (full rows) and hadis_pair_frontiers_compact
// (out_n_light != null: theta_pos, tau_pos, n_light, n_heavy, fid only).
static int pair_frontiers(const uint32_t* pre_cnt, const uint64_t* pre_hsum, int64_t n,
                          int32_t n_unique, int32_t hfix_shift, int32_t n_pairs,
                          const int32_t* pair_slot, const double* pair_params,
                          const int32_t* first_pos, int32_t n_thresholds,
                          const double* thr_unique, const double* h, const double* scores,
                          int32_t exact_fid, void* workspace, size_t workspace_bytes,
                          int64_t cand_cap, int64_t exact_cap, int64_t out_cap, int32_t* out_pair,
                          int32_t* out_theta_pos, int32_t* out_tau_pos, double* out_r_light,
                          double* out_r_heavy, double* out_fid, double* out_lat,
                          uint32_t* out_n_light, uint32_t* out_n_heavy, int64_t* stats,
                          void* stream) {
  if (!pre_cnt || !pre_hsum || n <= 0 || n > 0xffffffffll || n_unique <= 0 ||
      n_unique > kMaxRowU || n_pairs <= 0 || !pair_slot || !pair_params || !first_pos ||
      n_thresholds < n_unique || !thr_unique || !h || !scores || !workspace || cand_cap <= 0 ||
      exact_cap <= 0 || out_cap <= 0 || !stats || !out_theta_pos || !out_tau_pos || !out_fid)
    return HADIS_ERR_ARG;
  if (out_n_light ? !out_n_heavy : (!out_pair || !out_r_light || !out_r_heavy || !out_lat))
    return HADIS_ERR_ARG;
  if ((int64_t)n_unique * n_unique > 0xffffffffll) return HADIS_ERR_UNSUPPORTED;
  const int nb = buckets_for(n_unique);
  const Layout L = make_layout(n_pairs, n_unique, nb, cand_cap, exact_cap, out_cap);
  if (workspace_bytes < L.total) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  auto P = [&](size_t off) { return (void*)(ws + off); };

  PairConst* pcs = (PairConst*)P(L.pcs);
  int32_t* pk = (int32_t*)P(L.pk);
  int32_t* row_rep = (int32_t*)P(L.row_rep);
  uint8_t* row_start = (uint8_t*)P(L.row_start);
  int32_t* sorted = (int32_t*)P(L.sorted);
  unsigned long long* bmin = (unsigned long long*)P(L.bmin);
  double* gpre = (double*)P(L.gpre);
  unsigned long long* cmin = (unsigned long long*)P(L.cmin);
  double* cpre = (double*)P(L.cpre);
  unsigned long long* ctmin = (unsigned long long*)P(L.ctmin);
  uint32_t* bcnt = (uint32_t*)P(L.bcnt);
  unsigned long long* boff = (unsigned long long*)P(L.boff);
  Cands grp{(Cand*)P(L.grp)};
  ListCand* lst = (ListCand*)P(L.lst);
  uint32_t* kept = (uint32_t*)P(L.kept);
  uint32_t* reqbm = (uint32_t*)P(L.reqbm);
  Uncertain un{(uint32_t*)P(L.un[0]), (uint32_t*)P(L.un[1]), (uint32_t*)P(L.un[2])};
  uint32_t* req_pair = (uint32_t*)P(L.req[0]);
  uint32_t* req_cell = (uint32_t*)P(L.req[1]);
  double* req_fid = (double*)P(L.req[2]);
  unsigned long long* counters = (unsigned long long*)P(L.counters);
  int32_t* n_groups = (int32_t*)P(L.groups);
  int32_t* group_p0 = n_groups + 1;
  unsigned long long* tmin = (unsigned long long*)P(L.tmin);
  PwPlan* pwplan = (PwPlan*)P(L.pwplan);
  double* pwvals = (double*)P(L.pwvals);
  uint32_t* chunk_rows = (uint32_t*)P(L.pair_rows);
  unsigned long long* chunk_off = (unsigned long long*)P(L.chunk_off);
  unsigned long long* pair_off = (unsigned long long*)P(L.pair_off);
  uint32_t* row_cell = (uint32_t*)P(L.row_cell);
  int32_t* row_pair = (int32_t*)P(L.row_pair);

  const int64_t pb = (int64_t)n_pairs * nb;
  const int64_t cells = (int64_t)n_unique * n_unique;
  const int64_t words_per_pair = (cells + 31) / 32;
  HADIS_CUDA_TRY(cudaMemsetAsync(bmin, 0xff, 8 * pb, st));
  HADIS_CUDA_TRY(cudaMemsetAsync(cmin, 0xff, 8 * (pb >> kCoarseShift), st));
  HADIS_CUDA_TRY(cudaMemsetAsync(bcnt, 0, 4 * pb, st));
  HADIS_CUDA_TRY(cudaMemsetAsync(kept, 0, 4 * words_per_pair * n_pairs, st));
  HADIS_CUDA_TRY(cudaMemsetAsync(reqbm, 0, 4 * words_per_pair * n_pairs, st));
  HADIS_CUDA_TRY(cudaMemsetAsync(counters, 0, 8 * 8, st));

  Grid g{pre_cnt, pre_hsum, n, n_unique, n_unique + 1, ldexp(1.0, -hfix_shift), nb,
         n_thresholds, first_pos, words_per_pair * 32, pk, row_rep, row_start, sorted,
         1.0 / (double)n};
  int launches = 29;   // fixed kernels below (a CUB scan is 2); batched emulation adds 2 per batch
  pair_const_kernel<<<(unsigned)ceil_div(n_pairs, 128), 128, 0, st>>>(
      n_pairs, pair_slot, pair_params, n, hfix_shift, nb, pcs);
  if ((size_t)n_unique * 12 > 30 * 1024)   // opt in only near the 48 KB default (~17 KB static)
    HADIS_CUDA_TRY(hadis_ensure_smem((const void*)row_classes_kernel, (size_t)((size_t)n_unique * 12)));
  row_classes_kernel<<<1, 1024, (size_t)n_unique * 12, st>>>(pre_cnt, n_unique, n_unique + 1,
                                                            first_pos, pk, row_rep, row_start,
                                                            sorted);
  HADIS_LAUNCH_CHECK();

  const dim3 row_grid((unsigned)ceil_div(n_unique, kRowWarps), (unsigned)n_pairs);
  group_kernel<<<1, 32, 0, st>>>(pair_slot, n_pairs, group_p0, n_groups, counters, kMaxGroup);
  const size_t rsm = sizeof(RowSmem);
  const size_t fsm = rsm + (size_t)kRowWarps * kMaxGroup * 32;   // + per-window pass masks
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)bucket_min_kernel, (size_t)rsm));
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)filter_kernel, (size_t)fsm));
#ifndef HADIS_F1_STRIDE
#define HADIS_F1_STRIDE 4      // F1 over every 4th theta-row only
#endif
#ifndef HADIS_F1_CHUNKS
#define HADIS_F1_CHUNKS 2      // partner chunks per row (parallelism of the sampled F1)
#endif
  {
    constexpr int kS = HADIS_F1_STRIDE, kC = HADIS_F1_CHUNKS;
    const dim3 f1_grid((unsigned)ceil_div(ceil_div(n_unique, kS), kRowWarps),
                       (unsigned)(n_pairs * kC));
    bucket_min_kernel<<<f1_grid, kRowWarps * 32, rsm, st>>>(g, pcs, group_p0, n_groups, cmin, kS,
                                                            kC);
  }
  auto prefix = [&](const unsigned long long* mins, int nbk, unsigned long long* tm, double* pre) {
    const int tiles = (int)ceil_div(nbk, kPrefTile);
    prefix_tile_min_kernel<<<dim3(tiles, n_pairs), kScanThreads, 0, st>>>(mins, nbk, tm);
    prefix_carry_kernel<<<(unsigned)ceil_div(n_pairs, 128), 128, 0, st>>>(tm, tiles, n_pairs);
    prefix_apply_kernel<<<dim3(tiles, n_pairs), kScanThreads, 0, st>>>(mins, nbk, tm, pre);
  };
  prefix(cmin, nb >> kCoarseShift, ctmin, cpre);
  const DecideOut dout{kept, un, exact_cap, reqbm, req_pair, req_cell, exact_cap, counters};
  filter_kernel<<<row_grid, kRowWarps * 32, fsm, st>>>(g, pcs, group_p0, n_groups, cpre, bcnt, lst,
                                                     cand_cap, counters + 5);
  {
    size_t tb = L.scan_temp_bytes;
    HADIS_CUDA_TRY(count_offsets(P(L.scan_temp), tb, bcnt, pb, boff, st));
  }
  candidates_total_kernel<<<1, 1, 0, st>>>(boff + pb, counters);
  if (getenv("HADIS_DEBUG_BUCKETS")) {             // measurement aid: fine-bucket occupancy
    std::vector<uint32_t> hc(pb);
    cudaStreamSynchronize(st);
    cudaMemcpy(hc.data(), bcnt, 4 * pb, cudaMemcpyDeviceToHost);
    double s1 = 0, s2 = 0;
    uint32_t mx = 0;
    int64_t hist[33] = {0}, nz = 0;
    for (int64_t i = 0; i < pb; ++i) {
      const uint32_t m = hc[i];
      if (!m) continue;
      ++nz;
      s1 += m;
      s2 += (double)m * m;
      mx = m > mx ? m : mx;
      int lb = 0;
      while ((1u << (lb + 1)) <= m) ++lb;
      hist[lb] += m;
    }
    fprintf(stderr, "buckets: %lld non-empty of %lld, candidates %.0f, mates/cand %.2f, max %u\n",
            (long long)nz, (long long)pb, s1, s2 / (s1 > 0 ? s1 : 1), mx);
    for (int lb = 0; lb < 33; ++lb)
      if (hist[lb]) fprintf(stderr, "  bucket size [%u, %u): %lld candidates\n", 1u << lb,
                            lb < 31 ? 2u << lb : 0u, (long long)hist[lb]);
  }
  // grid sizes of the two grid-stride passes measured at c4 (4 / 32 CTAs per SM)
  group_cands_kernel<<<kNumSMs * HADIS_GROUP_CPS, 256, 0, st>>>(g, pcs, lst, counters + 5, cand_cap, nb, (double)n, boff,
                                                  bcnt, grp, bmin);
  prefix(bmin, nb, tmin, gpre);                    // exact fine G for decide
  HADIS_LAUNCH_CHECK();
  decide_kernel<<<kNumSMs * HADIS_DEC_CPS, kDecThreads, 0, st>>>(g, pcs, counters, cand_cap, boff, bcnt, gpre,
                                             grp, dout);
  if (getenv("HADIS_DEBUG_BUCKETS")) {
    unsigned long long* dk = nullptr;
    unsigned long long hk = 0;
    cudaMalloc(&dk, 8);
    cudaMemsetAsync(dk, 0, 8, st);
    debug_kills_kernel<<<kNumSMs * 8, 256, 0, st>>>(g, pcs, counters, cand_cap, gpre, grp, dk);
    cudaMemcpyAsync(&hk, dk, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(dk);
    fprintf(stderr, "candidates killed by the fine prefix G alone: %llu\n", hk);
  }
  const size_t row_smem = (size_t)n_unique * (8 + 8 + 4 + 4);
  // always opt in: the kernel's static shared memory counts against the 48 KB
  // default too (U = 2047 needs 49128 B dynamic + the static block-scan arrays)
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)nobypass_kernel, (size_t)row_smem));
  nobypass_kernel<<<n_pairs, kRowThreads, row_smem, st>>>(g, pcs, kept, un, exact_cap, reqbm,
                                                          req_pair, req_cell, exact_cap, counters);
  HADIS_LAUNCH_CHECK();
  partners_kernel<<<kNumSMs, 256, 0, st>>>(g, pcs, counters, cand_cap, exact_cap, un, grp, boff,
                                           reqbm, req_pair, req_cell, exact_cap, counters);
  pw_plan_kernel<<<1, 256, 0, st>>>(n, pwplan, exact_fid ? nullptr : counters + 2);
  {
    const CellList cl{req_pair, req_cell, counters + 2, nullptr, exact_cap};
    const int64_t batch = exact_cap < kPwCellsPerLaunch ? exact_cap : kPwCellsPerLaunch;
    for (int64_t first = 0; first < exact_cap; first += kPwCellsPerLaunch, launches += 2) {
      pw_roots_kernel<<<dim3(kPwPlanRoots / kPwRootThreads, (unsigned)min(batch, kPwRootGridY)),
                        kPwRootThreads, 0, st>>>(g, pcs, thr_unique, h, scores, cl, first, batch,
                                                 pwplan, pwvals);
      pw_combine_kernel<<<(unsigned)ceil_div(batch, 128), 128, 0, st>>>(cl, first, pwplan, pwvals,
                                                                        (double)n, req_fid);
    }
  }
  if (exact_cap > kSortMax) {
    unsigned long long* kin = (unsigned long long*)P(L.rsort[0]);
    unsigned long long* kout = (unsigned long long*)P(L.rsort[1]);
    double* vin = (double*)P(L.rsort[2]);
    double* vout = (double*)P(L.rsort[3]);
    const unsigned rg = (unsigned)std::min<int64_t>(ceil_div(exact_cap, 256), kNumSMs * 8);
    pack_requests_kernel<<<rg, 256, 0, st>>>(counters, exact_cap, cells, req_pair, req_cell,
                                            req_fid, kin, vin);
    size_t tb = L.rsort_bytes;
    HADIS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(P(L.rsort[4]), tb, kin, kout, vin, vout,
                                                   exact_cap, 0, 64, st));
    unpack_requests_kernel<<<rg, 256, 0, st>>>(counters, exact_cap, cells, kout, vout, req_pair,
                                              req_cell, req_fid);
    launches += 1;
  } else {
    sort_requests_kernel<<<1, 1024, 0, st>>>(counters, exact_cap, cells, req_pair, req_cell,
                                             req_fid);
  }
  const int64_t sort_max = exact_cap > kSortMax ? exact_cap : kSortMax;
  resolve_kernel<<<kNumSMs, 256, 0, st>>>(g, pcs, counters, cand_cap, exact_cap, exact_cap,
                                          sort_max, un, grp, boff, req_pair, req_cell, req_fid,
                                          kept, counters);
  HADIS_LAUNCH_CHECK();
  const int n_chunks = (int)ceil_div(words_per_pair, kEmitWords);
  const int64_t n_cw = (int64_t)n_chunks * n_pairs;
  count_chunks_kernel<<<dim3((unsigned)ceil_div(n_chunks, kCountWarps), n_pairs), kCountWarps * 32, 0,
                        st>>>(kept, words_per_pair, n_chunks, chunk_rows);
  {                                                // chunk row offsets (same CUB scan)
    size_t tb = L.scan_temp_bytes;
    HADIS_CUDA_TRY(count_offsets(P(L.scan_temp), tb, chunk_rows, n_cw, chunk_off, st));
  }
  pair_offsets_kernel<<<(unsigned)ceil_div(n_pairs, 128), 128, 0, st>>>(
      chunk_off, n_chunks, n_pairs, pair_off, stats, out_cap, counters);
  if (out_n_light != nullptr) out_pair = row_pair;   // compact: pair ids stay in the workspace
  Rows out{out_pair,    out_theta_pos, out_tau_pos, out_r_light, out_r_heavy,
           out_fid,     out_lat,       row_cell,    out_n_light, out_n_heavy};
  emit_rows_kernel<<<dim3(n_chunks, n_pairs), kEmitWords, 0, st>>>(
      g, pcs, kept, words_per_pair, n_chunks, chunk_off, out_cap, out, counters, exact_fid);
  if (exact_fid) {
    // every emitted row; out_cap bounds the batches launched (rows beyond the
    // device row count exit immediately)
    const CellList cl{reinterpret_cast<const uint32_t*>(out_pair), row_cell, nullptr,
                      pair_off + n_pairs, out_cap};
    const int64_t batch = out_cap < kPwCellsPerLaunch ? out_cap : kPwCellsPerLaunch;
    for (int64_t first = 0; first < out_cap; first += kPwCellsPerLaunch, launches += 2) {
      pw_roots_kernel<<<dim3(kPwPlanRoots / kPwRootThreads, (unsigned)min(batch, kPwRootGridY)),
                        kPwRootThreads, 0, st>>>(g, pcs, thr_unique, h, scores, cl, first, batch,
                                                 pwplan, pwvals);
      pw_combine_kernel<<<(unsigned)ceil_div(batch, 128), 128, 0, st>>>(cl, first, pwplan, pwvals,
                                                                        (double)n, out_fid);
    }
  } else {
    patch_rows_kernel<<<(unsigned)ceil_div(exact_cap, 256), 256, 0, st>>>(
        counters, exact_cap, req_pair, req_cell, req_fid, pair_off, out_cap, out);
  }
  finish_stats_kernel<<<1, 1, 0, st>>>(counters, cand_cap, exact_cap, exact_cap, stats);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(exact_fid ? launches - 1 : launches);
  return HADIS_OK;
}

extern "C" int hadis_pair_frontiers(const uint32_t* pre_cnt, const uint64_t* pre_hsum, int64_t n,
                                    int32_t n_unique, int32_t hfix_shift, int32_t n_pairs,
                                    const int32_t* pair_slot, const double* pair_params,
                                    const int32_t* first_pos, int32_t n_thresholds,
                                    const double* thr_unique, const double* h,
                                    const double* scores, int32_t exact_fid, void* workspace,
                                    size_t workspace_bytes, int64_t cand_cap, int64_t exact_cap,
                                    int64_t out_cap, int32_t* out_pair, int32_t* out_theta_pos,
                                    int32_t* out_tau_pos, double* out_r_light,
                                    double* out_r_heavy, double* out_fid, double* out_lat,
                                    int64_t* stats, void* stream) {
  return pair_frontiers(pre_cnt, pre_hsum, n, n_unique, hfix_shift, n_pairs, pair_slot,
                        pair_params, first_pos, n_thresholds, thr_unique, h, scores, exact_fid,
                        workspace, workspace_bytes, cand_cap, exact_cap, out_cap, out_pair,
                        out_theta_pos, out_tau_pos, out_r_light, out_r_heavy, out_fid, out_lat,
                        nullptr, nullptr, stats, stream);
}

extern "C" int hadis_pair_frontiers_compact(
    const uint32_t* pre_cnt, const uint64_t* pre_hsum, int64_t n, int32_t n_unique,
    int32_t hfix_shift, int32_t n_pairs, const int32_t* pair_slot, const double* pair_params,
    const int32_t* first_pos, int32_t n_thresholds, const double* thr_unique, const double* h,
    const double* scores, int32_t exact_fid, void* workspace, size_t workspace_bytes,
    int64_t cand_cap, int64_t exact_cap, int64_t out_cap, int32_t* out_theta_pos,
    int32_t* out_tau_pos, uint32_t* out_n_light, uint32_t* out_n_heavy, double* out_fid,
    int64_t* stats, void* stream) {
  if (!out_n_light) return HADIS_ERR_ARG;
  return pair_frontiers(pre_cnt, pre_hsum, n, n_unique, hfix_shift, n_pairs, pair_slot,
                        pair_params, first_pos, n_thresholds, thr_unique, h, scores, exact_fid,
                        workspace, workspace_bytes, cand_cap, exact_cap, out_cap, nullptr,
                        out_theta_pos, out_tau_pos, nullptr, nullptr, out_fid, nullptr,
                        out_n_light, out_n_heavy, stats, stream);
}

extern "C" int hadis_fid_exact(const double* h, const double* scores, int64_t n, int32_t n_cells,
                               const int32_t* cell_slot, const double* cell_theta,
                               const double* cell_tau, const double* cell_params, double* out_fid,
                               void* stream) {
  if (!h || !scores || n <= 0 || n_cells < 0 || (n_cells > 0 && (!cell_slot || !cell_theta ||
      !cell_tau || !cell_params || !out_fid)))
    return HADIS_ERR_ARG;
  if (n_cells == 0) return HADIS_OK;
  int grid = n_cells < kNumSMs * 4 ? n_cells : kNumSMs * 4;
  fid_exact_kernel<<<grid, kPwThreads, 0, (cudaStream_t)stream>>>(
      h, scores, n, n_cells, cell_slot, cell_theta, cell_tau, cell_params, out_fid);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}
