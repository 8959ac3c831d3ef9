// Multi-GPU merge of pair-sharded tables (SURVEY §8 row e; SPEC.md:309-310:
// pair x grid profiling is embarrassingly parallel, reduced in a
// deterministic (pair, theta, tau) order).
//
// Every rank's frontier pass writes its rows straight into one "slab" (no
// pack step): an int64 header (the frontier stats: row count, overflow bits,
// per-local-pair row counts, the record-validation flag; plus a host error
// word) followed by the rows in the compact form of
// hadis_pair_frontiers_compact -- theta_pos, tau_pos, n_light, n_heavy (4 x 32
// bit) and fid (float64): 24 bytes per row instead of the table's 44.  The
// merge rebuilds r_light = n_light / n, r_heavy = n_heavy / n and lat =
// (n_light L_l + n_heavy L_h) / n with the frontier's own operations (div_n),
// so the merged table is bit-identical to a one-GPU build.  One all_gather_into_tensor of the slabs
// (NCCL over NVLink) gives every rank every slab; this merge then writes the
// canonical table -- pairs in global (light, heavy) order, each pair's rows in
// the (theta, tau) order its owner emitted them -- with no host round trip:
//   M1 shard_offsets_kernel  one CTA: per global pair its owner's row count,
//                            source row (prefix within the owner's slab) and
//                            destination row (prefix over global pairs), plus
//                            the OR of every rank's status words;
//   M2 shard_copy_kernel     (row chunk, pair) CTAs expand the rows into the
//                            seven table columns, pair = global id.
// HBM-bound: 24 B read + 44 B written per row.
#include "common.cuh"

namespace hadis {

constexpr int kMergeThreads = 256;
constexpr int kMergeChunks = 16;          // CTAs per pair segment (grid-stride inside)

struct SlabView {
  const unsigned char* base;
  size_t slab_bytes;
  int64_t cap;
  int hdr_words;
  __device__ __forceinline__ const int64_t* hdr(int r) const {
    return reinterpret_cast<const int64_t*>(base + (size_t)r * slab_bytes);
  }
  __device__ __forceinline__ const unsigned char* col(int r, size_t off) const {
    return base + (size_t)r * slab_bytes + off;
  }
};

__host__ __device__ inline size_t slab_i32_off(int hdr_words, int64_t cap, int k) {
  return (size_t)hdr_words * 8 + (size_t)k * 4 * (size_t)cap;
}
__host__ __device__ inline size_t slab_f64_off(int hdr_words, int64_t cap, int k) {
  const size_t base = ((size_t)hdr_words * 8 + 16 * (size_t)cap + 7) & ~(size_t)7;
  return base + (size_t)k * 8 * (size_t)cap;
}

// a / n correctly rounded from rn = RN(1/n) -- frontier.cu's div_n, same ops
__device__ __forceinline__ double merge_div_n(double a, double dn, double rn) {
  const double q0 = __dmul_rn(a, rn);
  return __fma_rn(__fma_rn(-q0, dn, a), rn, q0);
}

__global__ void __launch_bounds__(1024)
shard_offsets_kernel(SlabView sv, int world, const int32_t* __restrict__ pair_rank,
                     const int32_t* __restrict__ pair_local,
                     const int32_t* __restrict__ rank_npairs, int n_pairs,
                     int64_t* __restrict__ seg, int64_t out_cap, int64_t* __restrict__ out_stats) {
  __shared__ int64_t carry;
  __shared__ int64_t warp_sums[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n_pairs; base += blockDim.x) {
    const int g = base + threadIdx.x;
    int64_t cnt = 0, src = 0;
    if (g < n_pairs) {
      const int r = pair_rank[g], j = pair_local[g];
      const int64_t* h = sv.hdr(r);
      cnt = h[HADIS_ST_PAIR0 + j];
      for (int jj = 0; jj < j; ++jj) src += h[HADIS_ST_PAIR0 + jj];
    }
    int64_t x = cnt;                                  // block inclusive scan of the counts
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int64_t incl = x + (wid > 0 ? warp_sums[wid - 1] : 0) + carry;
    if (g < n_pairs) {
      seg[3 * g] = src;
      seg[3 * g + 1] = incl - cnt;
      seg[3 * g + 2] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int64_t of = 0, bad = 0, err = 0, max_rows = 0;
    for (int r = 0; r < world; ++r) {
      const int64_t* h = sv.hdr(r);
      of |= h[HADIS_ST_OVERFLOW];
      bad |= h[HADIS_ST_PAIR0 + rank_npairs[r]];
      err |= h[sv.hdr_words - 1];
      const int64_t rows = h[HADIS_ST_ROWS];
      max_rows = rows > max_rows ? rows : max_rows;
      if (rows > sv.cap) of |= 8;                     // a rank's rows did not fit its slab
    }
    if (carry > out_cap) of |= 8;
    out_stats[0] = carry;
    out_stats[1] = of;
    out_stats[2] = bad;
    out_stats[3] = err;
    out_stats[4] = max_rows;
  }
}

__global__ void __launch_bounds__(kMergeThreads)
shard_copy_kernel(SlabView sv, const int32_t* __restrict__ pair_rank,
                  const int64_t* __restrict__ seg, int64_t out_cap,
                  const int64_t* __restrict__ out_stats, const double* __restrict__ pair_params,
                  double dn, double rn, int32_t* __restrict__ o_pair,
                  int32_t* __restrict__ o_theta, int32_t* __restrict__ o_tau,
                  double* __restrict__ o_rl, double* __restrict__ o_rh,
                  double* __restrict__ o_fid, double* __restrict__ o_lat) {
  if (out_stats[1] != 0 || out_stats[2] != 0 || out_stats[3] != 0) return;  // rerun or raise
  const int g = blockIdx.y;
  const int r = pair_rank[g];
  const int64_t src = seg[3 * g], dst = seg[3 * g + 1], cnt = seg[3 * g + 2];
  const int32_t* th = reinterpret_cast<const int32_t*>(sv.col(r, slab_i32_off(sv.hdr_words, sv.cap, 0)));
  const int32_t* ta = reinterpret_cast<const int32_t*>(sv.col(r, slab_i32_off(sv.hdr_words, sv.cap, 1)));
  const uint32_t* nl = reinterpret_cast<const uint32_t*>(sv.col(r, slab_i32_off(sv.hdr_words, sv.cap, 2)));
  const uint32_t* nh = reinterpret_cast<const uint32_t*>(sv.col(r, slab_i32_off(sv.hdr_words, sv.cap, 3)));
  const double* fi = reinterpret_cast<const double*>(sv.col(r, slab_f64_off(sv.hdr_words, sv.cap, 0)));
  const double Ll = pair_params[(int64_t)g * HADIS_PAIR_PARAMS + 0];
  const double Lh = pair_params[(int64_t)g * HADIS_PAIR_PARAMS + 1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = src + i, d = dst + i;
    if (d >= out_cap) break;
    const double a = (double)nl[s], b = (double)nh[s];   // eval_cell's integers
    o_pair[d] = g;
    o_theta[d] = th[s];
    o_tau[d] = ta[s];
    o_rl[d] = merge_div_n(a, dn, rn);
    o_rh[d] = merge_div_n(b, dn, rn);
    o_fid[d] = fi[s];
    o_lat[d] = merge_div_n(__dadd_rn(__dmul_rn(a, Ll), __dmul_rn(b, Lh)), dn, rn);
  }
}

}  // namespace hadis

using namespace hadis;

extern "C" size_t hadis_shard_slab_bytes(int32_t hdr_words, int64_t cap) {
  if (hdr_words < HADIS_ST_PAIR0 + 2 || cap < 0) return 0;
  const size_t end = slab_f64_off(hdr_words, cap, 1);
  return (end + 255) & ~(size_t)255;
}

extern "C" size_t hadis_shard_merge_workspace_bytes(int32_t n_pairs) {
  if (n_pairs <= 0) return 0;
  return (size_t)n_pairs * 3 * sizeof(int64_t);
}

extern "C" int hadis_shard_merge(const void* gathered, int32_t world, size_t slab_bytes,
                                 int64_t cap, int32_t hdr_words, const int32_t* pair_rank,
                                 const int32_t* pair_local, const int32_t* rank_npairs,
                                 int32_t n_pairs, const double* pair_params, int64_t n,
                                 int64_t out_cap, int32_t* out_pair,
                                 int32_t* out_theta_pos, int32_t* out_tau_pos,
                                 double* out_r_light, double* out_r_heavy, double* out_fid,
                                 double* out_lat, int64_t* out_stats, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (!gathered || world <= 0 || cap < 0 || n_pairs <= 0 || n_pairs > 65535 || !pair_rank ||
      !pair_params || n <= 0 || n > 0xffffffffll ||
      !pair_local || !rank_npairs || !out_stats || !workspace || out_cap < 0 ||
      hadis_shard_slab_bytes(hdr_words, cap) == 0 ||
      slab_bytes < hadis_shard_slab_bytes(hdr_words, cap) ||
      (out_cap > 0 && (!out_pair || !out_theta_pos || !out_tau_pos || !out_r_light ||
                       !out_r_heavy || !out_fid || !out_lat)))
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_shard_merge_workspace_bytes(n_pairs)) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  SlabView sv{(const unsigned char*)gathered, slab_bytes, cap, hdr_words};
  int64_t* seg = (int64_t*)workspace;
  shard_offsets_kernel<<<1, 1024, 0, st>>>(sv, world, pair_rank, pair_local, rank_npairs,
                                           n_pairs, seg, out_cap, out_stats);
  shard_copy_kernel<<<dim3(kMergeChunks, n_pairs), kMergeThreads, 0, st>>>(
      sv, pair_rank, seg, out_cap, out_stats, pair_params, (double)n, 1.0 / (double)n, out_pair,
      out_theta_pos, out_tau_pos, out_r_light,
      out_r_heavy, out_fid, out_lat);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(2);
  return HADIS_OK;
}
