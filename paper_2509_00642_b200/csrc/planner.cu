// K5: allocation search -- planner.solve over many (demand, SLO) points.
//
// Reference: pkg/src/cascadesim/planner.py
//   queue_delay       :81-85   alpha * Q / max(rate, 0.01), 0 when Q <= 0
//   _path_terms       :93-104  sum(latency + drain) over the row's models
//   _min_workers      :107-110 max(1, ceil((rate - 1e-9) / mu)), 1 when rate <= 0
//   _evaluate_row     :113-148 per row min (total, path), first combo wins
//   _solve_over_rows  :151-167 min (fidelity, total, path, row index)
//   fallback_plan     :170-214 max bottleneck capacity over worker splits,
//                              key (-capacity, L_light[1], L_heavy[1], row index)
//   solve             :217-227 negative demand -> PlannerError (host wrapper;
//                              the search itself takes any demand, like
//                              _solve_over_rows / fallback_plan do)
// One thread evaluates one (point, row) -- all batch combos -- and CTAs reduce
// to a per-(point, CTA) best; a second kernel reduces the CTA partials.  All
// float64 operations are the reference's, in its order, without FMA.
#include <cmath>

#include "common.cuh"

namespace hadis {

constexpr int kPlanThreads = 256;
constexpr int kMaxBatch = 16;
constexpr double kSlack = 1e-9;
constexpr double kRateFloor = 0.01;

struct Best {
  double k0;      // fidelity (solve) or -capacity (fallback)
  double k1;      // total workers (solve) or latency_s[1] light (fallback)
  double k2;      // path latency (solve) or latency_s[1] heavy (fallback)
  int32_t row;    // -1 = none
  int32_t xl, xh, bl, bh;
  double path;
};

__device__ __forceinline__ bool better(const Best& a, const Best& b) {
  if (a.row < 0) return false;
  if (b.row < 0) return true;
  if (a.k0 != b.k0) return a.k0 < b.k0;
  if (a.k1 != b.k1) return a.k1 < b.k1;
  if (a.k2 != b.k2) return a.k2 < b.k2;
  return a.row < b.row;
}

struct PlanIn {
  int n_rows;
  const int32_t* row_model;
  const double* row_share;
  const double* row_fid;
  int n_models, n_batch;
  const int32_t* batch;
  const double* lat;
  const double* mu;
  const double* lat1;
  int n_points;
  const double* lam;
  const double* t_slo;
  const int32_t* workers;
  const double* queues;
  double alpha;
};

__device__ __forceinline__ double drain(double q, double rate, double alpha) {
  if (!(q > 0.0)) return 0.0;
  const double r = rate > kRateFloor ? rate : (rate == kRateFloor ? rate : kRateFloor);
  return __ddiv_rn(__dmul_rn(alpha, q), r);
}

__device__ __forceinline__ int64_t min_workers(double rate, double mu) {
  if (rate <= 0.0) return 1;
  const double need = ceil(__ddiv_rn(__dadd_rn(rate, -kSlack), mu));
  if (!(need < 4.0e18)) return (int64_t)4e18;
  const int64_t x = (int64_t)need;
  return x > 1 ? x : 1;
}

struct RowShape {
  int ml, mh;          // model indices
  bool single;         // light == heavy
  double sl, sh;       // shares (sh unused when single)
  bool al, ah;         // active flags
};

__device__ __forceinline__ RowShape row_shape(const PlanIn& in, int r) {
  RowShape s;
  s.ml = in.row_model[2 * r];
  s.mh = in.row_model[2 * r + 1];
  s.single = s.ml == s.mh;
  const double rl = in.row_share[2 * r], rh = in.row_share[2 * r + 1];
  if (s.single) {
    s.sl = __dadd_rn(rl, rh);
    s.sh = 0.0;
  } else {
    s.sl = rl;
    s.sh = __dadd_rn(0.0, rh);
  }
  s.al = s.sl > 0.0;
  s.ah = !s.single && s.sh > 0.0;
  return s;
}

// path latency of the row's models at batch indices (il, ih) -- planner.py:93-104
__device__ __forceinline__ double path_latency(const PlanIn& in, const RowShape& s, int p, int il,
                                               int ih, double lamv) {
  const double* Q = in.queues + (int64_t)p * in.n_models;
  double path = __dadd_rn(0.0, __dadd_rn(in.lat[s.ml * in.n_batch + il],
                                         drain(Q[s.ml], __dmul_rn(lamv, s.sl), in.alpha)));
  if (!s.single)
    path = __dadd_rn(path, __dadd_rn(in.lat[s.mh * in.n_batch + ih],
                                     drain(Q[s.mh], __dmul_rn(lamv, s.sh), in.alpha)));
  return path;
}

// _evaluate_row (planner.py:113-148).  The drains and each model's worker
// count depend on the batch of that model only, so they are evaluated once per
// row (two drains) and once per batch size (min_workers), not once per combo;
// every value is the same float64 operation on the same operands as the
// reference's per-combo recomputation.
__device__ Best eval_row(const PlanIn& in, int p, int r) {
  Best best;
  best.row = -1;
  const RowShape s = row_shape(in, r);
  const double lamv = in.lam[p];
  const int W = in.workers[p];
  const double limit = __dadd_rn(in.t_slo[p], kSlack);
  const int nb = in.n_batch;
  const int nl = s.al ? nb : 1;
  const int nh = s.ah ? nb : 1;
  const double* Q = in.queues + (int64_t)p * in.n_models;
  const double rate_l = __dmul_rn(lamv, s.sl);
  const double dl = drain(Q[s.ml], rate_l, in.alpha);
  double rate_h = 0.0, dh = 0.0;
  if (!s.single) {
    rate_h = __dmul_rn(lamv, s.sh);
    dh = drain(Q[s.mh], rate_h, in.alpha);
  }
  int64_t xh_b[kMaxBatch];
  for (int ih = 0; ih < nh; ++ih)
    xh_b[ih] = s.ah ? min_workers(rate_h, in.mu[s.mh * nb + ih]) : 0;
  double best_total = 0.0, best_path = 0.0;
  for (int il = 0; il < nl; ++il) {
    const int64_t xl = s.al ? min_workers(rate_l, in.mu[s.ml * nb + il]) : 0;
    if (xl > W) continue;                             // every combo of this il is over budget
    const double pl = __dadd_rn(0.0, __dadd_rn(in.lat[s.ml * nb + il], dl));
    for (int ih = 0; ih < nh; ++ih) {
      const int64_t total = xl + xh_b[ih];
      if (total > W) continue;
      const double path = s.single ? pl : __dadd_rn(pl, __dadd_rn(in.lat[s.mh * nb + ih], dh));
      if (path > limit) continue;
      const double tot = (double)total;
      if (best.row < 0 || tot < best_total || (tot == best_total && path < best_path)) {
        best.row = r;
        best_total = tot;
        best_path = path;
        best.xl = (int32_t)xl;
        best.xh = (int32_t)xh_b[ih];
        best.bl = il;
        best.bh = ih;
      }
    }
  }
  if (best.row >= 0) {
    best.k0 = in.row_fid[r];
    best.k1 = best_total;
    best.k2 = best_path;
    best.path = best_path;
  }
  return best;
}

// eval_row with the batch loops unrolled for n_batch <= kNB: the heavy model's
// per-batch worker counts stay in registers (the generic version keeps them in
// a local-memory array), counts clamped to W + 1 (only "> W" is ever asked)
template <int kNB>
__device__ Best eval_row_small(const PlanIn& in, int p, int r) {
  Best best;
  best.row = -1;
  const RowShape s = row_shape(in, r);
  const double lamv = in.lam[p];
  const int W = in.workers[p];
  const double limit = __dadd_rn(in.t_slo[p], kSlack);
  const int nb = in.n_batch;
  const int nl = s.al ? nb : 1;
  const int nh = s.ah ? nb : 1;
  const double* Q = in.queues + (int64_t)p * in.n_models;
  const double rate_l = __dmul_rn(lamv, s.sl);
  const double dl = drain(Q[s.ml], rate_l, in.alpha);
  double rate_h = 0.0, dh = 0.0;
  if (!s.single) {
    rate_h = __dmul_rn(lamv, s.sh);
    dh = drain(Q[s.mh], rate_h, in.alpha);
  }
  auto clampw = [&](int64_t x) { return (int)(x > (int64_t)W ? (int64_t)W + 1 : x); };
  int xh_b[kNB];
#pragma unroll
  for (int ih = 0; ih < kNB; ++ih)
    xh_b[ih] = (ih < nh && s.ah) ? clampw(min_workers(rate_h, in.mu[s.mh * nb + ih])) : 0;
  double best_total = 0.0, best_path = 0.0;
#pragma unroll 1
  for (int il = 0; il < nl; ++il) {
    const int xl = s.al ? clampw(min_workers(rate_l, in.mu[s.ml * nb + il])) : 0;
    if (xl > W) continue;                             // every combo of this il is over budget
    const double pl = __dadd_rn(0.0, __dadd_rn(in.lat[s.ml * nb + il], dl));
#pragma unroll
    for (int ih = 0; ih < kNB; ++ih) {
      if (ih >= nh) break;
      const int total = xl + xh_b[ih];
      if (total > W) continue;
      const double path = s.single ? pl : __dadd_rn(pl, __dadd_rn(in.lat[s.mh * nb + ih], dh));
      if (path > limit) continue;
      const double tot = (double)total;
      if (best.row < 0 || tot < best_total || (tot == best_total && path < best_path)) {
        best.row = r;
        best_total = tot;
        best_path = path;
        best.xl = xl;
        best.xh = xh_b[ih];
        best.bl = il;
        best.bh = ih;
      }
    }
  }
  if (best.row >= 0) {
    best.k0 = in.row_fid[r];
    best.k1 = best_total;
    best.k2 = best_path;
    best.path = best_path;
  }
  return best;
}

// fallback_plan candidate of one row (planner.py:179-208)
__device__ Best fallback_row(const PlanIn& in, int p, int r) {
  Best best;
  best.row = -1;
  const RowShape s = row_shape(in, r);
  if (!s.al && !s.ah) return best;
  const int W = in.workers[p];
  const double lamv = in.lam[p];
  const double lat_l = in.lat1[s.ml], lat_h = in.lat1[s.mh];
  const int nl = s.al ? in.n_batch : 1;
  const int nh = s.ah ? in.n_batch : 1;
  const bool two = s.al && s.ah;
  for (int il = 0; il < nl; ++il) {
    for (int ih = 0; ih < nh; ++ih) {
      const double mul = s.al ? in.mu[s.ml * in.n_batch + il] : 0.0;
      const double muh = s.ah ? in.mu[s.mh * in.n_batch + ih] : 0.0;
      const int i0 = two ? 1 : 0, i1 = two ? W - 1 : 0;
      for (int i = i0; i <= i1; ++i) {
        int xl, xh;
        double cap;
        if (two) {
          xl = i;
          xh = W - i;
          const double cl = __ddiv_rn(__dmul_rn((double)xl, mul), s.sl);
          const double ch = __ddiv_rn(__dmul_rn((double)xh, muh), s.sh);
          cap = ch < cl ? ch : cl;
        } else if (s.al) {
          xl = W; xh = 0;
          cap = __ddiv_rn(__dmul_rn((double)W, mul), s.sl);
        } else {
          xl = 0; xh = W;
          cap = __ddiv_rn(__dmul_rn((double)W, muh), s.sh);
        }
        Best c;
        c.k0 = -cap; c.k1 = lat_l; c.k2 = lat_h; c.row = r;
        c.xl = xl; c.xh = xh; c.bl = il; c.bh = ih;
        if (better(c, best)) {
          c.path = path_latency(in, s, p, il, ih, lamv);
          best = c;
        }
      }
    }
  }
  return best;
}

__device__ void block_reduce_store(Best mine, Best* out) {
  __shared__ Best sh[kPlanThreads];
  sh[threadIdx.x] = mine;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off && better(sh[threadIdx.x + off], sh[threadIdx.x]))
      sh[threadIdx.x] = sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// grid: (row blocks, points)
#ifndef HADIS_K5_MINB
#define HADIS_K5_MINB 4      // 4 CTAs/SM (64 registers): c5 2.97 -> 1.92 ms; 1 or 2: 101-108 registers
#endif
__global__ void __launch_bounds__(kPlanThreads, HADIS_K5_MINB)
solve_rows_kernel(PlanIn in, int fallback, const int32_t* __restrict__ need_fb,
                  Best* __restrict__ partial) {
  const int p = blockIdx.y;
  if (fallback && !need_fb[p]) return;
  Best mine;
  mine.row = -1;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < in.n_rows;
       r += gridDim.x * blockDim.x) {
    const Best c = fallback ? fallback_row(in, p, r)
                            : (in.n_batch <= 8 ? eval_row_small<8>(in, p, r) : eval_row(in, p, r));
    if (better(c, mine)) mine = c;
  }
  block_reduce_store(mine, partial + (int64_t)p * gridDim.x + blockIdx.x);
}

__global__ void __launch_bounds__(kPlanThreads)
reduce_points_kernel(PlanIn in, int fallback, int nblk, const Best* __restrict__ partial,
                     int32_t* __restrict__ need_fb, int32_t* plan_row, int32_t* plan_x,
                     int32_t* plan_b, double* plan_path, int32_t* plan_flags) {
  const int p = blockIdx.x;
  if (fallback && !need_fb[p]) return;
  Best mine;
  mine.row = -1;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    const Best c = partial[(int64_t)p * nblk + b];
    if (better(c, mine)) mine = c;
  }
  __shared__ Best res;
  block_reduce_store(mine, &res);
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (!fallback) {
    need_fb[p] = res.row < 0;
    if (res.row < 0) return;
  }
  plan_row[p] = res.row;
  if (res.row >= 0) {
    plan_x[2 * p] = res.xl;
    plan_x[2 * p + 1] = res.xh;
    plan_b[2 * p] = in.batch[res.bl];
    plan_b[2 * p + 1] = in.batch[res.bh];
    plan_path[p] = res.path;
  }
  plan_flags[p] = fallback ? 1 : 0;
}

}  // namespace hadis

using namespace hadis;

static int plan_blocks(int n_rows) {
  int b = (n_rows + kPlanThreads - 1) / kPlanThreads;
  if (b < 1) b = 1;
  if (b > 64) b = 64;
  return b;
}

extern "C" size_t hadis_solve_workspace_bytes(int32_t n_points, int32_t n_rows) {
  if (n_points <= 0 || n_rows <= 0) return 0;
  return (size_t)n_points * plan_blocks(n_rows) * sizeof(Best) + (size_t)n_points * 4 + 256;
}

extern "C" int hadis_solve_many(int32_t n_rows, const int32_t* row_model, const double* row_share,
                                const double* row_fid, int32_t n_models, int32_t n_batch,
                                const int32_t* batch_sizes, const double* lat, const double* mu,
                                const double* lat1, int32_t n_points, const double* lam,
                                const double* t_slo, const int32_t* workers, const double* queues,
                                double alpha, int32_t* plan_row, int32_t* plan_x, int32_t* plan_b,
                                double* plan_path, int32_t* plan_flags, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (n_rows <= 0 || n_points <= 0 || n_models <= 0 || n_batch <= 0 || n_batch > kMaxBatch ||
      !row_model || !row_share || !row_fid || !batch_sizes || !lat || !mu || !lat1 || !lam ||
      !t_slo || !workers || !queues || !plan_row || !plan_x || !plan_b || !plan_path ||
      !plan_flags || !workspace || n_points > 65535)
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_solve_workspace_bytes(n_points, n_rows)) return HADIS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = plan_blocks(n_rows);
  Best* partial = (Best*)workspace;
  int32_t* need_fb = (int32_t*)((char*)workspace + (size_t)n_points * nblk * sizeof(Best));
  PlanIn in{n_rows, row_model, row_share, row_fid, n_models, n_batch, batch_sizes, lat, mu,
            lat1, n_points, lam, t_slo, workers, queues, alpha};
  dim3 grid(nblk, n_points);
  solve_rows_kernel<<<grid, kPlanThreads, 0, st>>>(in, 0, need_fb, partial);
  reduce_points_kernel<<<n_points, kPlanThreads, 0, st>>>(in, 0, nblk, partial, need_fb, plan_row,
                                                          plan_x, plan_b, plan_path, plan_flags);
  solve_rows_kernel<<<grid, kPlanThreads, 0, st>>>(in, 1, need_fb, partial);
  reduce_points_kernel<<<n_points, kPlanThreads, 0, st>>>(in, 1, nblk, partial, need_fb, plan_row,
                                                          plan_x, plan_b, plan_path, plan_flags);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(4);
  return HADIS_OK;
}
