// Bit-exact emulation of numpy's float64 pairwise summation, as used by
// float(np.where(heavy, cost_heavy, cost_light).mean())  (profiler.py:152-153).
//
// numpy reduces a contiguous float64 array recursively: blocks of <= 128
// elements are summed with 8 interleaved accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus an in-order tail; blocks of < 8
// elements are summed left to right from 0.0; longer ranges are split at
// n/2 rounded down to a multiple of 8 and the halves added.  The association
// order depends only on n, so one CTA can evaluate the same tree in parallel:
// thread 0 expands the top of the recursion breadth-first, every thread sums
// whole subtrees depth-first (same association), and thread 0 folds the top
// tree back bottom-up.  The result is bitwise equal to numpy's (checked
// against numpy in tests/test_gpu_parity.py).
#pragma once

#include "common.cuh"

namespace hadis {

constexpr int kPwBlock = 128;         // numpy PW_BLOCKSIZE
constexpr int kPwThreads = 256;       // threads per emulation CTA
constexpr int kPwTopNodes = 1024;     // top-of-tree nodes kept in shared memory

struct CellCost {
  double theta, tau, base_l, pen_l, base_h, pen_h;
};

// value numpy puts at position q of np.where(h > theta | s < tau, c_heavy, c_light)
__device__ __forceinline__ double cell_value(const double* __restrict__ h,
                                             const double* __restrict__ s, int64_t q,
                                             const CellCost& c) {
  const double hq = h[q];
  const bool heavy = (hq > c.theta) || (s[q] < c.tau);
  const double base = heavy ? c.base_h : c.base_l;
  const double pen = heavy ? c.pen_h : c.pen_l;
  return __dadd_rn(base, __dmul_rn(pen, hq));
}

__device__ double pw_leaf(const double* __restrict__ h, const double* __restrict__ s, int64_t lo,
                          int64_t m, const CellCost& c) {
  if (m < 8) {
    double acc = 0.0;
    for (int64_t i = 0; i < m; ++i) acc = __dadd_rn(acc, cell_value(h, s, lo + i, c));
    return acc;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = cell_value(h, s, lo + j, c);
  const int64_t stop = m - (m % 8);
  int64_t i = 8;
  for (; i < stop; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], cell_value(h, s, lo + i + j, c));
  }
  double acc = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < m; ++i) acc = __dadd_rn(acc, cell_value(h, s, lo + i, c));
  return acc;
}

__device__ __forceinline__ int64_t pw_split(int64_t m) {
  int64_t half = m / 2;
  return half - (half % 8);
}

// depth-first pairwise sum of [lo, lo+m) with an explicit stack
__device__ double pw_subtree(const double* __restrict__ h, const double* __restrict__ s,
                             int64_t lo, int64_t m, const CellCost& c) {
  struct Frame { int64_t lo, m; double left; int stage; };
  Frame st[64];
  int sp = 0;
  st[0] = {lo, m, 0.0, 0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.m <= kPwBlock) {
      ret = pw_leaf(h, s, f.lo, f.m, c);
      --sp;
    } else if (f.stage == 0) {
      f.stage = 1;
      const int64_t half = pw_split(f.m);
      st[sp + 1] = {f.lo, half, 0.0, 0};
      ++sp;
    } else if (f.stage == 1) {
      f.left = ret;
      f.stage = 2;
      const int64_t half = pw_split(f.m);
      st[sp + 1] = {f.lo + half, f.m - half, 0.0, 0};
      ++sp;
    } else {
      ret = __dadd_rn(f.left, ret);
      --sp;
    }
  }
  return ret;
}

struct PwShared {
  int64_t off[kPwTopNodes];
  int64_t len[kPwTopNodes];
  int32_t child[kPwTopNodes];  // index of left child (right = left + 1), -1 = subtree root
  double val[kPwTopNodes];
  int32_t n_nodes;
};

// Whole-CTA numpy-exact sum of the cell's values over n records.
// Must be called by all threads of the block; result valid in thread 0.
__device__ double pw_block_sum(const double* __restrict__ h, const double* __restrict__ s,
                               int64_t n, const CellCost& c, PwShared& sh) {
  if (threadIdx.x == 0) {
    // breadth-first expansion of the recursion until enough independent subtrees;
    // children are appended after their parent, so a reverse sweep folds bottom-up
    sh.off[0] = 0;
    sh.len[0] = n;
    sh.child[0] = -1;
    int count = 1, expanded = 0;
    const int target = 2 * blockDim.x;
    for (int i = 0; i < count; ++i) {
      if (count - expanded >= target || count + 2 > kPwTopNodes) break;
      if (sh.len[i] <= kPwBlock) continue;
      const int64_t half = pw_split(sh.len[i]);
      sh.child[i] = count;
      sh.off[count] = sh.off[i];
      sh.len[count] = half;
      sh.child[count] = -1;
      sh.off[count + 1] = sh.off[i] + half;
      sh.len[count + 1] = sh.len[i] - half;
      sh.child[count + 1] = -1;
      count += 2;
      ++expanded;
    }
    sh.n_nodes = count;
  }
  __syncthreads();
  const int nn = sh.n_nodes;
  for (int i = threadIdx.x; i < nn; i += blockDim.x)
    if (sh.child[i] < 0) sh.val[i] = pw_subtree(h, s, sh.off[i], sh.len[i], c);
  __syncthreads();
  double total = 0.0;
  if (threadIdx.x == 0) {
    for (int i = nn - 1; i >= 0; --i)
      if (sh.child[i] >= 0) sh.val[i] = __dadd_rn(sh.val[sh.child[i]], sh.val[sh.child[i] + 1]);
    total = sh.val[0];
  }
  __syncthreads();
  return total;
}

// ---------------------------------------------------------------------------
// Many-CTA form for batches of cells over large n: the top of the recursion
// (shared by every cell, it depends only on n) is expanded once into a node
// table; a 2-D grid (subtree roots x cells) sums every root subtree, and one
// thread per cell folds the top tree.  Same association order as numpy.

constexpr int kPwPlanNodes = 1024;
constexpr int kPwPlanRoots = 512;

struct PwPlan {
  int n_nodes, n_roots;
  int64_t off[kPwPlanNodes];
  int64_t len[kPwPlanNodes];
  int32_t child[kPwPlanNodes];   // left child index (right = +1) or -1 for a root
  int32_t root[kPwPlanNodes];    // node index of the r-th root
};

// built in shared memory by one thread, then copied out by the block
// skip (no exact cells needed) when *need is 0; need == nullptr: always build
__global__ void __launch_bounds__(256) pw_plan_kernel(int64_t n, PwPlan* plan,
                                                      const unsigned long long* need) {
  __shared__ PwPlan sp;
  if (need && *need == 0) return;
  if (threadIdx.x == 0) {
    sp.off[0] = 0;
    sp.len[0] = n;
    sp.child[0] = -1;
    int count = 1, expanded = 0;
    for (int i = 0; i < count; ++i) {
      if (count - expanded >= kPwPlanRoots || count + 2 > kPwPlanNodes) break;
      if (sp.len[i] <= kPwBlock) continue;
      const int64_t half = pw_split(sp.len[i]);
      sp.child[i] = count;
      sp.off[count] = sp.off[i];
      sp.len[count] = half;
      sp.child[count] = -1;
      sp.off[count + 1] = sp.off[i] + half;
      sp.len[count + 1] = sp.len[i] - half;
      sp.child[count + 1] = -1;
      count += 2;
      ++expanded;
    }
    int r = 0;
    for (int i = 0; i < count; ++i)
      if (sp.child[i] < 0) sp.root[r++] = i;
    sp.n_nodes = count;
    sp.n_roots = r;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPwPlanNodes; i += blockDim.x) {
    plan->off[i] = sp.off[i];
    plan->len[i] = sp.len[i];
    plan->child[i] = sp.child[i];
    plan->root[i] = sp.root[i];
  }
  if (threadIdx.x == 0) { plan->n_nodes = sp.n_nodes; plan->n_roots = sp.n_roots; }
}

}  // namespace hadis
