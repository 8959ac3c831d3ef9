// Router weight sweep (reference pkg/src/cascadesim/router.py:199-234).
//
// For every weight vector w of the normalized grid and a labeled corpus with
// feature matrix X[N][F]: scores = X w, candidate thresholds = the midpoints
// between consecutive distinct scores plus one below / above, and the best
// balanced accuracy ((tp / n_pos + tn / n_neg) / 2, "hard" = score > c) with
// the first maximising threshold.  One CTA per weight vector: scores in shared
// memory, bitonic sort, prefix count of positives, then one binary search per
// candidate threshold -- O(N log^2 N) instead of the reference's O(N^2) mask.
//
// Scores reproduce numpy's float64 matrix-vector product on the reference
// machine bit for bit: four FMA accumulators over features f % 4, combined as
// (acc0 + acc2) + (acc1 + acc3) (verified against numpy on the golden corpora).
#include <cfloat>

#include "common.cuh"

namespace hadis {

constexpr int kTwMaxN = 8192;       // corpus size held in shared memory
constexpr int kTwThreads = 512;

__device__ __forceinline__ double numpy_dot(const double* __restrict__ x,
                                            const double* __restrict__ w, int F) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int f = 0; f < F; ++f) acc[f & 3] = __fma_rn(x[f], w[f], acc[f & 3]);
  return __dadd_rn(__dadd_rn(acc[0], acc[2]), __dadd_rn(acc[1], acc[3]));
}

__global__ void __launch_bounds__(kTwThreads)
tune_weights_kernel(const double* __restrict__ X, const uint8_t* __restrict__ labels, int N,
                    int F, const double* __restrict__ W, int V, int n_pos,
                    double* __restrict__ out_acc, double* __restrict__ out_thr) {
  extern __shared__ __align__(16) unsigned char smem[];
  int npow = 1;
  while (npow < N) npow <<= 1;
  double* s = reinterpret_cast<double*>(smem);                 // [npow] scores
  int* pp = reinterpret_cast<int*>(s + npow);                   // [npow + 1] positives before i
  int* gs = pp + npow + 1;                                      // [npow] group starts
  uint8_t* lab = reinterpret_cast<uint8_t*>(gs + npow);         // [npow]
  __shared__ int s_ngroups;
  __shared__ double s_best_acc[kTwThreads / 32];
  __shared__ int s_best_idx[kTwThreads / 32];
  const int n_neg = N - n_pos;
  for (int v = blockIdx.x; v < V; v += gridDim.x) {
    const double* w = W + (int64_t)v * F;
    for (int i = threadIdx.x; i < npow; i += blockDim.x) {
      s[i] = i < N ? numpy_dot(X + (int64_t)i * F, w, F) : INFINITY;
      lab[i] = i < N ? labels[i] : 0;
    }
    __syncthreads();
    for (int size = 2; size <= npow; size <<= 1) {               // bitonic sort by score
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < npow; i += blockDim.x) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            if ((s[i] > s[j]) == up) {
              const double t = s[i]; s[i] = s[j]; s[j] = t;
              const uint8_t b = lab[i]; lab[i] = lab[j]; lab[j] = b;
            }
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {                                       // prefix counts + groups
      int run = 0, g = 0;
      for (int i = 0; i < N; ++i) {
        pp[i] = run;
        run += lab[i];
        if (i == 0 || s[i] != s[i - 1]) gs[g++] = i;
      }
      pp[N] = run;
      s_ngroups = g;
    }
    __syncthreads();
    const int u = s_ngroups;
    double best = -1.0;
    int best_j = 0x7fffffff;
    for (int j = threadIdx.x; j <= u; j += blockDim.x) {        // candidate thresholds
      double c;
      if (j == 0) c = __dadd_rn(s[gs[0]], -1.0);
      else if (j == u) c = __dadd_rn(s[gs[u - 1]], 1.0);
      else c = __ddiv_rn(__dadd_rn(s[gs[j - 1]], s[gs[j]]), 2.0);
      int lo = 0, hi = N;                                        // #{s <= c}
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (s[mid] <= c) lo = mid + 1; else hi = mid; }
      const int pos_le = pp[lo];
      const int tp = n_pos - pos_le, tn = lo - pos_le;
      const double acc = __ddiv_rn(__dadd_rn(__ddiv_rn((double)tp, (double)n_pos),
                                             __ddiv_rn((double)tn, (double)n_neg)), 2.0);
      if (acc > best || (acc == best && j < best_j)) { best = acc; best_j = j; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {                      // first maximum
      const double oa = __shfl_down_sync(0xffffffffu, best, off);
      const int oj = __shfl_down_sync(0xffffffffu, best_j, off);
      if (oa > best || (oa == best && oj < best_j)) { best = oa; best_j = oj; }
    }
    if (lane == 0) { s_best_acc[warp] = best; s_best_idx[warp] = best_j; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
        if (s_best_acc[k] > best || (s_best_acc[k] == best && s_best_idx[k] < best_j)) {
          best = s_best_acc[k];
          best_j = s_best_idx[k];
        }
      const int j = best_j;
      out_acc[v] = best;
      out_thr[v] = j == 0 ? __dadd_rn(s[gs[0]], -1.0)
                          : (j == u ? __dadd_rn(s[gs[u - 1]], 1.0)
                                    : __ddiv_rn(__dadd_rn(s[gs[j - 1]], s[gs[j]]), 2.0));
    }
    __syncthreads();
  }
}

}  // namespace hadis

using namespace hadis;

extern "C" int hadis_tune_weights(const double* features, const uint8_t* labels, int32_t n,
                                  int32_t n_features, const double* weights, int32_t n_vectors,
                                  int32_t n_pos, double* out_acc, double* out_threshold,
                                  void* stream) {
  if (!features || !labels || n <= 1 || n_features <= 0 || n_features > 64 || !weights ||
      n_vectors <= 0 || n_pos <= 0 || n_pos >= n || !out_acc || !out_threshold)
    return HADIS_ERR_ARG;
  if (n > kTwMaxN) return HADIS_ERR_UNSUPPORTED;
  int npow = 1;
  while (npow < n) npow <<= 1;
  const size_t smem = (size_t)npow * 8 + (size_t)(npow + 1) * 4 + (size_t)npow * 4 + npow + 16;
  HADIS_CUDA_TRY(hadis_ensure_smem((const void*)tune_weights_kernel, (size_t)smem));
  const int grid = n_vectors < kNumSMs * 4 ? n_vectors : kNumSMs * 4;
  tune_weights_kernel<<<grid, kTwThreads, smem, (cudaStream_t)stream>>>(
      features, labels, n, n_features, weights, n_vectors, n_pos, out_acc, out_threshold);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}
