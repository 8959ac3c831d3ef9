// Cascade-depth frontier points (reference
// pkg/src/cascadesim/frontier.py:60-120): every two-stage (light i < heavy j)
// and three-stage (light i < middle j < heavy k) operating point over a
// hardness population, from 3-D prefix tables instead of per-point masks.
//
// With u = the sorted distinct thresholds, bh = #{u < h}, bs_m = #{u <= s_m}:
//   T_ij[a][b][c] = #{q : bh <= a, bs_i <= b, bs_j <= c}  (+ fixed-point hardness sums)
// and for theta = u[a], tau1 = u[b], tau2 = u[c]:
//   not bypassed  R  = T[a][U][U]      reject1  C1 = T[a][b][U]   reject2 C2 = T[a][b][c]
//   two-stage  (i, j):   heavy = (n - R) + C1
//   three-stage (i, j, k): light = R - C1, middle = C1 - C2, heavy = (n - R) + C2
// Latencies follow the reference's float expressions exactly (-fmad=false):
//   two:   ((n - nb) L_i + (nb + nr) L_j) / n
//   three: ((R L_i + C1 L_j) + heavy L_k) / n
// Fidelity: sum over the stages of (b_m count + p_m hardness_sum 2^-shift), / n
// (a rounding-level restatement of numpy's sums; exact two-stage values come
// from hadis_fid_exact).
#include "common.cuh"

namespace hadis {

constexpr int kCascMaxModels = 16;

// model_params[m] = {latency_s[1], base cost, hardness penalty}, latency order
struct CascModels {
  const double* mp;
  __device__ double L(int m) const { return mp[3 * m]; }
  __device__ double b(int m) const { return mp[3 * m + 1]; }
  __device__ double p(int m) const { return mp[3 * m + 2]; }
};

// k-th (i < j < l) triple in lexicographic order
__device__ void triple_of(int idx, int M, int* ti, int* tj, int* tk) {
  for (int i = 0; i < M; ++i)
    for (int j = i + 1; j < M; ++j) {
      const int cnt = M - 1 - j;
      if (idx < cnt) { *ti = i; *tj = j; *tk = j + 1 + idx; return; }
      idx -= cnt;
    }
  *ti = *tj = *tk = 0;
}

// k-th (i < j) pair in lexicographic order
__device__ void pair_of(int idx, int M, int* pi, int* pj) {
  for (int i = 0; i < M; ++i) {
    const int cnt = M - 1 - i;
    if (idx < cnt) { *pi = i; *pj = i + 1 + idx; return; }
    idx -= cnt;
  }
  *pi = *pj = 0;
}

__device__ __forceinline__ int pair_index(int i, int j, int M) {   // i < j, row-major upper triangle
  return i * M - i * (i + 1) / 2 + (j - i - 1);
}

__global__ void cascade_hist_kernel(const double* __restrict__ h, const double* __restrict__ s,
                                    int64_t n, int M, const double* __restrict__ thr, int U,
                                    double hscale, uint32_t* __restrict__ cnt,
                                    unsigned long long* __restrict__ hs,
                                    uint32_t* __restrict__ bad) {
  const int B1 = U + 1;
  const int64_t cells = (int64_t)B1 * B1 * B1;
  uint32_t my_bad = 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double x = h[q];
    const bool ok = x >= 0.0 && x <= 1.0;
    my_bad += !ok;
    const int bh = count_less(thr, U, x);
    const unsigned long long hf = (unsigned long long)__dmul_rn(ok ? x : 0.0, hscale);
    int bs[kCascMaxModels];
    for (int m = 0; m < M; ++m) bs[m] = count_less_equal(thr, U, s[(int64_t)m * n + q]);
    for (int i = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j) {
        const int64_t at = (int64_t)pair_index(i, j, M) * cells + ((int64_t)bh * B1 + bs[i]) * B1 + bs[j];
        atomicAdd(&cnt[at], 1u);
        atomicAdd(&hs[at], hf);
      }
  }
  if (my_bad) atomicAdd(bad, my_bad);
}

// inclusive prefix along one axis of every table: line = (table, the other two
// coordinates), stride = the axis' element stride
__global__ void cascade_prefix_kernel(uint32_t* __restrict__ cnt,
                                      unsigned long long* __restrict__ hs, int n_tables, int B1,
                                      int axis) {
  const int64_t lines_per = (int64_t)B1 * B1;
  const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= lines_per * n_tables) return;
  const int64_t tbl = line / lines_per, r = line % lines_per;
  const int64_t o1 = r / B1, o2 = r % B1;
  int64_t base, stride;
  if (axis == 2) { base = (o1 * B1 + o2) * B1; stride = 1; }
  else if (axis == 1) { base = o1 * B1 * B1 + o2; stride = B1; }
  else { base = o1 * B1 + o2; stride = (int64_t)B1 * B1; }
  base += tbl * lines_per * B1;
  uint32_t c = 0;
  unsigned long long v = 0;
  for (int k = 0; k < B1; ++k) {
    c += cnt[base + k * stride];
    v += hs[base + k * stride];
    cnt[base + k * stride] = c;
    hs[base + k * stride] = v;
  }
}

// one thread per point; two-stage points first ([pair][a][b]), then
// three-stage ([triple][a][b][c]); out = (lat, fid) pairs
__global__ void cascade_points_kernel(const uint32_t* __restrict__ cnt,
                                      const unsigned long long* __restrict__ hs, int64_t n, int M,
                                      int U, double inv_scale, CascModels cp,
                                      double* __restrict__ out2, double* __restrict__ out3,
                                      int64_t n2, int64_t n3) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int B1 = U + 1;
  const int64_t cells = (int64_t)B1 * B1 * B1;
  const double dn = (double)n;
  auto at = [&](int a, int b, int c) { return ((int64_t)a * B1 + b) * B1 + c; };
  if (gid < n2) {
    const int64_t per = (int64_t)U * U;
    const int pr = (int)(gid / per);
    const int a = (int)(gid % per / U), b = (int)(gid % U);
    int i, j;
    pair_of(pr, M, &i, &j);
    const int64_t t = (int64_t)pair_index(i, j, M) * cells;
    const uint32_t R = cnt[t + at(a, U, U)], C1 = cnt[t + at(a, b, U)];
    const unsigned long long Htot = hs[t + at(U, U, U)], HR = hs[t + at(a, U, U)],
                             H1 = hs[t + at(a, b, U)];
    const uint32_t nb = (uint32_t)n - R, nH = nb + C1;
    const double lat = __ddiv_rn(__dadd_rn(__dmul_rn((double)((uint32_t)n - nb), cp.L(i)),
                                           __dmul_rn((double)nH, cp.L(j))), dn);
    const unsigned long long SH = (Htot - HR) + H1, SL = Htot - SH;
    const double fl = __dadd_rn(__dmul_rn(cp.b(i), (double)((uint32_t)n - nH)),
                                __dmul_rn(cp.p(i), __dmul_rn((double)SL, inv_scale)));
    const double fh = __dadd_rn(__dmul_rn(cp.b(j), (double)nH),
                                __dmul_rn(cp.p(j), __dmul_rn((double)SH, inv_scale)));
    out2[2 * gid] = lat;
    out2[2 * gid + 1] = __ddiv_rn(__dadd_rn(fh, fl), dn);
    return;
  }
  const int64_t g3 = gid - n2;
  if (g3 >= n3) return;
  const int64_t per = (int64_t)U * U * U;
  const int tr = (int)(g3 / per);
  const int64_t r = g3 % per;
  const int a = (int)(r / ((int64_t)U * U)), b = (int)(r / U % U), c = (int)(r % U);
  int i, j, k;
  triple_of(tr, M, &i, &j, &k);
  const int64_t t = (int64_t)pair_index(i, j, M) * cells;
  const uint32_t R = cnt[t + at(a, U, U)], C1 = cnt[t + at(a, b, U)], C2 = cnt[t + at(a, b, c)];
  const unsigned long long Htot = hs[t + at(U, U, U)], HR = hs[t + at(a, U, U)],
                           H1 = hs[t + at(a, b, U)], H2 = hs[t + at(a, b, c)];
  const uint32_t nL = R - C1, nM = C1 - C2, nH = ((uint32_t)n - R) + C2;
  const unsigned long long SL = HR - H1, SM = H1 - H2, SH = (Htot - HR) + H2;
  const double lat = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)R, cp.L(i)),
                                                   __dmul_rn((double)C1, cp.L(j))),
                                         __dmul_rn((double)nH, cp.L(k))), dn);
  auto part = [&](int m, uint32_t cn, unsigned long long sm) {
    return __dadd_rn(__dmul_rn(cp.b(m), (double)cn), __dmul_rn(cp.p(m), __dmul_rn((double)sm, inv_scale)));
  };
  out3[2 * g3] = lat;
  out3[2 * g3 + 1] = __ddiv_rn(__dadd_rn(__dadd_rn(part(i, nL, SL), part(j, nM, SM)), part(k, nH, SH)), dn);
}

}  // namespace hadis

using namespace hadis;

extern "C" size_t hadis_cascade_workspace_bytes(int32_t n_models, int32_t n_unique) {
  if (n_models < 2 || n_models > kCascMaxModels || n_unique <= 0) return 0;
  const size_t B1 = (size_t)n_unique + 1;
  const size_t tables = (size_t)n_models * (n_models - 1) / 2;
  return tables * B1 * B1 * B1 * 12 + 256;
}

extern "C" int hadis_cascade_points(const double* h, const double* scores, int64_t n,
                                    int32_t n_models, const double* model_params,
                                    const double* thr_unique, int32_t n_unique,
                                    int32_t hfix_shift, double* out_two, double* out_three,
                                    uint32_t* bad_records, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (!h || !scores || n <= 0 || n > 0xffffffffll || n_models < 2 ||
      n_models > kCascMaxModels || !model_params || !thr_unique || n_unique <= 0 ||
      !out_two || (n_models >= 3 && !out_three) || !bad_records || !workspace ||
      hfix_shift < 1 || hfix_shift > 62)
    return HADIS_ERR_ARG;
  if (workspace_bytes < hadis_cascade_workspace_bytes(n_models, n_unique)) return HADIS_ERR_CAPACITY;
  const CascModels cp{model_params};
  cudaStream_t st = (cudaStream_t)stream;
  const int B1 = n_unique + 1;
  const int M = n_models;
  const int tables = M * (M - 1) / 2;
  const int64_t cells = (int64_t)B1 * B1 * B1;
  uint32_t* cnt = (uint32_t*)workspace;
  unsigned long long* hs =
      (unsigned long long*)((char*)workspace + (((size_t)tables * cells * 4 + 255) & ~(size_t)255));
  HADIS_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)tables * cells * 4, st));
  HADIS_CUDA_TRY(cudaMemsetAsync(hs, 0, (size_t)tables * cells * 8, st));
  HADIS_CUDA_TRY(cudaMemsetAsync(bad_records, 0, 4, st));
  int64_t grid = ceil_div(n, 256);
  if (grid > kNumSMs * 8) grid = kNumSMs * 8;
  cascade_hist_kernel<<<(unsigned)grid, 256, 0, st>>>(h, scores, n, M, thr_unique, n_unique,
                                                      ldexp(1.0, hfix_shift), cnt, hs, bad_records);
  HADIS_LAUNCH_CHECK();
  const int64_t lines = (int64_t)tables * B1 * B1;
  for (int axis = 2; axis >= 0; --axis)
    cascade_prefix_kernel<<<(unsigned)ceil_div(lines, 256), 256, 0, st>>>(cnt, hs, tables, B1, axis);
  HADIS_LAUNCH_CHECK();
  const int64_t n2 = (int64_t)tables * n_unique * n_unique;
  const int64_t n3 = (int64_t)M * (M - 1) * (M - 2) / 6 * n_unique * n_unique * n_unique;
  cascade_points_kernel<<<(unsigned)ceil_div(n2 + n3, 256), 256, 0, st>>>(
      cnt, hs, n, M, n_unique, ldexp(1.0, -hfix_shift), cp, out_two, out_three, n2, n3);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(5);
  return HADIS_OK;
}
