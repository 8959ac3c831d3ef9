/*
 * hadis_b200.h -- C ABI of libhadis_b200.so, the B200 (sm_100a) implementation
 * of HADIS's offline cascade-profiling + runtime-allocation hot path.
 *
 * The reference (cascadesim 0.1.0, pure Python + numpy) has no native code and
 * no FFI; its Python entry points are the contract.  Each function below is
 * the device-side replacement of one stage of those entry points and cites the
 * reference code it replaces (paths relative to /root/reference/pkg/src/cascadesim).
 * INTEGRATION.md shows the ctypes binding cascadesim would add.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers owned by the caller (allocate with
 *     cudaMalloc, torch, cupy ...).  Nothing here allocates device memory except
 *     out of a caller-provided workspace.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every call only enqueues work; nothing synchronises the host.
 *   - Return value: 0 (HADIS_OK) or a hadis_status code.  Data-dependent
 *     failures that can only be known on the device (bad records, capacity
 *     overflow) are reported through the `stats` arrays documented per call.
 *   - float64 arithmetic that must match the reference bit for bit is compiled
 *     without FMA contraction (-fmad=false + __d*_rn intrinsics).
 */
#ifndef HADIS_B200_H
#define HADIS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HADIS_ABI_VERSION 1

enum hadis_status {
  HADIS_OK = 0,
  HADIS_ERR_ARG = 1,          /* invalid argument (sizes, null pointers)          */
  HADIS_ERR_RECORDS = 2,      /* hardness not finite or outside [0, 1]            */
  HADIS_ERR_CAPACITY = 3,     /* caller buffer / workspace too small              */
  HADIS_ERR_CUDA = 4,         /* CUDA runtime error (hadis_last_cuda_error)       */
  HADIS_ERR_NO_ROWS = 5,      /* planner: "fallback: no serveable rows"           */
  HADIS_ERR_NEG_DEMAND = 6,   /* planner: "solve: negative demand"                */
  HADIS_ERR_UNSUPPORTED = 7   /* outside the implemented envelope */
};

int hadis_abi_version(void);
const char* hadis_status_string(int status);
const char* hadis_last_cuda_error(void);
/* Number of CUDA kernels this library has launched in the process (monotone). */
int64_t hadis_kernel_launches(void);

/* ------------------------------------------------------------------------- */
/* Profiling: grid evaluator + Pareto extractor                               */
/* replaces profiler.profile_config's numeric core (profiler.py:133-174) and   */
/* catalog.pareto_prune as it is used there (catalog.py:171-192).              */
/* ------------------------------------------------------------------------- */

/* Fixed-point scale for hardness sums: h_fix = floor(h * 2^shift), with
 * shift = min(48, 63 - bit_length(n)) so every sum of n values fits in 63 bits
 * and one record's h_fix (relative to its row's lower bound) splits into at most
 * three 16-bit K1 shared-memory limbs. */
int hadis_hfix_shift(int64_t n);

/* K1 -- bin + 2-D histogram (profiler.py:138, 145-150: bypass h > theta,
 * reject score < tau), records in any order.  For every record q and light
 * model l:
 *   bh = #{u < h[q]},  bs = #{u <= s_l[q]}   (u = sorted distinct thresholds)
 *   hist_cnt [l][bh][bs] += 1 ;  hist_hsum[l][bh][bs] += floor(h[q] * 2^shift)
 * scores: n_light rows of n float64 (row stride n).  Histograms have
 * (n_unique+1)^2 cells per light model and are zeroed by this call; L2
 * integer atomics (or shared-memory privatisation for small grids).
 * bad_records (device uint32) counts records with h outside [0, 1] / NaN. */
int hadis_bin_hist(const double* h, const double* scores, int64_t n, int32_t n_light,
                   const double* thr_unique, int32_t n_unique, int32_t hfix_shift,
                   uint32_t* hist_cnt, uint64_t* hist_hsum, uint32_t* bad_records,
                   void* stream);

/* Row-bucketed record store (profiler.py:138, 145-150), per threshold grid:
 * records are grouped by their theta-row bh = #{u < h} so that K1 needs no
 * global atomics.  One pass reads h and the n_light score rows (row stride n)
 * once and writes, row-bucketed (rows in bh order, order within a row
 * unspecified):
 *   hfix_rows[i]            = floor(h * 2^hfix_shift)      (uint64[n])
 *   bs_rows[l/4][i][l%4]    = #{u <= s_l}  (the tau-bin)    (uint16, model quads)
 * bs_rows holds hadis_bs_store_elems(n, n_light) uint16 (light models padded
 * to a multiple of 4, quad rows of n rounded up to even records): one 8-byte
 * word per record and quad of models.
 * row_plan (hadis_row_plan_bytes) receives the row offsets and K1's work
 * items; pass it unchanged to hadis_bin_hist_rows.  bad_records (device
 * uint32, may be NULL) counts hardness values that are NaN or outside [0, 1].
 * Supports up to 2047 distinct thresholds (hadis_bin_hist covers larger). */
size_t hadis_row_plan_bytes(int32_t n_unique);
int64_t hadis_bs_store_elems(int64_t n, int32_t n_light);
int hadis_records_bucket(const double* h, const double* scores, int64_t n, int32_t n_light,
                         const double* thr_unique, int32_t n_unique, int32_t hfix_shift,
                         uint64_t* hfix_rows, uint16_t* bs_rows, uint32_t* bad_records,
                         void* row_plan, size_t row_plan_bytes, void* stream);
/* The same in two steps: hadis_records_plan reads h only (guides, row counts,
 * row offsets, K1 items -> row_plan); hadis_records_scatter is the
 * HBM-bound pass over every record array (needs the plan). */
int hadis_records_plan(const double* h, int64_t n, const double* thr_unique, int32_t n_unique,
                       int32_t hfix_shift, uint32_t* bad_records, void* row_plan,
                       size_t row_plan_bytes, void* stream);
int hadis_records_scatter(const double* h, const double* scores, int64_t n, int32_t n_light,
                          const double* thr_unique, int32_t n_unique, int32_t hfix_shift,
                          uint64_t* hfix_rows, uint16_t* bs_rows, void* row_plan,
                          size_t row_plan_bytes, void* stream);

/* K1 on the row-bucketed store: the same histogram as hadis_bin_hist, one CTA
 * per (row chunk, light model) accumulating in shared memory.  Rows a CTA
 * owns whole are stored already prefix-summed along bs and flagged in
 * row_scanned[l][k] (may be NULL: plain histogram). */
int hadis_bin_hist_rows(const uint64_t* hfix_rows, const uint16_t* bs_rows, int64_t n,
                        int32_t n_light, int32_t n_unique, const void* row_plan,
                        uint32_t* hist_cnt, uint64_t* hist_hsum, uint8_t* row_scanned,
                        void* stream);

/* K2 -- in-place 2-D inclusive prefix sums of the K1 histograms:
 *   cnt[l][k][t] = #{q : bh(q) <= k, bs_l(q) <= t}  (and the same for hsum).
 * row_scanned[l][k] != 0 (may be NULL) marks rows K1 already prefix-summed
 * along bs (hadis_bin_hist_sorted does so for every row it owns whole). */
int hadis_hist_scan(uint32_t* hist_cnt, uint64_t* hist_hsum, int32_t n_light,
                    int32_t n_unique, const uint8_t* row_scanned, void* stream);

/* Per-pair parameters, row-major [n_pairs][HADIS_PAIR_PARAMS] doubles:
 * {latency_s[1] light, latency_s[1] heavy, base cost light, penalty light,
 *  base cost heavy, penalty heavy}. */
#define HADIS_PAIR_PARAMS 6

/* Layout of the `stats` int64 array written by hadis_pair_frontiers. */
enum hadis_frontier_stat {
  HADIS_ST_ROWS = 0,        /* total output rows                                  */
  HADIS_ST_CANDIDATES = 1,  /* main-universe candidates that passed the filter    */
  HADIS_ST_UNCERTAIN = 2,   /* decisions resolved with the exact numpy emulation  */
  HADIS_ST_EXACT_CELLS = 3, /* cells whose fidelity was recomputed exactly        */
  HADIS_ST_OVERFLOW = 4,    /* nonzero: a capacity was exceeded, rerun bigger     */
  HADIS_ST_PAIR0 = 8        /* then n_pairs per-pair output row counts            */
};

size_t hadis_frontier_workspace_bytes(int32_t n_pairs, int32_t n_unique, int64_t cand_cap,
                                      int64_t exact_cap, int64_t out_cap);

/* K3 + K4 -- per pair (light slot, heavy): evaluate every (theta, tau) cell
 * from the K2 prefix tables, extract the latency/fidelity Pareto frontier and
 * the theta = max(thresholds) no-bypass frontier, merge them and emit the rows
 * sorted by (theta, tau) -- profiler.py:140-174.  Decisions are exact: cells
 * whose order against another cell cannot be certified from the fixed-point
 * fidelity bound are recomputed with a bit-exact emulation of numpy's
 * pairwise mean over (h, scores) and decided on those values.
 *
 *   pre_cnt / pre_hsum : K2 output, slots indexed by pair_slot[p]
 *   pair_slot[p]       : light-model slot (row of `scores`, K1/K2 slot)
 *   pair_params        : [n_pairs][HADIS_PAIR_PARAMS]
 *   first_pos[r]       : smallest position in the caller's threshold list of
 *                        the r-th smallest distinct threshold value
 *   n_thresholds       : length of the caller's threshold list (K)
 *   exact_fid          : nonzero = recompute the fidelity of every OUTPUT row
 *                        with the numpy emulation (bit-identical rows)
 *   outputs (capacity out_cap rows, pair-major, (theta, tau) order):
 *     out_pair, out_theta_pos, out_tau_pos (positions in the caller's list),
 *     out_r_light, out_r_heavy, out_fid, out_lat
 *   stats              : int64[HADIS_ST_PAIR0 + n_pairs], see hadis_frontier_stat */
int hadis_pair_frontiers(const uint32_t* pre_cnt, const uint64_t* pre_hsum, int64_t n,
                         int32_t n_unique, int32_t hfix_shift, int32_t n_pairs,
                         const int32_t* pair_slot, const double* pair_params,
                         const int32_t* first_pos, int32_t n_thresholds,
                         const double* thr_unique, const double* h, const double* scores,
                         int32_t exact_fid, void* workspace, size_t workspace_bytes,
                         int64_t cand_cap, int64_t exact_cap, int64_t out_cap,
                         int32_t* out_pair, int32_t* out_theta_pos, int32_t* out_tau_pos,
                         double* out_r_light, double* out_r_heavy, double* out_fid,
                         double* out_lat, int64_t* stats, void* stream);
/* The same frontier with compact rows (the multi-GPU slab, 24 bytes per row):
 * theta_pos, tau_pos, fid as above, n_light = records the light stage serves
 * (r_light * n), n_heavy = records the heavy stage serves (r_heavy * n); the
 * pair of a row is implied by the per-pair row counts in stats. */
int hadis_pair_frontiers_compact(const uint32_t* pre_cnt, const uint64_t* pre_hsum, int64_t n,
                                 int32_t n_unique, int32_t hfix_shift, int32_t n_pairs,
                                 const int32_t* pair_slot, const double* pair_params,
                                 const int32_t* first_pos, int32_t n_thresholds,
                                 const double* thr_unique, const double* h,
                                 const double* scores, int32_t exact_fid, void* workspace,
                                 size_t workspace_bytes, int64_t cand_cap, int64_t exact_cap,
                                 int64_t out_cap, int32_t* out_theta_pos, int32_t* out_tau_pos,
                                 uint32_t* out_n_light, uint32_t* out_n_heavy, double* out_fid,
                                 int64_t* stats, void* stream);

/* numpy-exact mean of where(h > theta | s < tau, cost_heavy, cost_light)
 * (profiler.py:152-153) for n_cells cells: cell c uses score row
 * cell_slot[c], thresholds cell_theta[c] / cell_tau[c] and cost parameters
 * cell_params[c] = {base_l, pen_l, base_h, pen_h}.  out_fid[c] is bitwise
 * equal to float(np.where(...).mean()) on the same float64 inputs. */
int hadis_fid_exact(const double* h, const double* scores, int64_t n, int32_t n_cells,
                    const int32_t* cell_slot, const double* cell_theta, const double* cell_tau,
                    const double* cell_params, double* out_fid, void* stream);

/* ------------------------------------------------------------------------- */
/* Cascade-depth frontier (frontier.py:60-120): every two-stage */
/* (light i < heavy j) and three-stage (light i < middle j < heavy k) point.  */
/* ------------------------------------------------------------------------- */

/* h[n]; scores[M][n] noise-free accept scores (frontier.py:52-57) and
 * model_params[M][3] = {latency_s[1], base cost, hardness penalty}, both in
 * latency order (M <= 16); thr_unique = sorted distinct thresholds (U).
 * Outputs (lat, fid) float64 pairs:
 *   out_two  [M(M-1)/2][U][U][2]         pairs   lexicographic, (theta, tau) ranks
 *   out_three[M(M-1)(M-2)/6][U][U][U][2] triples lexicographic, (theta, tau1, tau2)
 * Latencies are the reference's float expressions bit for bit; fidelities use
 * fixed-point hardness sums (hadis_fid_exact gives numpy-exact two-stage values).
 * bad_records counts hardness outside [0, 1]. */
size_t hadis_cascade_workspace_bytes(int32_t n_models, int32_t n_unique);
int hadis_cascade_points(const double* h, const double* scores, int64_t n, int32_t n_models,
                         const double* model_params, const double* thr_unique, int32_t n_unique,
                         int32_t hfix_shift, double* out_two, double* out_three,
                         uint32_t* bad_records, void* workspace, size_t workspace_bytes,
                         void* stream);

/* ------------------------------------------------------------------------- */
/* Multi-GPU merge of pair-sharded tables (SURVEY §8 e)     */
/* ------------------------------------------------------------------------- */

/* A rank's "slab": int64 header[hdr_words] then the compact rows of
 * hadis_pair_frontiers_compact -- theta_pos, tau_pos (int32[cap]), n_light,
 * n_heavy (uint32[cap]), back to back from byte 8*hdr_words, then fid
 * (float64[cap], from the next 8-byte boundary): 24 bytes per row.  The header
 * holds the frontier's stats array for the rank's local pairs (HADIS_ST_*,
 * per-local-pair row counts at HADIS_ST_PAIR0 + j, the record-validation flag
 * right after them) and a host error word at hdr_words - 1.  The frontier pass
 * writes straight into these columns (no pack step). */
size_t hadis_shard_slab_bytes(int32_t hdr_words, int64_t cap);
size_t hadis_shard_merge_workspace_bytes(int32_t n_pairs);

/* gathered = world slabs back to back (all_gather_into_tensor of the slabs),
 * global pair g owned by rank pair_rank[g] as its local pair pair_local[g];
 * rank r holds rank_npairs[r] pairs; pair_params = the global pairs'
 * hadis_pair_frontiers parameters ([n_pairs][HADIS_PAIR_PARAMS], device), n =
 * the record count.  Writes the canonical table (pairs in global order, rows
 * of a pair in the owner's (theta, tau) order, pair column = global id;
 * r_light, r_heavy, lat rebuilt from n_light / n_heavy bit-identically to
 * hadis_pair_frontiers) and out_stats[5] = {total rows, OR of overflow bits (8
 * = a slab or out_cap overflowed), OR of record flags, OR of host error words,
 * max rows of one rank}.  Rows are copied only when all three status words
 * are 0. */
int hadis_shard_merge(const void* gathered, int32_t world, size_t slab_bytes, int64_t cap,
                      int32_t hdr_words, const int32_t* pair_rank, const int32_t* pair_local,
                      const int32_t* rank_npairs, int32_t n_pairs, const double* pair_params,
                      int64_t n, int64_t out_cap,
                      int32_t* out_pair, int32_t* out_theta_pos, int32_t* out_tau_pos,
                      double* out_r_light, double* out_r_heavy, double* out_fid,
                      double* out_lat, int64_t* out_stats, void* workspace,
                      size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------- */
/* Text -> records: the record prep of profile_config        */
/* (profiler.py:125-132) -- router.hardness (router.py:92-196), seeds          */
/* stable_text_key / _digest / stream_normal (seeds.py:18-55).                 */
/* ------------------------------------------------------------------------- */

#define HADIS_LEX_TABLE 2048          /* open-addressing slots (power of two)   */
#define HADIS_LEX_MAX_WORDS 1024
#define HADIS_LEX_MAX_PHRASES 128
#define HADIS_LEX_MAX_PHRASE_LEN 8
#define HADIS_LEX_POOL 16384
#define HADIS_LEX_MAX_WORD_BYTES 64

enum hadis_lex_flag {                 /* hadis_lexicon.word_flags bits           */
  HADIS_LEX_DETERMINER = 1,           /* noun_markers.txt                        */
  HADIS_LEX_ADJECTIVE = 2,            /* adjectives.txt                          */
  HADIS_LEX_ABSTRACT = 4,             /* abstract_nouns.txt                      */
  HADIS_LEX_ACTION = 8,               /* action_verbs.txt                        */
  HADIS_LEX_FREQ = 16                 /* word_frequency.tsv (rarity[] is valid)  */
};

/* Router lexicons (router.load_lexicons, router.py:64-87) as one flat image,
 * built on the host by paper_2509_00642_b200.text.Lexicon and copied to the
 * device once.  Words are the lowered forms tokens are compared with
 * (router.py:157-172); `table` maps FNV-1a-32(word bytes) & (TABLE-1) by
 * linear probing to a word id (-1 = empty).  rarity[w] is router._rarity(w)
 * (router.py:107-114, evaluated with the host libm at build time).  Spatial
 * phrases (as word ids) are grouped by first word in the reference's scan
 * order (longest first, then lexicographic; router.py:71-76, 134-151). */
typedef struct hadis_lexicon {
  double rarity[HADIS_LEX_MAX_WORDS];
  int32_t n_words, n_phrases, max_phrase_len, max_word_bytes;
  int16_t table[HADIS_LEX_TABLE];
  uint16_t word_off[HADIS_LEX_MAX_WORDS];
  uint16_t phrase_begin[HADIS_LEX_MAX_WORDS];
  uint8_t phrase_count[HADIS_LEX_MAX_WORDS];
  uint8_t word_len[HADIS_LEX_MAX_WORDS];
  uint8_t word_flags[HADIS_LEX_MAX_WORDS];
  uint8_t phrase_len[HADIS_LEX_MAX_PHRASES];
  int16_t phrase_words[HADIS_LEX_MAX_PHRASES][HADIS_LEX_MAX_PHRASE_LEN];
  char pool[HADIS_LEX_POOL];
} hadis_lexicon;

/* sizeof(hadis_lexicon), for bindings that build the image themselves. */
size_t hadis_lexicon_bytes(void);

/* Prompts are UTF-8 byte strings: text i = text_bytes[offsets[i] .. offsets[i+1]).
 *
 * hadis_text_records -- the whole record prep of profile_config:
 *   key[i]   = SHA-256(text)[0:8] big-endian >> 1           (stable_text_key)
 *   order    = stable ascending sort of the keys             (profiler.py:125)
 * and, in that sorted order (out index j <-> input prompt order_out[j]):
 *   key_out[j], h_out[j] = router.hardness(text, weights)    (router.py:192-196)
 *   u1_out[j], u2_out[j] = the two uniforms of stream_normal(seed, key, channel)
 *       (seeds.py:38-46): d = BLAKE2b-128(seed_part | "i" key_be64 "\x1f" |
 *       channel_part); u1 = (d[0:8] + 1.0) / 2^64, u2 = d[8:16] / 2^64.
 *       seed_part / channel_part are the already-packed _digest parts
 *       (seeds.py:18-30, including their "\x1f").
 *   raw_out[j][8] (optional) = router.raw_features in FEATURE_NAMES order.
 * weights: device double[8] (router.check_weights already applied).
 * Box-Muller itself is hadis_keyed_normal_host (libm, see below).
 * The workspace (hadis_text_workspace_bytes) holds the unsorted keys and the
 * radix-sort scratch. */
size_t hadis_text_workspace_bytes(int64_t n_prompts);
int hadis_text_records(const uint8_t* text_bytes, const int64_t* offsets, int64_t n,
                       const hadis_lexicon* lexicon, const double* weights,
                       const uint8_t* seed_part, int32_t seed_len,
                       const uint8_t* channel_part, int32_t channel_len,
                       int64_t* order_out, uint64_t* key_out, double* h_out, double* u1_out,
                       double* u2_out, double* raw_out, void* workspace,
                       size_t workspace_bytes, void* stream);

/* router.raw_features / features / hardness for every prompt in input order
 * (order = NULL) or in the order given (out[j] <-> prompt order[j]); any of
 * h_out / raw_out ([n][8]) / feat_out ([n][8]) may be NULL. */
int hadis_text_features(const uint8_t* text_bytes, const int64_t* offsets, int64_t n,
                        const hadis_lexicon* lexicon, const double* weights,
                        const int64_t* order, double* h_out, double* raw_out, double* feat_out,
                        void* stream);

/* stable_text_key of every prompt (input order). */
int hadis_text_keys(const uint8_t* text_bytes, const int64_t* offsets, int64_t n,
                    uint64_t* key_out, void* stream);

/* HOST pointers.  out[i] = sigma * sqrt(-2.0 * log(u1[i])) * cos(2.0 * pi * u2[i])
 * evaluated left to right with the process's libm -- the same log/cos/sqrt
 * CPython's math module calls in seeds.stream_normal (seeds.py:44-46), so the
 * noise is bit-identical to the reference on the machine it runs on (GPU
 * libdevice log/cos are not the glibc functions).  threads <= 0: all cores. */
int hadis_keyed_normal_host(const double* u1, const double* u2, int64_t n, double sigma,
                            double* out, int32_t threads);

/* ------------------------------------------------------------------------- */
/* Router weight sweep (router.py:199-234)                      */
/* ------------------------------------------------------------------------- */

/* features[n][n_features] (row-major), labels[n] (1 = should bypass to the
 * heavy model), weights[n_vectors][n_features] (normalized grid vectors).
 * Per vector v: scores = features . w (numpy's float64 order on the reference
 * machine), candidate thresholds = midpoints between consecutive distinct
 * scores plus min - 1 and max + 1, predicted hard = score > threshold;
 * out_acc[v] = best balanced accuracy (tp/n_pos + tn/n_neg)/2, out_threshold[v]
 * = its first maximising threshold.  n <= 8192 (HADIS_ERR_UNSUPPORTED above). */
int hadis_tune_weights(const double* features, const uint8_t* labels, int32_t n,
                       int32_t n_features, const double* weights, int32_t n_vectors,
                       int32_t n_pos, double* out_acc, double* out_threshold, void* stream);

/* Generic pareto_prune (catalog.py:171-192) over n (latency, quality) keys:
 * out_idx receives the kept original indices in the reference's output order
 * ((latency, quality, index) ascending); out_count[0] their number.
 * NaN keys are rejected with HADIS_ERR_ARG by the host wrapper. */
size_t hadis_pareto_workspace_bytes(int64_t n);
int hadis_pareto_prune(const double* lat, const double* qual, int64_t n, int64_t* out_idx,
                       int64_t* out_count, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ------------------------------------------------------------------------- */
/* Allocation search: planner.solve over many (demand, SLO) points           */
/* replaces _solve_over_rows / _evaluate_row / fallback_plan                  */
/* (planner.py:81-227).                                                       */
/* ------------------------------------------------------------------------- */

/* Rows: row_model[r][2] = {light model, heavy model} (indices into the model
 * tables; equal for single-model rows), row_share[r][2] = {r_light, r_heavy},
 * row_fid[r] = fidelity_cost.  Models: lat[m][n_batch], mu[m][n_batch]
 * (latency_s / throughput_qps in catalog.batch_sizes order), lat1[m] =
 * latency_s[1].  batch_sizes[n_batch].  Points: lam[p], t_slo[p],
 * workers[p], queues[p][n_models] (0 = no backlog), alpha (shared).
 *
 * Per point the result is written to:
 *   plan_row[p]      chosen row index (-1 = no serveable rows -> PlannerError)
 *   plan_x[p][2]     worker counts {light, heavy} (heavy unused for 1-model rows)
 *   plan_b[p][2]     batch sizes   {light, heavy}
 *   plan_path[p]     path latency (bit-exact with the reference)
 *   plan_flags[p]    bit0 = infeasible (fallback plan), bit1 = negative demand
 * Ties are broken exactly as the reference: per row min (total, path) first
 * combo wins; globally min (fidelity, total, path, row index); fallback max
 * capacity then (latency_s[1] light, latency_s[1] heavy, row index). */
size_t hadis_solve_workspace_bytes(int32_t n_points, int32_t n_rows);
int hadis_solve_many(int32_t n_rows, const int32_t* row_model, const double* row_share,
                     const double* row_fid, int32_t n_models, int32_t n_batch,
                     const int32_t* batch_sizes, const double* lat, const double* mu,
                     const double* lat1, int32_t n_points, const double* lam,
                     const double* t_slo, const int32_t* workers, const double* queues,
                     double alpha, int32_t* plan_row, int32_t* plan_x, int32_t* plan_b,
                     double* plan_path, int32_t* plan_flags, void* workspace,
                     size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HADIS_B200_H */
