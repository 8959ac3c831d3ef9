// Text -> records: the record prep of profile_config
// (reference pkg/src/cascadesim/profiler.py:125-132) on the GPU.
//
//   T1 text_keys_kernel     SHA-256 of every prompt -> stable_text_key
//                           (seeds.py:49-55), one thread per prompt.
//   T2 CUB radix sort       (key, prompt index) pairs: the stable key order
//                           `sorted(prompts, key=stable_text_key)` (profiler.py:125).
//   T3 text_records_kernel  one thread per prompt in key order: tokenizer +
//                           lexicon features + hardness (router.py:92-196) and
//                           the BLAKE2b-128 digest of stream_normal's key
//                           (seeds.py:18-46) -> the two uniforms u1, u2.
//
// Exactness: every float64 step is the reference's own operation in its order
// (Python's float division, min/max selection rules, CPython 3.12's
// Neumaier-compensated builtin sum for the rarity mean and the weighted
// feature sum), compiled without FMA contraction.  Lexicon rarities are
// evaluated on the host with the same libm (text.Lexicon).  Box-Muller's
// log/cos are left to the host libm (hadis_keyed_normal_host) because the
// reference's values are glibc's, which libdevice does not reproduce.
//
// The lexicon image (~38 KB) is staged in shared memory once per CTA; the
// Unicode facts the reference's str methods use (split whitespace, isupper,
// lower onto ASCII) come from unicode_tables.inc, generated from the
// interpreter that runs the reference (tools/gen_unicode_tables.py).
#include <cmath>
#include <thread>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"

namespace hadis {

#include "unicode_tables.inc"

constexpr int kTextThreads = 256;

// ------------------------------------------------------------------ UTF-8

__device__ __forceinline__ uint32_t utf8_at(const uint8_t* __restrict__ p, int64_t pos,
                                            int64_t end, int* len) {
  const uint32_t b0 = p[pos];
  if (b0 < 0x80u) { *len = 1; return b0; }
  int n = (b0 >= 0xF0u) ? 4 : (b0 >= 0xE0u) ? 3 : (b0 >= 0xC0u) ? 2 : 1;
  if (pos + n > end) n = 1;                                 // truncated: one byte
  uint32_t cp = n == 4 ? (b0 & 0x07u) : n == 3 ? (b0 & 0x0Fu) : n == 2 ? (b0 & 0x1Fu) : b0;
  for (int k = 1; k < n; ++k) cp = (cp << 6) | (p[pos + k] & 0x3Fu);
  *len = n;
  return cp;
}

__device__ __forceinline__ bool uni_space(uint32_t cp) {     // str.split() separators
  if (cp < 0x80u) return (cp >= 0x09u && cp <= 0x0Du) || (cp >= 0x1Cu && cp <= 0x20u);
  for (int i = 0; i < HADIS_UNI_SPACE_RANGES; ++i)
    if (cp >= kUniSpace[i][0] && cp <= kUniSpace[i][1]) return true;
  return false;
}

__device__ __forceinline__ bool uni_upper(uint32_t cp) {     // str.isupper() of one char
  if (cp < 0x80u) return cp >= 'A' && cp <= 'Z';
  int lo = 0, hi = HADIS_UNI_UPPER_RANGES;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (kUniUpper[mid][1] < cp) lo = mid + 1; else hi = mid;
  }
  return lo < HADIS_UNI_UPPER_RANGES && cp >= kUniUpper[lo][0];
}

// str.lower() of one char when it is a single ASCII char, else -1 (the
// lowered token then contains non-ASCII and matches no ASCII lexicon word)
__device__ __forceinline__ int lower_ascii(uint32_t cp) {
  if (cp < 0x80u) return (cp >= 'A' && cp <= 'Z') ? int(cp + 32u) : int(cp);
  for (int i = 0; i < HADIS_UNI_LOWER_ASCII; ++i)
    if (cp == kUniLowerAscii[i][0]) return int(kUniLowerAscii[i][1]);
  return -1;
}

__device__ __forceinline__ bool is_punct(uint8_t c) {        // router._PUNCT (router.py:37)
  switch (c) {
    case '.': case ',': case ';': case ':': case '!': case '?': case '"': case '\'':
    case '(': case ')': case '[': case ']': case '{': case '}': case '`': return true;
    default: return false;
  }
}

// ------------------------------------------------------------------ SHA-256

__constant__ uint32_t kSha256K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int r) { return __funnelshift_r(x, x, r); }

// first 8 bytes of SHA-256(p[s..e)) as a big-endian integer
__device__ uint64_t sha256_prefix64(const uint8_t* __restrict__ p, int64_t s, int64_t e) {
  uint32_t H[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  const uint64_t L = uint64_t(e - s);
  const uint64_t padded = ((L + 9 + 63) / 64) * 64;
  const uint64_t bits = L * 8;
  for (uint64_t blk = 0; blk < padded; blk += 64) {
    uint32_t W[64];
#pragma unroll
    for (int w = 0; w < 16; ++w) {
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t i = blk + 4 * w + k;
        uint32_t b;
        if (i < L) b = p[s + int64_t(i)];
        else if (i == L) b = 0x80u;
        else if (i >= padded - 8) b = uint32_t(bits >> (8 * (padded - 1 - i))) & 0xFFu;
        else b = 0u;
        v = (v << 8) | b;
      }
      W[w] = v;
    }
#pragma unroll
    for (int t = 16; t < 64; ++t) {
      const uint32_t s0 = rotr32(W[t - 15], 7) ^ rotr32(W[t - 15], 18) ^ (W[t - 15] >> 3);
      const uint32_t s1 = rotr32(W[t - 2], 17) ^ rotr32(W[t - 2], 19) ^ (W[t - 2] >> 10);
      W[t] = W[t - 16] + s0 + W[t - 7] + s1;
    }
    uint32_t a = H[0], b = H[1], c = H[2], d = H[3], f4 = H[4], f5 = H[5], f6 = H[6], f7 = H[7];
#pragma unroll
    for (int t = 0; t < 64; ++t) {
      const uint32_t S1 = rotr32(f4, 6) ^ rotr32(f4, 11) ^ rotr32(f4, 25);
      const uint32_t ch = (f4 & f5) ^ (~f4 & f6);
      const uint32_t t1 = f7 + S1 + ch + kSha256K[t] + W[t];
      const uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
      const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
      const uint32_t t2 = S0 + mj;
      f7 = f6; f6 = f5; f5 = f4; f4 = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += f4; H[5] += f5; H[6] += f6; H[7] += f7;
  }
  return (uint64_t(H[0]) << 32) | H[1];
}

// ------------------------------------------------------------------ BLAKE2b

__constant__ uint64_t kBlakeIV[8] = {
    0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
    0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

__constant__ uint8_t kBlakeSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }

#define HADIS_B2_G(a, b, c, d, x, y)      \
  do {                                     \
    v[a] = v[a] + v[b] + (x);              \
    v[d] = rotr64(v[d] ^ v[a], 32);        \
    v[c] = v[c] + v[d];                    \
    v[b] = rotr64(v[b] ^ v[c], 24);        \
    v[a] = v[a] + v[b] + (y);              \
    v[d] = rotr64(v[d] ^ v[a], 16);        \
    v[c] = v[c] + v[d];                    \
    v[b] = rotr64(v[b] ^ v[c], 63);        \
  } while (0)

__device__ void blake2b_compress(uint64_t h[8], const uint64_t m[16], uint64_t t, bool last) {
  uint64_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[i + 8] = kBlakeIV[i]; }
  v[12] ^= t;                        // messages here are far below 2^64 bytes: t_hi = 0
  if (last) v[14] = ~v[14];
#pragma unroll 1
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kBlakeSigma[r];
    HADIS_B2_G(0, 4, 8, 12, m[s[0]], m[s[1]]);
    HADIS_B2_G(1, 5, 9, 13, m[s[2]], m[s[3]]);
    HADIS_B2_G(2, 6, 10, 14, m[s[4]], m[s[5]]);
    HADIS_B2_G(3, 7, 11, 15, m[s[6]], m[s[7]]);
    HADIS_B2_G(0, 5, 10, 15, m[s[8]], m[s[9]]);
    HADIS_B2_G(1, 6, 11, 12, m[s[10]], m[s[11]]);
    HADIS_B2_G(2, 7, 8, 13, m[s[12]], m[s[13]]);
    HADIS_B2_G(3, 4, 9, 14, m[s[14]], m[s[15]]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// stream_normal's two uniforms (seeds.py:38-46) for key parts
// seed_part | "i" key_be64 "\x1f" | channel_part  (_digest, seeds.py:18-30)
__device__ void keyed_uniforms(const uint8_t* __restrict__ seed_part, int seed_len,
                               uint64_t key, const uint8_t* __restrict__ chan_part, int chan_len,
                               double* u1, double* u2) {
  const int L = seed_len + 10 + chan_len;
  auto byte_at = [&](int i) -> uint64_t {
    if (i < seed_len) return seed_part[i];
    i -= seed_len;
    if (i == 0) return 'i';
    if (i <= 8) return (key >> (8 * (8 - i))) & 0xFFu;
    if (i == 9) return 0x1F;
    return chan_part[i - 10];
  };
  uint64_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = kBlakeIV[i];
  h[0] ^= 0x01010000ull ^ 16ull;                          // fanout 1, depth 1, digest 16 bytes
  const int nblk = L == 0 ? 1 : (L + 127) / 128;
  for (int b = 0; b < nblk; ++b) {
    uint64_t m[16];
    for (int w = 0; w < 16; ++w) {
      uint64_t x = 0;
      for (int k = 7; k >= 0; --k) {
        const int i = b * 128 + w * 8 + k;
        x = (x << 8) | (i < L ? byte_at(i) : 0ull);
      }
      m[w] = x;
    }
    const bool last = b == nblk - 1;
    blake2b_compress(h, m, last ? uint64_t(L) : uint64_t(b + 1) * 128u, last);
  }
  // digest bytes are h[0], h[1] little-endian; int.from_bytes(.., "big")
  const uint64_t d0 = __byte_perm(uint32_t(h[0] >> 32), 0, 0x0123) |
                      (uint64_t(__byte_perm(uint32_t(h[0]), 0, 0x0123)) << 32);
  const uint64_t d1 = __byte_perm(uint32_t(h[1] >> 32), 0, 0x0123) |
                      (uint64_t(__byte_perm(uint32_t(h[1]), 0, 0x0123)) << 32);
  const double two64 = 18446744073709551616.0;           // _TWO64 + 2.0 rounds to 2^64
  *u1 = __ddiv_rn(__dadd_rn(__ull2double_rn(d0), 1.0), two64);
  *u2 = __ddiv_rn(__ull2double_rn(d1), two64);
}

// ------------------------------------------------------------------ features

// CPython 3.12 builtin sum() over floats: Neumaier-compensated (the first
// float enters exactly: 0 + x == x), compensation added once at the end
struct PySum {
  double f = 0.0, c = 0.0;
  bool any = false;
  __device__ __forceinline__ void add(double x) {
    if (!any) { f = x; any = true; return; }
    const double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dadd_rn(f, -t), x));
    else c = __dadd_rn(c, __dadd_rn(__dadd_rn(x, -t), f));
    f = t;
  }
  __device__ __forceinline__ double result() const {
    return (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f;
  }
};

__device__ __forceinline__ bool word_equal(const hadis_lexicon& lex, int w,
                                           const uint8_t* __restrict__ p, int64_t a, int64_t b) {
  const char* s = lex.pool + lex.word_off[w];
  int k = 0;
  for (int64_t pos = a; pos < b;) {
    int l;
    const int c = lower_ascii(utf8_at(p, pos, b, &l));
    if (c != (uint8_t)s[k]) return false;
    ++k;
    pos += l;
  }
  return true;
}

// word id of the lowered token p[a..b) (-1: in no lexicon)
__device__ __forceinline__ int lookup_word(const hadis_lexicon& lex,
                                           const uint8_t* __restrict__ p, int64_t a, int64_t b) {
  uint32_t fnv = 2166136261u;
  int n = 0;
  for (int64_t pos = a; pos < b;) {
    int l;
    const int c = lower_ascii(utf8_at(p, pos, b, &l));
    if (c < 0 || ++n > lex.max_word_bytes) return -1;
    fnv = (fnv ^ uint32_t(c)) * 16777619u;
    pos += l;
  }
  uint32_t slot = fnv & (HADIS_LEX_TABLE - 1);
  for (int probe = 0; probe < HADIS_LEX_TABLE; ++probe) {
    const int w = lex.table[slot];
    if (w < 0) return -1;
    if (lex.word_len[w] == n && word_equal(lex, w, p, a, b)) return w;
    slot = (slot + 1) & (HADIS_LEX_TABLE - 1);
  }
  return -1;
}

struct SpatialScan {                 // router._count_spatial as a streaming scan
  int16_t ring[8];
  int64_t sp = 0;                    // next position to test
  int64_t count = 0;
  __device__ __forceinline__ int64_t step(const hadis_lexicon& lex, int64_t pos, int64_t avail) {
    const int w = ring[pos & 7];
    if (w >= 0) {
      const int beg = lex.phrase_begin[w], cnt = lex.phrase_count[w];
      for (int k = beg; k < beg + cnt; ++k) {
        const int L = lex.phrase_len[k];
        if (pos + L > avail) continue;
        bool ok = true;
        for (int j = 0; j < L; ++j) ok = ok && ring[(pos + j) & 7] == lex.phrase_words[k][j];
        if (ok) { ++count; return pos + L; }
      }
    }
    return pos + 1;
  }
};

// router.raw_features (router.py:154-172) of p[s..e)
__device__ void raw_features(const hadis_lexicon& lex, const uint8_t* __restrict__ p, int64_t s,
                             int64_t e, double raw[8]) {
  const int maxlen = lex.max_phrase_len > 1 ? lex.max_phrase_len : 1;
  int64_t n = 0, objects = 0, adjectives = 0, abstract_ = 0, actions = 0, named = 0;
  bool obj_seek = false;             // after a determiner, skipping adjectives
  bool sentence_start = true;
  PySum rar;
  SpatialScan sc;
  int64_t pos = s;
  while (pos < e) {
    int l;
    if (uni_space(utf8_at(p, pos, e, &l))) { pos += l; continue; }
    const int64_t ts = pos;                                       // raw token [ts, te)
    while (pos < e && !uni_space(utf8_at(p, pos, e, &l))) pos += l;
    const int64_t te = pos;
    int64_t a = ts, b = te;
    while (a < b && is_punct(p[a])) ++a;
    while (b > a && is_punct(p[b - 1])) --b;
    const uint8_t last = p[te - 1];
    const bool ends = last == '.' || last == '!' || last == '?';
    if (a < b) {
      int l0;
      const bool upper = uni_upper(utf8_at(p, a, b, &l0));
      const int w = lookup_word(lex, p, a, b);
      const int fl = w >= 0 ? lex.word_flags[w] : 0;
      rar.add((fl & HADIS_LEX_FREQ) ? lex.rarity[w] : 1.0);
      adjectives += (fl & HADIS_LEX_ADJECTIVE) ? 1 : 0;
      abstract_ += (fl & HADIS_LEX_ABSTRACT) ? 1 : 0;
      actions += (fl & HADIS_LEX_ACTION) ? 1 : 0;
      named += (upper && !sentence_start) ? 1 : 0;
      // _count_objects (router.py:117-131): determiners and adjectives are
      // disjoint (checked when the lexicon is built), so the scan is this
      // two-state machine
      if (fl & HADIS_LEX_DETERMINER) obj_seek = true;
      else if (obj_seek && !(fl & HADIS_LEX_ADJECTIVE)) { ++objects; obj_seek = false; }
      sc.ring[n & 7] = int16_t(w);
      ++n;
      while (sc.sp + maxlen <= n) sc.sp = sc.step(lex, sc.sp, n);
      sentence_start = ends;
    } else if (ends) {
      sentence_start = true;
    }
  }
  while (sc.sp < n) sc.sp = sc.step(lex, sc.sp, n);
  raw[0] = double(n);
  raw[1] = n ? __ddiv_rn(rar.result(), double(n)) : 0.0;
  raw[2] = double(objects);
  raw[3] = double(abstract_);
  raw[4] = __ddiv_rn(double(adjectives), double(objects > 1 ? objects : 1));
  raw[5] = double(sc.count);
  raw[6] = double(actions);
  raw[7] = double(named);
}

__constant__ double kFeatureCaps[8] = {40.0, 1.0, 5.0, 1.0, 1.0, 5.0, 5.0, 5.0};

// features (router.py:175-179) and hardness (router.py:192-196)
__device__ __forceinline__ double hardness_of(const double raw[8], const double w[8],
                                              double feat[8]) {
  PySum acc;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double r = __ddiv_rn(raw[k], kFeatureCaps[k]);
    feat[k] = (1.0 < r) ? 1.0 : r;                          // min(r, 1.0)
    acc.add(__dmul_rn(w[k], feat[k]));
  }
  const double sum = acc.result();
  const double lo = (sum > 0.0) ? sum : 0.0;                // max(0.0, sum)
  return (lo < 1.0) ? lo : 1.0;                             // min(1.0, .)
}

__device__ __forceinline__ void stage_lexicon(hadis_lexicon* dst, const hadis_lexicon* src) {
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = threadIdx.x; i < int(sizeof(hadis_lexicon) / 16); i += blockDim.x) d[i] = s[i];
  __syncthreads();
}

__global__ void __launch_bounds__(kTextThreads)
text_keys_kernel(const uint8_t* __restrict__ p, const int64_t* __restrict__ offs, int64_t n,
                 uint64_t* __restrict__ keys, int64_t* __restrict__ iota) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    keys[i] = sha256_prefix64(p, offs[i], offs[i + 1]) >> 1;
    if (iota) iota[i] = i;
  }
}

__global__ void __launch_bounds__(kTextThreads)
text_records_kernel(const uint8_t* __restrict__ p, const int64_t* __restrict__ offs, int64_t n,
                    const hadis_lexicon* __restrict__ lex_g, const double* __restrict__ weights,
                    const int64_t* __restrict__ order, const uint64_t* __restrict__ keys,
                    const uint8_t* __restrict__ seed_part, int seed_len,
                    const uint8_t* __restrict__ chan_part, int chan_len,
                    double* __restrict__ h_out, double* __restrict__ raw_out,
                    double* __restrict__ feat_out, double* __restrict__ u1_out,
                    double* __restrict__ u2_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  hadis_lexicon& lex = *reinterpret_cast<hadis_lexicon*>(smem);
  stage_lexicon(&lex, lex_g);
  double w[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = weights[k];
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = order ? order[j] : j;
    double raw[8], feat[8];
    raw_features(lex, p, offs[q], offs[q + 1], raw);
    const double h = hardness_of(raw, w, feat);
    if (h_out) h_out[j] = h;
    if (raw_out) {
#pragma unroll
      for (int k = 0; k < 8; ++k) raw_out[j * 8 + k] = raw[k];
    }
    if (feat_out) {
#pragma unroll
      for (int k = 0; k < 8; ++k) feat_out[j * 8 + k] = feat[k];
    }
    if (u1_out) keyed_uniforms(seed_part, seed_len, keys[j], chan_part, chan_len, &u1_out[j],
                               &u2_out[j]);
  }
}

int text_grid(int64_t n) {
  const int64_t want = ceil_div(n, kTextThreads);
  const int64_t cap = int64_t(kNumSMs) * 8;
  return int(want < 1 ? 1 : (want < cap ? want : cap));
}

struct TextWs {
  uint64_t* keys;
  int64_t* iota;
  void* cub;
  size_t cub_bytes;
  size_t total;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

TextWs text_ws_layout(int64_t n, void* base) {
  TextWs w{};
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (const int64_t*)nullptr,
                                  (int64_t*)nullptr, n > 0 ? n : 1, 0, 64);
  unsigned char* b = static_cast<unsigned char*>(base);
  size_t off = 0;
  w.keys = reinterpret_cast<uint64_t*>(b + off);
  off += align256(sizeof(uint64_t) * size_t(n > 0 ? n : 1));
  w.iota = reinterpret_cast<int64_t*>(b + off);
  off += align256(sizeof(int64_t) * size_t(n > 0 ? n : 1));
  w.cub = b + off;
  w.cub_bytes = cub_bytes;
  off += align256(cub_bytes);
  w.total = off;
  return w;
}

}  // namespace hadis

using namespace hadis;

static_assert(sizeof(hadis_lexicon) % 16 == 0, "lexicon image is staged with 16-byte copies");

extern "C" size_t hadis_lexicon_bytes(void) { return sizeof(hadis_lexicon); }

extern "C" size_t hadis_text_workspace_bytes(int64_t n) {
  if (n < 0 || n > (int64_t(1) << 31) - 1) return 0;
  return text_ws_layout(n, nullptr).total;
}

static int text_smem_optin() {
  static int done = 0;
  if (!done) {
    HADIS_CUDA_TRY(hadis_ensure_smem((const void*)text_records_kernel, (size_t)int(sizeof(hadis_lexicon))));
    done = 1;
  }
  return HADIS_OK;
}

extern "C" int hadis_text_keys(const uint8_t* text_bytes, const int64_t* offsets, int64_t n,
                               uint64_t* key_out, void* stream) {
  if (n < 0 || (n > 0 && (!text_bytes || !offsets || !key_out))) return HADIS_ERR_ARG;
  if (n == 0) return HADIS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  text_keys_kernel<<<text_grid(n), kTextThreads, 0, st>>>(text_bytes, offsets, n, key_out,
                                                          nullptr);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}

extern "C" int hadis_text_features(const uint8_t* text_bytes, const int64_t* offsets, int64_t n,
                                   const hadis_lexicon* lexicon, const double* weights,
                                   const int64_t* order, double* h_out, double* raw_out,
                                   double* feat_out, void* stream) {
  if (n < 0 || (n > 0 && (!text_bytes || !offsets || !lexicon || !weights))) return HADIS_ERR_ARG;
  if (n == 0) return HADIS_OK;
  int rc = text_smem_optin();
  if (rc != HADIS_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  text_records_kernel<<<text_grid(n), kTextThreads, sizeof(hadis_lexicon), st>>>(
      text_bytes, offsets, n, lexicon, weights, order, nullptr, nullptr, 0, nullptr, 0, h_out,
      raw_out, feat_out, nullptr, nullptr);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(1);
  return HADIS_OK;
}

extern "C" int hadis_text_records(const uint8_t* text_bytes, const int64_t* offsets, int64_t n,
                                  const hadis_lexicon* lexicon, const double* weights,
                                  const uint8_t* seed_part, int32_t seed_len,
                                  const uint8_t* channel_part, int32_t channel_len,
                                  int64_t* order_out, uint64_t* key_out, double* h_out,
                                  double* u1_out, double* u2_out, double* raw_out,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || n > (int64_t(1) << 31) - 1 || seed_len < 0 || channel_len < 0) return HADIS_ERR_ARG;
  if (n == 0) return HADIS_OK;
  if (!text_bytes || !offsets || !lexicon || !weights || !order_out || !key_out || !h_out ||
      !u1_out || !u2_out || (seed_len && !seed_part) || (channel_len && !channel_part))
    return HADIS_ERR_ARG;
  TextWs ws = text_ws_layout(n, workspace);
  if (!workspace || workspace_bytes < ws.total) return HADIS_ERR_CAPACITY;
  int rc = text_smem_optin();
  if (rc != HADIS_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  text_keys_kernel<<<text_grid(n), kTextThreads, 0, st>>>(text_bytes, offsets, n, ws.keys,
                                                          ws.iota);
  HADIS_LAUNCH_CHECK();
  size_t cub_bytes = ws.cub_bytes;
  HADIS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws.cub, cub_bytes, ws.keys, key_out, ws.iota,
                                                 order_out, n, 0, 64, st));
  text_records_kernel<<<text_grid(n), kTextThreads, sizeof(hadis_lexicon), st>>>(
      text_bytes, offsets, n, lexicon, weights, order_out, key_out, seed_part, seed_len,
      channel_part, channel_len, h_out, raw_out, nullptr, u1_out, u2_out);
  HADIS_LAUNCH_CHECK();
  hadis_count_launches(2);
  return HADIS_OK;
}

// Box-Muller with the process's libm (seeds.py:44-46).  Host code: built by
// the host compiler without -ffast-math / FMA, so each operation is the
// IEEE double operation CPython performs, and log / cos are the same
// glibc entry points CPython's math module resolves.
static void keyed_normal_range(const double* u1, const double* u2, int64_t lo, int64_t hi,
                               double sigma, double* out) {
  const double two_pi = 2.0 * 3.141592653589793;
  for (int64_t i = lo; i < hi; ++i) {
    out[i] = sigma * std::sqrt(-2.0 * std::log(u1[i])) * std::cos(two_pi * u2[i]);
  }
}

extern "C" int hadis_keyed_normal_host(const double* u1, const double* u2, int64_t n,
                                       double sigma, double* out, int32_t threads) {
  if (n < 0 || (n > 0 && (!u1 || !u2 || !out))) return HADIS_ERR_ARG;
  if (n == 0) return HADIS_OK;
  if (sigma == 0.0) {                                   // seeds.py:41-42
    for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
    return HADIS_OK;
  }
  int t = threads > 0 ? threads : int(std::thread::hardware_concurrency());
  if (t < 1) t = 1;
  const int64_t per = int64_t(1) << 16;
  if (int64_t(t) * per > n) t = int((n + per - 1) / per);
  if (t <= 1) {
    keyed_normal_range(u1, u2, 0, n, sigma, out);
    return HADIS_OK;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (n + t - 1) / t;
  for (int k = 0; k < t; ++k) {
    const int64_t lo = k * chunk, hi = lo + chunk < n ? lo + chunk : n;
    if (lo >= hi) break;
    pool.emplace_back(keyed_normal_range, u1, u2, lo, hi, sigma, out);
  }
  for (auto& th : pool) th.join();
  return HADIS_OK;
}
