/*
 * pact_oracle.c -- CPU restatement of the PacTrain gradient-sync hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see pact_oracle.h). Plain C11, single-threaded,
 * no dependencies. Each function cites the reference function it restates
 * (paths relative to /root/reference/proj).
 */
#include "pact_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */

uint64_t orc_splitmix64(uint64_t x) { /* include/pact/rng.hpp:15-20 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t orc_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:24-30 */
  uint64_t h = orc_splitmix64(base);
  h = orc_splitmix64(h ^ (a + 0x100000001b3ULL));
  h = orc_splitmix64(h ^ (b + 0xcbf29ce484222325ULL));
  h = orc_splitmix64(h ^ c);
  return h;
}

/* ---------------------------------------------------------------- masks */

uint64_t orc_fnv1a64(const void* data, size_t len) { /* src/tensor.cpp:11-19 */
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

size_t orc_word_count(size_t len) { return (len + 63) / 64; } /* tensor.cpp:83 */

void orc_mask_from_bytes(const uint8_t* keep, size_t len, uint64_t* words) { /* tensor.cpp:97-105 */
  memset(words, 0, orc_word_count(len) * sizeof(uint64_t));
  for (size_t i = 0; i < len; ++i)
    if (keep[i]) words[i >> 6] |= (uint64_t)1 << (i & 63);
}

uint64_t orc_mask_nnz(const uint64_t* words, size_t len) { /* tensor.cpp:117-120 */
  uint64_t n = 0;
  size_t nw = orc_word_count(len);
  for (size_t i = 0; i < nw; ++i) n += (uint64_t)__builtin_popcountll(words[i]);
  return n;
}

uint64_t orc_mask_digest(const uint64_t* words, size_t len) { /* tensor.cpp:122-128 */
  /* FNV-1a over the words serialised little-endian, 8 bytes per word */
  uint64_t h = 0xcbf29ce484222325ULL;
  size_t nw = orc_word_count(len);
  for (size_t i = 0; i < nw; ++i) {
    uint64_t w = words[i];
    for (int b = 0; b < 8; ++b) {
      h ^= (w >> (8 * b)) & 0xffu;
      h *= 0x100000001b3ULL;
    }
  }
  return h;
}

static int orc_test(const uint64_t* words, size_t i) { /* tensor.hpp:93 */
  return (int)((words[i >> 6] >> (i & 63)) & 1u);
}

/* ---------------------------------------------------------------- prune */

int orc_drop_count(float ratio, uint64_t len, uint64_t* k_out) { /* src/sparsity.cpp:33-40 */
  if (!(ratio >= 0.0f && ratio < 1.0f)) return ORC_INVALID_RATIO;
  /* identical double expression: floor(double(ratio)*len + len*1e-7) */
  *k_out = (uint64_t)floor((double)ratio * (double)len + (double)len * 1e-7);
  return ORC_OK;
}

/* fabs ordering of finite floats == unsigned ordering of bits & 0x7fffffff */
static uint32_t orc_key(float v) {
  uint32_t b;
  memcpy(&b, &v, 4);
  return b & 0x7fffffffu;
}

/* k-th smallest (0-based position kth) of a distinct-valued u64 array,
 * partially reordering it (quickselect with a deterministic pivot stream). */
static uint64_t orc_select_u64(uint64_t* a, size_t n, size_t kth) {
  size_t lo = 0, hi = n - 1;
  uint64_t rng = 0x243f6a8885a308d3ULL;
  while (lo < hi) {
    rng = orc_splitmix64(rng);
    uint64_t pivot = a[lo + (size_t)(rng % (hi - lo + 1))];
    size_t i = lo, j = hi;
    while (i <= j) {
      while (a[i] < pivot) ++i;
      while (a[j] > pivot) --j;
      if (i <= j) {
        uint64_t t = a[i];
        a[i] = a[j];
        a[j] = t;
        ++i;
        if (j == 0) break;
        --j;
      }
    }
    if (kth <= j)
      hi = j;
    else if (kth >= i)
      lo = i;
    else
      return a[kth];
  }
  return a[kth];
}

/* src/sparsity.cpp:44-59. std::stable_sort by fabs followed by dropping the
 * first k positions is the same as dropping the k smallest (|w_i|, i) pairs;
 * the pair is encoded as the distinct u64 (key << 32 | i) and the k-th
 * smallest is found by selection instead of a full sort. */
static void orc_prune_range(const float* w, size_t begin, size_t len, uint64_t k, uint64_t* comp,
                            uint64_t* words) {
  for (size_t i = 0; i < len; ++i) words[(begin + i) >> 6] |= (uint64_t)1 << ((begin + i) & 63);
  if (k == 0) return;
  for (size_t i = 0; i < len; ++i) comp[i] = ((uint64_t)orc_key(w[begin + i]) << 32) | (uint64_t)i;
  uint64_t cut = orc_select_u64(comp, len, (size_t)(k - 1));
  for (size_t i = 0; i < len; ++i) {
    uint64_t c = ((uint64_t)orc_key(w[begin + i]) << 32) | (uint64_t)i;
    if (c <= cut) words[(begin + i) >> 6] &= ~((uint64_t)1 << ((begin + i) & 63));
  }
}

int orc_magnitude_prune(const float* w, size_t len, float ratio, uint64_t* words) {
  uint64_t k;
  int st = orc_drop_count(ratio, len, &k);
  if (st) return st;
  if (len > 0xffffffffULL) return ORC_SHAPE_MISMATCH;
  memset(words, 0, orc_word_count(len) * sizeof(uint64_t));
  uint64_t* comp = (uint64_t*)malloc((len ? len : 1) * sizeof(uint64_t));
  if (!comp) return ORC_RUN_FAILURE;
  orc_prune_range(w, 0, len, k, comp, words);
  free(comp);
  return ORC_OK;
}

int orc_magnitude_prune_segmented(const float* w, size_t len, const uint64_t* seg, size_t nseg,
                                  float ratio, uint64_t* words) {
  uint64_t k0;
  int st = orc_drop_count(ratio, 0, &k0);
  if (st) return st;
  if (nseg == 0 || seg[0] != 0 || seg[nseg] != len) return ORC_INVALID_VIEW;
  memset(words, 0, orc_word_count(len) * sizeof(uint64_t));
  size_t maxl = 1;
  for (size_t s = 0; s < nseg; ++s) {
    if (seg[s + 1] <= seg[s]) return ORC_INVALID_VIEW; /* tensor.cpp:41 zero-length entry */
    if (seg[s + 1] - seg[s] > maxl) maxl = seg[s + 1] - seg[s];
  }
  uint64_t* comp = (uint64_t*)malloc(maxl * sizeof(uint64_t));
  if (!comp) return ORC_RUN_FAILURE;
  for (size_t s = 0; s < nseg; ++s) {
    uint64_t k;
    orc_drop_count(ratio, seg[s + 1] - seg[s], &k);
    orc_prune_range(w, seg[s], seg[s + 1] - seg[s], k, comp, words);
  }
  free(comp);
  return ORC_OK;
}

int orc_prune_threshold(const float* w, size_t len, uint64_t k, uint32_t* T, uint64_t* c_lt) {
  if (k > len) return ORC_INVALID_RATIO;
  if (k == 0) {
    *T = 0;
    *c_lt = 0;
    return ORC_OK;
  }
  /* radix select over the 31-bit key, digits 11/10/10 */
  static const int shifts[3] = {20, 10, 0};
  static const int widths[3] = {11, 10, 10};
  uint32_t prefix = 0, pmask = 0;
  uint64_t rem = k; /* 1-based rank among elements matching the prefix */
  uint64_t below = 0;
  uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) << 11);
  for (int p = 0; p < 3; ++p) {
    size_t nb = (size_t)1 << widths[p];
    memset(hist, 0, nb * sizeof(uint64_t));
    for (size_t i = 0; i < len; ++i) {
      uint32_t key = orc_key(w[i]);
      if ((key & pmask) == prefix) ++hist[(key >> shifts[p]) & (nb - 1)];
    }
    size_t d = 0;
    while (hist[d] < rem) {
      rem -= hist[d];
      below += hist[d];
      ++d;
    }
    prefix |= (uint32_t)d << shifts[p];
    pmask |= (uint32_t)(nb - 1) << shifts[p];
  }
  free(hist);
  *T = prefix;
  *c_lt = below;
  return ORC_OK;
}

int orc_gse(const float* g, const uint64_t* words, size_t len, float* out) { /* sparsity.cpp:112-119 */
  for (size_t i = 0; i < len; ++i) out[i] = orc_test(words, i) ? g[i] : 0.0f;
  return ORC_OK;
}

/* ---------------------------------------------------------------- codec */

int orc_pack(const float* g, const uint64_t* words, size_t len, float* packed, uint64_t* count_out) {
  /* src/codec.cpp:14-25: kept values, ascending index, bit-copied */
  uint64_t j = 0;
  for (size_t i = 0; i < len; ++i)
    if (orc_test(words, i)) packed[j++] = g[i];
  *count_out = j;
  return ORC_OK;
}

int orc_unpack(const float* packed, uint64_t count, uint64_t packed_digest, const uint64_t* words,
               size_t len, float* out) {
  /* src/codec.cpp:27-38 */
  if (packed_digest != orc_mask_digest(words, len)) return ORC_MASK_MISMATCH;
  if (count != orc_mask_nnz(words, len)) return ORC_CORRUPT_PAYLOAD;
  uint64_t j = 0;
  for (size_t i = 0; i < len; ++i) out[i] = orc_test(words, i) ? packed[j++] : 0.0f;
  return ORC_OK;
}

static void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = (uint8_t)((v >> (8 * i)) & 0xff);
}
static uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

void orc_encode_header(const orc_header* h, uint8_t out[26]) { /* codec.cpp:243-259 (header_bytes, encode_header) */
  out[0] = 'P';
  out[1] = 'A';
  out[2] = 'C';
  out[3] = 'T';
  out[4] = 1; /* kVersion, codec.hpp:91 */
  out[5] = h->kind;
  put_le(out + 6, h->epoch, 4);
  put_le(out + 10, h->mask_digest, 8);
  put_le(out + 18, h->value_count, 8);
}

int orc_decode_header(const uint8_t* f, size_t len, orc_header* h) { /* codec.cpp:261-275 */
  if (len < 26) return ORC_CORRUPT_PAYLOAD;
  if (f[0] != 'P' || f[1] != 'A' || f[2] != 'C' || f[3] != 'T') return ORC_CORRUPT_PAYLOAD;
  if (f[4] != 1) return ORC_CORRUPT_PAYLOAD;
  if (f[5] > 4) return ORC_CORRUPT_PAYLOAD;
  h->kind = f[5];
  h->epoch = (uint32_t)get_le(f + 6, 4);
  h->mask_digest = get_le(f + 10, 8);
  h->value_count = get_le(f + 18, 8);
  return ORC_OK;
}

/* -------------------------------------------------------------- tracker */

void orc_tracker_init(orc_tracker* t, uint32_t threshold) { /* sparsity.hpp:40-41 */
  t->has_last = 0;
  t->last_digest = 0;
  t->stable_count = 0;
  t->threshold = threshold == 0 ? 1 : threshold;
}

int orc_tracker_observe(orc_tracker* t, uint64_t d) { /* sparsity.cpp:17-25 */
  if (t->has_last && t->last_digest == d)
    ++t->stable_count;
  else
    t->stable_count = 0;
  t->has_last = 1;
  t->last_digest = d;
  return t->stable_count >= t->threshold;
}

int orc_decide_sync_mode(int requested, int tracker_stable) { /* collective.cpp:62-67 */
  /* SyncMode: 0 Full, 1 Packed, 2 Ternary, 3 TopK, 4 Fp16 (collective.hpp:58-64) */
  if ((requested == 1 || requested == 2) && !tracker_stable) return 0;
  return requested;
}

/* ----------------------------------------------------------- collective */

static int imod(int a, int n) { return ((a % n) + n) % n; } /* collective.cpp:91 */

typedef struct {
  size_t len, chunk;
} chunkmap; /* collective.cpp:93-99 */
static size_t cm_begin(chunkmap c, int i) {
  size_t b = (size_t)i * c.chunk;
  return b < c.len ? b : c.len;
}
static size_t cm_end(chunkmap c, int i) {
  size_t e = ((size_t)i + 1) * c.chunk;
  return e < c.len ? e : c.len;
}

void orc_ring_allreduce(int n, const float* const* in, size_t count, float* const* out) {
  /* collective.cpp:165-216: reduce-scatter leaves chunk c reduced as
   * ((x_c + x_{c+1}) + ...) + x_{c-1} at position c-1; all-gather copies
   * those bits to every position. */
  chunkmap cm = {count, (count + (size_t)n - 1) / (size_t)n};
  for (int c = 0; c < n; ++c) {
    size_t b = cm_begin(cm, c), e = cm_end(cm, c);
    for (size_t i = b; i < e; ++i) {
      float acc = in[c][i];
      for (int s = 1; s < n; ++s) acc = acc + in[imod(c + s, n)][i];
      for (int r = 0; r < n; ++r) out[r][i] = acc;
    }
  }
}

uint64_t orc_ring_bytes(int n, int p, uint64_t count) {
  /* collective.cpp:178-206 with account_round (75-83): per reduce-scatter
   * step s position p sends chunk p-s, per all-gather step chunk p+1-s. */
  chunkmap cm = {count, (count + (size_t)n - 1) / (size_t)n};
  uint64_t bytes = 0;
  for (int s = 0; s < n - 1; ++s) {
    int c1 = imod(p - s, n), c2 = imod(p + 1 - s, n);
    bytes += 4 * (cm_end(cm, c1) - cm_begin(cm, c1));
    bytes += 4 * (cm_end(cm, c2) - cm_begin(cm, c2));
  }
  return bytes;
}

int orc_masked_allreduce(int n, const float* const* grads, const uint64_t* const* masks,
                         const uint64_t* digests, const uint64_t* advertised, const int* stable,
                         uint32_t epoch, size_t len, float* const* outputs, int* mode_out,
                         uint64_t* bytes_out) {
  /* collective.cpp:269-309 */
  if (n < 2) return ORC_BAD_TOPOLOGY; /* collective.cpp:25 */
  uint8_t* frames = (uint8_t*)malloc((size_t)n * 26);
  orc_header* mine = (orc_header*)malloc((size_t)n * sizeof(orc_header));
  for (int r = 0; r < n; ++r) {
    mine[r].kind = (uint8_t)(stable[r] ? 1 : 0);
    mine[r].epoch = epoch;
    mine[r].mask_digest = advertised ? advertised[r] : digests[r];
    mine[r].value_count = orc_mask_nnz(masks[r], len);
    orc_encode_header(&mine[r], frames + 26 * r);
  }
  /* every rank evaluates the same unanimity rule over the gathered frames */
  int agree0 = -1;
  for (int r = 0; r < n; ++r) {
    int agree = stable[r];
    for (int q = 0; q < n && agree; ++q) {
      orc_header h;
      if (orc_decode_header(frames + 26 * q, 26, &h)) return ORC_CORRUPT_PAYLOAD;
      if (h.kind != 1 || h.mask_digest != mine[r].mask_digest ||
          h.value_count != mine[r].value_count)
        agree = 0;
    }
    if (agree0 < 0) agree0 = agree;
    if (agree != agree0) return ORC_RUN_FAILURE; /* cannot happen: the rule is unanimous */
  }
  if (agree0) {
    uint64_t nnz = mine[0].value_count;
    float** packed = (float**)malloc((size_t)n * sizeof(float*));
    float** summed = (float**)malloc((size_t)n * sizeof(float*));
    for (int r = 0; r < n; ++r) {
      uint64_t cnt;
      packed[r] = (float*)malloc((nnz ? nnz : 1) * sizeof(float));
      summed[r] = (float*)malloc((nnz ? nnz : 1) * sizeof(float));
      orc_pack(grads[r], masks[r], len, packed[r], &cnt);
    }
    orc_ring_allreduce(n, (const float* const*)packed, nnz, summed);
    for (int r = 0; r < n; ++r) {
      orc_unpack(summed[r], nnz, digests[r], masks[r], len, outputs[r]);
      free(packed[r]);
      free(summed[r]);
    }
    free(packed);
    free(summed);
  } else {
    orc_ring_allreduce(n, grads, len, outputs);
  }
  for (int r = 0; r < n; ++r) {
    mode_out[r] = agree0;
    /* allgather of n 26-byte frames: (n-1) rounds of 26 bytes (collective.cpp:238-242) */
    bytes_out[r] = (uint64_t)(n - 1) * 26 + orc_ring_bytes(n, r, agree0 ? mine[0].value_count : len);
  }
  free(frames);
  free(mine);
  return ORC_OK;
}

/* --------------------------------------------------------- caller side */

void orc_to_mean(const float* sum, size_t len, int n, float* mean) { /* trainer.cpp:268-273 */
  const float inv_n = 1.0f / (float)n;
  for (size_t i = 0; i < len; ++i) mean[i] = sum[i] * inv_n;
}

void orc_sgd_step(float* P, const float* g, size_t len, float lr, const uint64_t* words) {
  /* trainer.cpp:202-214; compiled with -ffp-contract=off so lr*g rounds */
  for (size_t i = 0; i < len; ++i) {
    if (words && !orc_test(words, i))
      P[i] = 0.0f;
    else
      P[i] -= lr * g[i];
  }
}

/* ---------------------------------------------------- ternary (8f-2) */

void orc_ternarize_ctr(const float* v, size_t n, uint64_t seed, float* scale_out,
                       uint8_t* sign_bytes) {
  /* codec.cpp:50-68 */
  float s = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    const float a = fabsf(v[i]);
    if (s < a) s = a; /* std::max(s, a): a NaN a leaves s */
  }
  *scale_out = s;
  memset(sign_bytes, 0, (n + 3) / 4);
  if (s == 0.0f) return;
  for (size_t i = 0; i < n; ++i) {
    const double keep_p = (double)fabsf(v[i]) / (double)s;
    /* SplitMix64 stream: state_i = seed + (i + 1) * golden, output = mix(state_i) */
    const double u = (double)(orc_splitmix64(seed + (uint64_t)i * 0x9e3779b97f4a7c15ULL) >> 11) *
                     0x1.0p-53;
    if (u < keep_p) {
      const uint8_t pair = v[i] > 0.0f ? 0x1 : 0x2;
      sign_bytes[i >> 2] |= (uint8_t)(pair << (2 * (i & 3)));
    }
  }
}

static int orc_pair(const uint8_t* b, size_t i) { return (b[i >> 2] >> (2 * (i & 3))) & 3; }

int orc_ternary_check(float scale, const uint8_t* b, size_t count) {
  /* codec.cpp:330-341 */
  if (!(scale >= 0.0f) || isinf(scale)) return ORC_CORRUPT_PAYLOAD;
  const size_t words = (count + 3) / 4;
  for (size_t i = 0; i < count; ++i)
    if (orc_pair(b, i) == 3) return ORC_CORRUPT_PAYLOAD;
  for (size_t i = count; i < words * 4; ++i)
    if (orc_pair(b, i)) return ORC_CORRUPT_PAYLOAD;
  if (scale == 0.0f)
    for (size_t i = 0; i < count; ++i)
      if (orc_pair(b, i)) return ORC_CORRUPT_PAYLOAD;
  return ORC_OK;
}

int orc_ternary_mean(int n, const float* scales, const uint8_t* const* b, size_t count, float* mean) {
  /* collective.cpp:355-360 */
  for (int r = 0; r < n; ++r) {
    const int rc = orc_ternary_check(scales[r], b[r], count);
    if (rc) return rc;
  }
  for (size_t j = 0; j < count; ++j) {
    double acc = 0.0;
    for (int r = 0; r < n; ++r) {
      const int p = orc_pair(b[r], j);
      acc += (double)scales[r] * (double)(p == 1 ? 1 : (p == 2 ? -1 : 0));
    }
    mean[j] = (float)(acc / n);
  }
  return ORC_OK;
}

/* ------------------------------------------------ binary16 wire (8f-3) */

static uint16_t f2h(float v) { /* codec.cpp:79-111 */
  uint32_t bits;
  memcpy(&bits, &v, 4);
  const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
  const int32_t exp = (int32_t)((bits >> 23) & 0xff) - 127;
  uint32_t mant = bits & 0x7fffffu;
  if (exp == 128) return (uint16_t)(sign | (mant != 0 ? 0x7e00u : 0x7bffu));
  if (exp > 15) return (uint16_t)(sign | 0x7bffu);
  if (exp >= -14) {
    uint32_t m = mant >> 13;
    const uint32_t rest = mant & 0x1fffu;
    if (rest > 0x1000u || (rest == 0x1000u && (m & 1u))) ++m;
    const uint32_t h = ((uint32_t)(exp + 15) << 10) + m;
    if (h >= 0x7c00u) return (uint16_t)(sign | 0x7bffu);
    return (uint16_t)(sign | h);
  }
  if (exp >= -25) {
    mant |= 0x800000u;
    const int shift = -exp - 14 + 13;
    uint32_t m = mant >> shift;
    const uint32_t cut = mant & ((1u << shift) - 1u);
    const uint32_t half_ulp = 1u << (shift - 1);
    if (cut > half_ulp || (cut == half_ulp && (m & 1u))) ++m;
    return (uint16_t)(sign | m);
  }
  return sign;
}

static float h2f(uint16_t h) { /* codec.cpp:113-140 */
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1f;
  const uint32_t mant = h & 0x3ffu;
  uint32_t bits;
  if (exp == 0) {
    if (mant == 0) {
      bits = sign;
    } else {
      int e = 1;
      uint32_t m = mant;
      while ((m & 0x400u) == 0) {
        m <<= 1;
        --e;
      }
      bits = sign | ((uint32_t)(e + 112) << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (mant << 13);
  } else {
    bits = sign | ((exp + 112) << 23) | (mant << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

void orc_float_to_half(const float* in, size_t n, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = f2h(in[i]);
}
void orc_half_to_float(const uint16_t* in, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = h2f(in[i]);
}

void orc_ring_allreduce_fp16(int n, const float* const* in, size_t len, float* const* out) {
  /* collective.cpp:165-216 with F16Wire: chunk c starts at position c, every
   * hop sends encode(partial), the receiver adds decode() to its own value,
   * the owner (position c - 1) rounds once more; the all-gather copies. */
  const size_t chunk = (len + (size_t)n - 1) / (size_t)n;
  for (int c = 0; c < n; ++c) {
    const size_t b = (size_t)c * chunk < len ? (size_t)c * chunk : len;
    const size_t e = ((size_t)c + 1) * chunk < len ? ((size_t)c + 1) * chunk : len;
    for (size_t i = b; i < e; ++i) {
      float p = in[c][i];
      for (int k = 1; k < n; ++k) p = in[(c + k) % n][i] + h2f(f2h(p));
      const float fin = h2f(f2h(p));
      for (int r = 0; r < n; ++r) out[r][i] = fin;
    }
  }
}

/* ------------------------------------------------------------ TopK (8f-4) */

typedef struct {
  uint32_t key, idx;
} orc_kv;

static int orc_kv_desc(const void* a, const void* b) {
  /* stable_sort by descending |g| == sort by (key desc, index asc) */
  const orc_kv* x = (const orc_kv*)a;
  const orc_kv* y = (const orc_kv*)b;
  if (x->key != y->key) return x->key > y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int orc_u32_asc(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}

int orc_topk_select(const float* g, size_t len, float rate, uint32_t* idx, float* val, uint64_t* k_out) {
  if (!(rate > 0.0f && rate <= 1.0f)) return ORC_INVALID_RATE; /* codec.cpp:148-149 */
  double kd = floor((double)rate * (double)len + (double)len * 1e-7);
  uint64_t k = kd < 1.0 ? 1 : (uint64_t)kd;
  if (k > len) k = len;
  orc_kv* kv = (orc_kv*)malloc((len ? len : 1) * sizeof(orc_kv));
  if (!kv) return ORC_NUMERICAL_FAILURE;
  for (size_t i = 0; i < len; ++i) {
    uint32_t b;
    memcpy(&b, &g[i], 4);
    kv[i].key = b & 0x7fffffffu; /* fabs order for finite values */
    kv[i].idx = (uint32_t)i;
  }
  qsort(kv, len, sizeof(orc_kv), orc_kv_desc);
  for (uint64_t j = 0; j < k; ++j) idx[j] = kv[j].idx;
  qsort(idx, k, sizeof(uint32_t), orc_u32_asc);
  for (uint64_t j = 0; j < k; ++j) val[j] = g[idx[j]];
  free(kv);
  *k_out = k;
  return ORC_OK;
}

int orc_topk_mean(int n, const uint32_t* const* idx, const float* const* val, size_t k, size_t len,
                  float* mean) {
  double* acc = (double*)calloc(len ? len : 1, sizeof(double));
  if (!acc) return ORC_NUMERICAL_FAILURE;
  for (int r = 0; r < n; ++r)
    for (size_t j = 0; j < k; ++j) {
      if (idx[r][j] >= len) {
        free(acc);
        return ORC_CORRUPT_PAYLOAD;
      }
      acc[idx[r][j]] += val[r][j];
    }
  for (size_t i = 0; i < len; ++i) mean[i] = (float)(acc[i] / n);
  free(acc);
  return ORC_OK;
}
