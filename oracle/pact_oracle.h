/*
 * pact_oracle.h -- CPU restatement of the PacTrain gradient-sync hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * sm_100a product path in paper_2505_18563_b200/. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. The product path never links, imports or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj); the restatement is pinned against the reference
 * itself (oracle/_ref/libpactref.so, built from the reference sources by
 * oracle/Makefile) and against the reference's own known-answer tests
 * (tests/golden/).
 *
 * Status codes mirror pact::Errc (include/pact/error.hpp:10-26), 1-based in
 * declaration order: 0 = ok.
 */
#ifndef PACT_ORACLE_H
#define PACT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_DUPLICATE_PARAM = 1,
  ORC_INVALID_VIEW = 2,
  ORC_INVALID_RATIO = 3,
  ORC_INVALID_RATE = 4,
  ORC_NUMERICAL_FAILURE = 5,
  ORC_SHAPE_MISMATCH = 6,
  ORC_MASK_MISMATCH = 7,
  ORC_CORRUPT_PAYLOAD = 8,
  ORC_LINK_ERROR = 9,
  ORC_UNDEFINED_METRIC = 10,
  ORC_MISSING_FILE = 11,
  ORC_PARSE_ERROR = 12,
  ORC_UNKNOWN_KEY = 13,
  ORC_BAD_TOPOLOGY = 14,
  ORC_RUN_FAILURE = 15,
};

/* rng.hpp:15-20 */
uint64_t orc_splitmix64(uint64_t x);
/* rng.hpp:24-30 */
uint64_t orc_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c);

/* tensor.cpp:11-19 */
uint64_t orc_fnv1a64(const void* data, size_t len);

/* tensor.cpp:83-129: words = ceil(len/64), bit i at words[i>>6] bit (i&63),
 * tail bits zero; nnz = sum popcount; digest = fnv1a64 over LE word bytes. */
size_t orc_word_count(size_t len);
void orc_mask_from_bytes(const uint8_t* keep, size_t len, uint64_t* words);
uint64_t orc_mask_nnz(const uint64_t* words, size_t len);
uint64_t orc_mask_digest(const uint64_t* words, size_t len);

/* sparsity.cpp:33-40 */
int orc_drop_count(float ratio, uint64_t len, uint64_t* k_out);

/* sparsity.cpp:44-59 (global magnitude prune, stable-sort tie rule).
 * words must hold orc_word_count(len) entries. */
int orc_magnitude_prune(const float* w, size_t len, float ratio, uint64_t* words);

/* Per-layer mode: reference magnitude_prune applied to each
 * segment [seg[s], seg[s+1]) independently; bits written into one global
 * word array. */
int orc_magnitude_prune_segmented(const float* w, size_t len, const uint64_t* seg_offsets,
                                  size_t nseg, float ratio, uint64_t* words);

/* Threshold view of the prune: the k-th smallest key (key = bits & 0x7fffffff)
 * T and c_lt = #(key < T); k = 0 yields T = 0, c_lt = 0 (nothing dropped). */
int orc_prune_threshold(const float* w, size_t len, uint64_t k, uint32_t* T, uint64_t* c_lt);

/* sparsity.cpp:112-119 */
int orc_gse(const float* g, const uint64_t* words, size_t len, float* out);

/* codec.cpp:14-25; returns the value count in *count_out */
int orc_pack(const float* g, const uint64_t* words, size_t len, float* packed, uint64_t* count_out);

/* codec.cpp:27-38: MaskMismatch if digests differ, CorruptPayload if the
 * count differs from nnz. */
int orc_unpack(const float* packed, uint64_t count, uint64_t packed_digest, const uint64_t* words,
               size_t len, float* out);

/* codec.hpp:80-103, codec.cpp:204-275: 26-byte LE frame header */
typedef struct orc_header {
  uint8_t kind;
  uint32_t epoch;
  uint64_t mask_digest;
  uint64_t value_count;
} orc_header;
void orc_encode_header(const orc_header* h, uint8_t out[26]);
int orc_decode_header(const uint8_t* frame, size_t len, orc_header* h);

/* sparsity.cpp:17-25, sparsity.hpp:37-54 */
typedef struct orc_tracker {
  int has_last;
  uint64_t last_digest;
  uint32_t stable_count;
  uint32_t threshold;
} orc_tracker;
void orc_tracker_init(orc_tracker* t, uint32_t threshold);
int orc_tracker_observe(orc_tracker* t, uint64_t digest); /* 1 = Stable */

/* collective.cpp:62-67 (SyncMode enum order collective.hpp:58-64) */
int orc_decide_sync_mode(int requested, int tracker_stable);

/* collective.cpp:93-99, 165-216: sequential restatement of the F32Wire ring.
 * inputs[r] / outputs[r] for r in [0,n), all of length count. The reduced
 * value of chunk c is (((x_c + x_{c+1}) + ...) + x_{c-1}); every output
 * receives the same bits. */
void orc_ring_allreduce(int n, const float* const* inputs, size_t count, float* const* outputs);

/* collective.cpp:75-83, 178-206, 238-242: bytes this position puts on its
 * link for one ring allreduce of `count` fp32 values. */
uint64_t orc_ring_bytes(int n, int position, uint64_t count);

/* collective.cpp:269-309 for all n ranks at once. masks[r] (len bits),
 * digests[r] = true digest of masks[r], advertised[r] = digest rank r
 * announces, nnz[r]. outputs[r]: SUM result. mode_out[r]: 1 = packed,
 * 0 = full. bytes_out[r]: SyncStats.bytes_on_wire. */
int orc_masked_allreduce(int n, const float* const* grads, const uint64_t* const* masks,
                         const uint64_t* digests, const uint64_t* advertised, const int* stable,
                         uint32_t epoch, size_t len, float* const* outputs, int* mode_out,
                         uint64_t* bytes_out);

/* trainer.cpp:268-273 (to_mean) and trainer.cpp:202-214 (sgd_step with mask) */
void orc_to_mean(const float* sum, size_t len, int n, float* mean);
void orc_sgd_step(float* params, const float* mean_grad, size_t len, float lr,
                  const uint64_t* words_or_null);

/* ------------------------------------------------------ TopK (8f-4) */

/* codec.cpp:147-172: k = max(1, floor(rate*len + len*1e-7)) (capped at len);
 * the k largest |g| with ties to the lower index, indices ascending. idx/val
 * hold len entries; *k_out = k. ORC_INVALID_RATE unless 0 < rate <= 1. */
int orc_topk_select(const float* g, size_t len, float rate, uint32_t* idx, float* val, uint64_t* k_out);
/* collective.cpp:383-388: acc over ranks in order (double), mean = float(acc/n) */
int orc_topk_mean(int n, const uint32_t* const* idx, const float* const* val, size_t k, size_t len,
                  float* mean);

/* ------------------------------------------------- binary16 wire (8f-3) */

/* codec.cpp:79-111 / 113-140, element-wise over arrays */
void orc_float_to_half(const float* in, size_t n, uint16_t* out);
void orc_half_to_float(const uint16_t* in, size_t n, float* out);
/* collective.cpp:165-216 with F16Wire (133-163): outputs[r] = the binary16
 * ring's SUM as rank r sees it (identical bits on every rank) */
void orc_ring_allreduce_fp16(int n, const float* const* inputs, size_t len, float* const* outputs);

/* ------------------------------------------------- ternary */

/* codec.cpp:50-68 ternarize with the product's counter-based draws: u_i =
 * (splitmix64(seed + i * 0x9e3779b97f4a7c15) >> 11) * 2^-53 (the i-th output
 * of a SplitMix64 stream seeded with `seed`) instead of the i-th mt19937_64
 * draw. sign_bytes: ceil(n/4) bytes, reference layout (codec.hpp:73-78). */
void orc_ternarize_ctr(const float* v, size_t n, uint64_t seed, float* scale_out,
                       uint8_t* sign_bytes);
/* codec.cpp:320-343 decode checks on (scale, sign bytes, count) */
int orc_ternary_check(float scale, const uint8_t* sign_bytes, size_t count);
/* collective.cpp:355-360: mean[j] = float(sum_r double(scale_r) * sign_r(j) / n),
 * ranks in order */
int orc_ternary_mean(int n, const float* scales, const uint8_t* const* sign_bytes, size_t count,
                     float* mean);

#ifdef __cplusplus
}
#endif

#endif
