/*
 * pact_c.h -- C-ABI of the B200-native PacTrain gradient-sync hot path.
 *
 * This is the drop-in boundary: plain pointers, sizes and opaque handles, no
 * torch or C++ types. Every entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj). The reference has no FFI
 * of its own; its operator API is the C++ free-function API in
 * include/pact/{tensor,sparsity,codec,collective}.hpp, which
 * include/pact_b200.hpp restates on top of this header.
 *
 * Conventions
 *  - Device pointers are CUDA global-memory pointers on the ctx's device.
 *  - Calls taking a `pact_stream_t` are asynchronous on that stream unless
 *    documented otherwise (prune and the collectives synchronise where the
 *    reference semantics need a host decision).
 *  - Status codes 1..15 mirror pact::Errc in declaration order
 *    (include/pact/error.hpp:10-26); 100+ are CUDA/NCCL/argument errors.
 *    No exception crosses this boundary; pact_last_error() gives the message
 *    of the calling thread's last failure.
 *  - Element counts are limited to PACT_MAX_LEN (2^31 - 1 fp32 values, 8 GiB: element
 *    indices travel as 31-bit fields, packed offsets as u32).
 */
#ifndef PACT_C_H
#define PACT_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PACT_ABI_VERSION 1
#define PACT_TILE 1024              /* elements per offset tile (16 words)   */
#define PACT_MAX_LEN ((1ull << 31) - 1)
#define PACT_HEADER_BYTES 26        /* codec.hpp:90 kHeaderSize              */
#define PACT_UNIQUE_ID_BYTES 128    /* NCCL unique id                        */

typedef struct CUstream_st* pact_stream_t; /* == cudaStream_t */
typedef struct pact_ctx pact_ctx;
typedef struct pact_mask pact_mask;
typedef struct pact_comm pact_comm;

typedef enum pact_status {
  PACT_OK = 0,
  PACT_E_DUPLICATE_PARAM = 1, /* Errc::DuplicateParam  */
  PACT_E_INVALID_VIEW = 2,    /* Errc::InvalidView     */
  PACT_E_INVALID_RATIO = 3,   /* Errc::InvalidRatio    */
  PACT_E_INVALID_RATE = 4,    /* Errc::InvalidRate     */
  PACT_E_NUMERICAL = 5,       /* Errc::NumericalFailure*/
  PACT_E_SHAPE_MISMATCH = 6,  /* Errc::ShapeMismatch   */
  PACT_E_MASK_MISMATCH = 7,   /* Errc::MaskMismatch    */
  PACT_E_CORRUPT_PAYLOAD = 8, /* Errc::CorruptPayload  */
  PACT_E_LINK = 9,            /* Errc::LinkError       */
  PACT_E_UNDEFINED_METRIC = 10,
  PACT_E_MISSING_FILE = 11,
  PACT_E_PARSE = 12,
  PACT_E_UNKNOWN_KEY = 13,
  PACT_E_BAD_TOPOLOGY = 14,   /* Errc::BadTopology     */
  PACT_E_RUN_FAILURE = 15,    /* Errc::RunFailure      */
  PACT_E_CUDA = 100,
  PACT_E_NCCL = 101,
  PACT_E_INVALID_ARG = 102,
  PACT_E_NO_DEVICE = 103,
  PACT_E_OOM = 104
} pact_status;

/* collective.hpp:58-64 SyncMode, same order */
typedef enum pact_sync_mode {
  PACT_SYNC_FULL = 0,
  PACT_SYNC_PACKED = 1,
  PACT_SYNC_TERNARY = 2,
  PACT_SYNC_TOPK = 3,
  PACT_SYNC_FP16 = 4
} pact_sync_mode;

/* codec.hpp:80-86 wire::PayloadKind */
typedef enum pact_payload_kind {
  PACT_KIND_FULL = 0,
  PACT_KIND_PACKED = 1,
  PACT_KIND_TERNARY = 2,
  PACT_KIND_FP16 = 3,
  PACT_KIND_TOPK = 4
} pact_payload_kind;

/* codec.hpp:93-98 wire::FrameHeader */
typedef struct pact_frame_header {
  uint8_t kind;
  uint32_t epoch;
  uint64_t mask_digest;
  uint64_t value_count;
} pact_frame_header;

/* sparsity.hpp:37-54 MaskTracker state (plain struct, host-only) */
typedef struct pact_tracker {
  uint32_t threshold;    /* K; 0 is promoted to 1 (sparsity.hpp:41) */
  uint32_t stable_count;
  int has_last;
  uint64_t last_digest;
} pact_tracker;

/* collective.hpp:73-77 SyncStats, plus the device-side breakdown */
typedef struct pact_sync_stats {
  uint64_t bytes_on_wire; /* identical semantics to the reference (analytic) */
  double seconds;         /* measured device time of the sync (not virtual) */
  int mode_used;          /* pact_sync_mode */
  int buckets;            /* packed buckets issued */
  uint64_t value_count;   /* fp32 values allreduced */
  int fallback_reason;    /* 0 none, 1 unstable, 2 vote disagreed, 3 density */
  int transport;          /* exchange used: 0 none (single GPU), 1 NCCL, 2 NVLink P2P */
  double t_pack, t_exchange, t_unpack; /* device seconds per stage (time_stages, single bucket) */
} pact_sync_stats;

/* Adaptive policy knobs. Zero-initialised = reference policy:
 * never fall back on density, one bucket. */
typedef struct pact_policy {
  double density_threshold; /* fall back to dense when agreed nnz/len > this; <=0 or >=1: never */
  uint64_t bucket_bytes;    /* packed bytes per bucket; 0 = auto = one bucket (measured
                               faster than pipelined buckets on B200) */
  float scale;              /* applied in unpack; 0 => 1.0 (SUM, as the reference returns) */
  int time_stages;          /* record CUDA events around the stages */
  int transport;            /* packed exchange: 0 auto (the measured-faster one: P2P for
                               n = 2 up to 1 GiB packed, else NCCL), 1 NCCL allreduce
                               (single bucket on an NCCL symmetric-memory window),
                               2 NVLink P2P (peer-memory reduce in the reference fold
                               order; bit-identical to the reference ring) */
  int wire;                 /* packed exchange payload: PACT_WIRE_F32 (0, the reference's
                               masked_allreduce) or PACT_WIRE_F16 (binary16 ring with
                               per-hop re-rounding, F16Wire collective.cpp:133-163, on the
                               packed values) */
  int gse_dense;            /* the caller's gradient is NOT yet masked: the dense
                               fallback applies enforce_gradient_sparsity first, as the
                               trainer does before aggregating (trainer.cpp:369-372);
                               the packed path needs nothing (unpack writes +0) */
} pact_policy;

/* transport values of pact_policy */
#define PACT_TRANSPORT_AUTO 0
#define PACT_TRANSPORT_NCCL 1
#define PACT_TRANSPORT_P2P 2
/* wire values of pact_policy */
#define PACT_WIRE_F32 0
#define PACT_WIRE_F16 1

typedef struct pact_mask_info {
  uint64_t len;
  uint64_t nnz;
  uint64_t digest;      /* valid iff digest_valid */
  int digest_valid;
  int changed;          /* last prune changed the words vs the previous content */
  uint64_t ntiles;
  uint64_t* words;      /* device, ceil(len/64) u64, tail bits zero */
  uint32_t* tile_off;   /* device, ntiles+1 exclusive prefix of kept counts */
} pact_mask_info;

typedef struct pact_prune_stats {
  uint64_t k;           /* drop count (sparsity.cpp:33-40) */
  uint32_t threshold;   /* k-th smallest |w| key (bits & 0x7fffffff) */
  uint64_t c_lt;        /* #(key < threshold) */
  int path;             /* 0 trivial, 1 sampled window, 2 full radix fallback */
  uint64_t candidates;  /* window candidates compacted */
} pact_prune_stats;

/* ------------------------------------------------------------ diagnostics */
const char* pact_status_name(int status);
const char* pact_last_error(void);
int pact_abi_version(void);

/* ------------------------------------------------ host-side scalar helpers */

/* sparsity.cpp:33-40 drop_count: k = floor(double(ratio)*len + len*1e-7);
 * PACT_E_INVALID_RATIO unless 0 <= ratio < 1. */
pact_status pact_drop_count(float ratio, uint64_t len, uint64_t* k_out);

/* codec.cpp:243-259 encode_header / codec.cpp:261-275 decode_header */
pact_status pact_header_encode(const pact_frame_header* h, uint8_t out[PACT_HEADER_BYTES]);
pact_status pact_header_decode(const uint8_t* frame, size_t len, pact_frame_header* out);

/* sparsity.hpp:40-41 constructor / sparsity.cpp:17-25 MaskTracker::observe.
 * observe returns 1 for Stable, 0 for Unstable. */
void pact_tracker_init(pact_tracker* t, uint32_t threshold);
int pact_tracker_observe(pact_tracker* t, uint64_t digest);
int pact_tracker_status(const pact_tracker* t);

/* collective.cpp:62-67 decide_sync_mode */
int pact_decide_sync_mode(int requested, int tracker_stable);

/* collective.cpp:280-293: unanimity rule over n gathered 26-byte frames.
 * Sets *agree to 1 iff `stable` and every frame is Packed with mine's digest
 * and count. Corrupt frames -> PACT_E_CORRUPT_PAYLOAD. */
pact_status pact_vote_decide(const uint8_t* frames, int n, const pact_frame_header* mine,
                             int stable, int* agree);

/* collective.cpp:75-83, 178-206: bytes ring position `position` of n puts on
 * its link for one ring allreduce of `count` fp32 values; masked adds the
 * (n-1)*26 vote term (collective.cpp:238-242). */
uint64_t pact_ring_bytes(int n, int position, uint64_t count);
uint64_t pact_masked_bytes(int n, int position, uint64_t count);

/* ------------------------------------------------------------------ ctx */
pact_status pact_ctx_create(int device, pact_ctx** out);
pact_status pact_ctx_destroy(pact_ctx* ctx);
/* number of this library's kernels launched through ctx so far */
uint64_t pact_ctx_kernel_launches(const pact_ctx* ctx);

/* ---------------------------------------------------------------- masks
 * tensor.hpp:78-106 SparsityMask, device resident. Words use the reference
 * layout (bit i at words[i>>6] bit i&63, tail bits zero) so a D2H copy of
 * info.words is a valid reference mask. */
pact_status pact_mask_create(pact_ctx* ctx, uint64_t len, pact_mask** out);
pact_status pact_mask_destroy(pact_mask* m);
pact_status pact_mask_info_get(const pact_mask* m, pact_mask_info* out);
/* tensor.cpp:87-95 all_ones / all_zeros */
pact_status pact_mask_fill(pact_mask* m, int keep, pact_stream_t stream);
/* tensor.cpp:97-105 from_bits, from device words (tail bits are cleared);
 * recomputes tile offsets and nnz (synchronises the stream). */
pact_status pact_mask_set_words(pact_mask* m, const uint64_t* words_dev, pact_stream_t stream);
/* tensor.cpp:117-129 refresh(): FNV-1a-64 over the LE word bytes, computed on
 * the GPU (segment-parallel automaton + affine scan); cached until the words
 * change. Synchronises the stream. */
pact_status pact_mask_digest(pact_mask* m, pact_stream_t stream, uint64_t* digest_out);

/* Sub-mask view for a DDP bucket (BucketView/flatten,
 * tensor.hpp:54-74, tensor.cpp:49-79): dst bits [o_s, o_s + seg_len[s]) =
 * src bits [src_begin[s], src_begin[s] + seg_len[s]), o_s = sum of the
 * earlier seg_len. dst->len must equal the sum of seg_len and every segment
 * must lie inside src (else PACT_E_SHAPE_MISMATCH). Host tables; tile
 * offsets, nnz refreshed (synchronises the stream), digest invalidated. */
pact_status pact_mask_gather(const pact_mask* src, uint64_t nseg, const uint64_t* src_begin,
                             const uint64_t* seg_len, pact_mask* dst, pact_stream_t stream);

/* ---------------------------------------------------------------- prune */

/* sparsity.cpp:44-59 magnitude_prune: keep all but the k smallest
 * (|w_i|, i) pairs (global threshold, ties drop the lower index first).
 * Writes words, tile offsets and nnz into `out` (same len as w); the digest
 * is invalidated (computed lazily by pact_mask_digest). `changed` reports
 * whether the words differ from the mask's previous content. Synchronises
 * the stream. stats may be NULL. */
pact_status pact_prune_magnitude(pact_ctx* ctx, const float* w, uint64_t len, float ratio,
                                 pact_mask* out, pact_stream_t stream, pact_prune_stats* stats);

/* Per-layer mode (north_star "per-layer k-th threshold"): the
 * reference rule applied to each [seg[s], seg[s+1]) with
 * k_s = drop_count(ratio, len_s). seg_offsets is a HOST array of nseg+1
 * entries, seg[0]=0, seg[nseg]=len, strictly increasing. */
pact_status pact_prune_magnitude_segmented(pact_ctx* ctx, const float* w, uint64_t len,
                                           const uint64_t* seg_offsets, uint64_t nseg, float ratio,
                                           pact_mask* out, pact_stream_t stream);

/* --------------------------------------------------------------- codecs */

/* sparsity.cpp:112-119 enforce_gradient_sparsity: out[i] = bit ? g[i] : +0.0f.
 * out may alias g. */
pact_status pact_gse(pact_ctx* ctx, const float* g, uint64_t len, const pact_mask* m, float* out,
                     pact_stream_t stream);

/* codec.cpp:14-25 pack: packed[j] = g[idx_j], ascending idx, bit-copied.
 * packed must hold nnz floats. Tile range [tile_begin, tile_end) restricts
 * the work to a bucket (pass 0, UINT64_MAX for all). */
pact_status pact_pack(pact_ctx* ctx, const float* g, uint64_t len, const pact_mask* m,
                      float* packed, uint64_t tile_begin, uint64_t tile_end, pact_stream_t stream);

/* Diagnostic (NVLink counters of the n = 2 push exchange under ncu, one
 * process, no peer flags): pack() into `packed` and, with the same offsets,
 * into `remote` -- memory of another GPU (peer access is enabled here) --
 * with the push kernel the 2-rank exchange uses. No signals, no waits. */
pact_status pact_debug_pack_push(pact_ctx* ctx, const float* g, uint64_t len, const pact_mask* m,
                                 float* packed, float* remote, pact_stream_t stream);

/* codec.cpp:27-38 unpack: PACT_E_MASK_MISMATCH if packed_digest != digest
 * (skipped when check_digest = 0), PACT_E_CORRUPT_PAYLOAD if count != nnz;
 * out[i] = bit ? packed[rank(i)] * scale : +0.0f (scale 1 => bit copy;
 * the multiply is round-to-nearest, trainer.cpp:268-273). */
pact_status pact_unpack(pact_ctx* ctx, const float* packed, uint64_t count, uint64_t packed_digest,
                        int check_digest, const pact_mask* m, float scale, float* out,
                        uint64_t tile_begin, uint64_t tile_end, pact_stream_t stream);

/* Fused unpack + to_mean + masked SGD (trainer.cpp:268-273 and 202-214):
 * g = bit ? packed*scale : 0; w = bit ? w - lr*g : 0.0f (no FMA contraction).
 * grad_out may be NULL. */
pact_status pact_unpack_sgd(pact_ctx* ctx, const float* packed, uint64_t count, const pact_mask* m,
                            float scale, float lr, float* grad_out, float* weights,
                            pact_stream_t stream);

/* Synthetic inputs (integer hashing only so host and
 * device agree bit-for-bit): x[i] = recipe(splitmix64(seed ^ (index_base+i)))
 * * scale. recipe: 0 W-ties, 1 W-real, 2 G-dyadic, 3 G-full. */
pact_status pact_synth_fill(pact_ctx* ctx, float* x, uint64_t len, uint64_t seed,
                            uint64_t index_base, int recipe, float scale, pact_stream_t stream);

/* ---------------------------------------------------------- collectives */

/* NCCL-backed Comm (collective.hpp:89-116): one per GPU/process. The unique
 * id is produced by rank 0 and distributed by the caller. */
pact_status pact_comm_unique_id(uint8_t out[PACT_UNIQUE_ID_BYTES]);
pact_status pact_comm_create(pact_ctx* ctx, const uint8_t id[PACT_UNIQUE_ID_BYTES], int nranks,
                             int rank, pact_comm** out);
pact_status pact_comm_destroy(pact_comm* c);
/* Fail-fast (reference SimCluster::poison + LinkError, collective.cpp:430-458):
 * waits for `stream` with a deadline (timeout_ms <= 0: PACT_LINK_TIMEOUT_MS,
 * default 30 s). A peer that stopped publishing (NVLink flags, the vote
 * board) or an NCCL asynchronous error returns PACT_E_LINK; on the deadline
 * the NCCL communicator is aborted (its kernels exit) and PACT_E_LINK is
 * returned. After a PACT_E_LINK every collective on the comm returns
 * PACT_E_LINK immediately. */
pact_status pact_comm_check(pact_comm* c, pact_stream_t stream, int timeout_ms);
int pact_comm_failed(const pact_comm* c);
int pact_comm_rank(const pact_comm* c);
int pact_comm_size(const pact_comm* c);

/* collective.cpp:165-216 ring_allreduce (SUM, fp32). in may equal out. */
pact_status pact_allreduce_sum(pact_comm* c, const float* in, float* out, uint64_t count,
                               pact_stream_t stream);

/* collective.cpp:93-131, 165-216 ring_allreduce in the reference's exact
 * arithmetic: every element of ChunkMap(count, n) chunk c is folded as
 * ((x_c + x_{c+1}) + ...) + x_{c-1}, so every rank receives bits identical to
 * the reference ring (NCCL's order is unspecified). Runs over NVLink peer
 * memory (one node); the counts are agreed first, PACT_E_SHAPE_MISMATCH on
 * every rank if they differ (the reference's size check);
 * PACT_E_BAD_TOPOLOGY if the ranks cannot map each other's memory. */
pact_status pact_ring_allreduce(pact_comm* c, const float* in, float* out, uint64_t count,
                                pact_stream_t stream);

/* collective.cpp:222-247 allgather of one fixed-size frame per rank (host
 * buffers; frames_out holds n*frame_bytes, indexed by rank). Synchronous. */
pact_status pact_allgather_frames(pact_comm* c, const uint8_t* frame, size_t frame_bytes,
                                  uint8_t* frames_out, pact_stream_t stream);

/* collective.cpp:253-259 full_allreduce (SUM). Synchronous w.r.t. stats. */
pact_status pact_full_allreduce(pact_comm* c, const float* grad, float* out, uint64_t len,
                                float scale, pact_sync_stats* stats, pact_stream_t stream);

/* collective.cpp:269-309 masked_allreduce: vote over 26-byte headers
 * {kind=stable?Packed:Full, epoch, advertised?:digest, nnz}; on a unanimous
 * Packed vote with equal digests and counts (and the density rule of
 * `policy`) pack -> sum-allreduce -> unpack, otherwise a dense
 * sum-allreduce. Returns the SUM (times policy->scale) in out (may alias
 * grad). len must equal the mask length (PACT_E_SHAPE_MISMATCH otherwise,
 * collective.cpp:272). c == NULL runs the single-GPU path (pack -> unpack,
 * no exchange).
 * advertised_digest may be NULL. Blocks the host until the vote decision. */
pact_status pact_masked_allreduce(pact_comm* c, pact_ctx* ctx, const float* grad, uint64_t len,
                                  pact_mask* m, int tracker_stable, uint32_t epoch,
                                  const uint64_t* advertised_digest, const pact_policy* policy,
                                  float* out, pact_sync_stats* stats, pact_stream_t stream);

/* Adaptive dense/sparse policy, measured (north_star (4)): times
 * pact_masked_allreduce's packed path at each probe density (a magnitude
 * mask of synthetic weights at ratio 1 - d) against its dense path, for this
 * communicator and length, max over ranks, and returns the crossover density
 * (linear interpolation between the last winning and first losing probe; 1.0
 * when packing always wins). Feed it to policy->density_threshold. densities
 * may be NULL (a default grid 0.01 .. 0.95); t_packed_out (ndens entries) and
 * t_dense_out may be NULL. Collective (same arguments on every rank);
 * allocates 12 * len bytes of scratch for its duration. c may be NULL (the
 * single-GPU path, where nothing is exchanged). */
pact_status pact_calibrate_density(pact_comm* c, pact_ctx* ctx, uint64_t len, const pact_policy* policy,
                                   const double* densities, int ndens, double* t_packed_out,
                                   double* t_dense_out, double* threshold_out, pact_stream_t stream);

/* Same as pact_masked_allreduce on HOST fp32 buffers: H2D of grad, device
 * sync path, D2H of the result (pinned staging owned by ctx). Synchronous. */
pact_status pact_masked_allreduce_host(pact_comm* c, pact_ctx* ctx, const float* grad_host,
                                       uint64_t len, pact_mask* m, int tracker_stable, uint32_t epoch,
                                       const uint64_t* advertised_digest,
                                       const pact_policy* policy, float* out_host,
                                       pact_sync_stats* stats, pact_stream_t stream);

/* ------------------------------------------------------------ TopK */

/* codec.cpp:148-155: k = max(1, floor(rate*len + len*1e-7)) capped at len;
 * PACT_E_INVALID_RATE unless 0 < rate <= 1. */
pact_status pact_topk_count(uint64_t len, float rate, uint64_t* k_out);

/* codec.cpp:147-172 topk_select: the k largest |g_i| (ties select the lower
 * index), indices strictly increasing, values bit-copied. Selection by the
 * prune kernels (radix-selected threshold, bitmap, tie fix-up). Outputs hold
 * pact_topk_count(len, rate) entries. Synchronises the stream. Inputs are
 * finite (the reference's comparator has no order for NaN). */
pact_status pact_topk_select(pact_ctx* ctx, const float* grad, uint64_t len, float rate,
                             uint32_t* indices, float* values, uint64_t* k_out, pact_stream_t stream);

/* codec.cpp:174-182 topk_densify: zeros, then out[indices[j]] = values[j];
 * PACT_E_CORRUPT_PAYLOAD on an index >= len. Synchronises. */
pact_status pact_topk_densify(pact_ctx* ctx, const uint32_t* indices, const float* values, uint64_t k,
                              uint64_t len, float* out, pact_stream_t stream);

/* collective.cpp:370-390 topk_allgather_aggregate: select, NCCL all-gather
 * of (indices, values), per-element double sum over ranks in rank order,
 * float(acc / n). Returns the MEAN. bytes_on_wire: ring all-gather of the
 * n frames (26 + 8k bytes each). */
pact_status pact_topk_allgather_aggregate(pact_comm* c, pact_ctx* ctx, const float* grad, uint64_t len,
                                          float rate, uint32_t epoch, float* out, pact_sync_stats* stats,
                                          pact_stream_t stream);

/* ------------------------------------------------- binary16 wire */

/* codec.cpp:142-146 fp16_roundtrip with the reference's hand-rolled RNE and
 * clamping (codec.cpp:79-140); out may alias in. */
pact_status pact_fp16_roundtrip(pact_ctx* ctx, const float* in, float* out, uint64_t len,
                                pact_stream_t stream);

/* collective.cpp:261-267 fp16_allreduce: the dense ring with binary16 chunks
 * re-rounded at every hop (F16Wire), bit-identical to ring_allreduce_fp16 on
 * every rank; SUM. comm NULL: the single owner's rounding. */
pact_status pact_fp16_allreduce(pact_comm* c, pact_ctx* ctx, const float* grad, float* out,
                                uint64_t len, pact_sync_stats* stats, pact_stream_t stream);

/* ------------------------------------------- ternary-on-packed */

/* Device sign buffer size for `count` values: 4 * ceil(count / 16) bytes. The
 * first ceil(count / 4) bytes are the reference's sign bytes (codec.hpp:73-78:
 * element i at byte i >> 2, bits 2 (i & 3); 00 = 0, 01 = +1, 10 = -1); the
 * rest are zero. */
uint64_t pact_ternary_sign_bytes(uint64_t count);

/* codec.cpp:50-68 ternarize: *scale_dev = max |v_i| (NaN skipped); element i
 * keeps its sign iff u_i < |v_i| / scale (double), else 0. u_i is the i-th
 * draw of a counter-based SplitMix64 stream of `seed` (the reference's
 * sequential mt19937_64 stream is replaced; see ternary.cu), so results are
 * exact wherever no draw matters (|v_i| in {0, scale}) and unbiased always. */
pact_status pact_ternarize(pact_ctx* ctx, const float* values, uint64_t count, uint64_t seed,
                           float* scale_dev, uint8_t* signs_dev, pact_stream_t stream);

/* codec.cpp:70-75 deternarize with decode_ternary's checks (codec.cpp:324-340:
 * reserved pattern 11, bits past count, negative / non-finite scale, zero
 * scale with non-zero signs -> PACT_E_CORRUPT_PAYLOAD). Synchronises. */
pact_status pact_deternarize(pact_ctx* ctx, const float* scale_dev, const uint8_t* signs_dev,
                             uint64_t count, float* out, pact_stream_t stream);

/* collective.cpp:311-368 ternary_allgather_aggregate: vote (kind Ternary when
 * the tracker is stable), then pack -> ternarize -> NCCL all-gather of
 * (signs, scale) -> per-element double mean over ranks in rank order ->
 * unpack; any disagreement: dense all-reduce then sum / float(n). Returns
 * the MEAN. bytes_on_wire follows the reference's ring all-gather of the
 * frames (+ the ring all-reduce on fallback). Blocks until the decision. */
pact_status pact_ternary_allgather_aggregate(pact_comm* c, pact_ctx* ctx, const float* grad,
                                             uint64_t len, pact_mask* m, int tracker_stable,
                                             uint64_t seed, uint32_t epoch, float* out,
                                             pact_sync_stats* stats, pact_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PACT_C_H */
