// launch.h -- host-callable launchers of the sm_100a kernels (internal).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace pactk {

// ---- NVLink P2P exchange types (p2p.cu, codec.cu) ---------------------------
constexpr int kP2PMaxRanks = 8;
constexpr int kP2PPacked = 0, kP2PReduced = 1, kP2PRead = 2;  // flags[kind * 8 + src]
struct P2PView {  // device-visible pointers into every rank's symmetric buffer
  const float* packed[kP2PMaxRanks];   // packed gradient of rank r (current parity)
  const float* reduced[kP2PMaxRanks];  // reduced chunks of rank r, at absolute index
  uint64_t* flags[kP2PMaxRanks];       // flag array of rank r
  int rank, n;
  uint64_t M, C;                       // packed count, ChunkMap chunk = ceil(M/n)
};
// Failure state of the NVLink exchange (device memory). A consumer that
// waits longer than timeout_ns for a peer's flag sets `flag` and the
// host-mapped `*host` (the library reads it before the next call: LinkError),
// and every later consumer skips its peer reads and its own signals, so a
// dead peer fails the step instead of hanging it or folding stale memory.
struct P2PErr {
  int flag;
  int pad;
  volatile int* host;
  unsigned long long timeout_ns;
};
// signals fused into the exchange kernels: `entry` published by block 0 at
// start (the producer ran before on the stream), `exit` by the last CTA to
// finish; kind < 0 = none. counter: a zeroed u32, self-resetting.
struct P2PSig {
  int entry_kind = -1;
  uint64_t entry_val = 0;
  int exit_kind = -1;
  uint64_t exit_val = 0;
  unsigned* counter = nullptr;
  int trace = 0;  // PACT_P2P_TRACE: stamp the push exchange's phases (codec.cu)
};

// ---- codec.cu --------------------------------------------------------------
// PACT_P2P_TRACE diagnostics of the n = 2 push exchange (codec.cu)
void pair_trace_reset(cudaStream_t s);
void pair_trace_read(unsigned long long out[5], cudaStream_t s);
// chunk range [cb, ce) of 1024-element chunks; all pointers device.
// pdl_trigger: let a programmatic dependent (launch_unpack(..., pdl)) start early
// grid_frac > 0: at most that fraction of the persistent grid (bucket
// pipelines leave SMs to the exchange on the other streams)
void launch_pack(const float* g, uint64_t len, const uint64_t* words, const uint32_t* chunk_off,
                 float* packed, uint64_t cb, uint64_t ce, cudaStream_t s, bool pdl_trigger = false,
                 float grid_frac = 0.f);
// pack into `packed` and, with the same offsets, into `remote` (the peer's
// incoming region, NVLink stores); the last CTA publishes sg's exit flag
void launch_pack_push(const float* g, uint64_t len, const uint64_t* words, const uint32_t* chunk_off,
                      float* packed, float* remote, const P2PView& v, const P2PSig& sg, cudaStream_t s);
// pdl: launched as a programmatic dependent of the kernel before it on the
// stream (which must not write words / chunk_off): its CTAs start while the
// predecessor drains and load their first mask words, then wait
// (griddepcontrol.wait) before touching the packed runs
void launch_unpack(const float* packed, uint64_t len, const uint64_t* words,
                   const uint32_t* chunk_off, float scale, int do_scale, float* out, uint64_t cb,
                   uint64_t ce, cudaStream_t s, bool pdl = false, float grid_frac = 0.f);
// unpack with the exchange fused in (NVLink P2P, B == 1): one-shot (n == 2)
// sums the local and the peer's packed runs (waits PACKED); two-shot reads
// each run from its owner's reduced chunk (waits REDUCED; needs C >= 1024).
// Publishes sg's exit flag (READ) when every CTA is done.
void launch_unpack_p2p(const float* packed_local, uint64_t len, const uint64_t* words,
                       const uint32_t* chunk_off, float scale, int do_scale, float* out, const P2PView& v,
                       int two_shot, const uint64_t* flags, uint64_t target, P2PErr* err, const P2PSig& sg,
                       cudaStream_t s);
void launch_unpack_sgd(const float* packed, uint64_t len, const uint64_t* words,
                       const uint32_t* chunk_off, float scale, int do_scale, float lr,
                       float* grad_out, float* weights, cudaStream_t s);
void launch_scale(const float* in, float* out, uint64_t len, float scale, cudaStream_t s);
void launch_gse(const float* g, uint64_t len, const uint64_t* words, float* out, cudaStream_t s);
void launch_mask_fill(uint64_t* words, uint64_t len, int keep, uint32_t* chunk_off, cudaStream_t s);
void launch_clear_tail(uint64_t* words, uint64_t len, cudaStream_t s);
void launch_tile_popc(const uint64_t* words, uint64_t len, uint32_t* chunk_popc, cudaStream_t s);
// *flag |= 1 when the two word arrays differ (nwords rounded up to pairs)
void launch_words_differ(const uint64_t* a, const uint64_t* b, uint64_t nwords, int* flag, cudaStream_t s);
// out[j] = src[idx[j]] for j < n (n <= kGatherMax): a few chunk offsets for
// the host in one readback (bucket boundaries of the copy-engine exchange)
constexpr int kGatherMax = 65;
struct GatherIdx {
  uint64_t i[kGatherMax];
  int n;
};
void launch_gather_u32(const uint32_t* src, const GatherIdx& idx, uint32_t* out, cudaStream_t s);
// dst bits [dst_start[s], dst_start[s+1]) <- src bits from src_begin[s]
// (device tables, nseg entries + 1 for dst_start); all dst_words_padded
// words are written (zero past dst_len)
void launch_mask_gather(const uint64_t* src, uint64_t src_len, const uint64_t* src_begin,
                        const uint64_t* dst_start, uint64_t nseg, uint64_t* dst, uint64_t dst_len,
                        uint64_t dst_words_padded, cudaStream_t s);
// exclusive scan of n u32 -> out[0..n], out[n] = total (single pass, look-back)
size_t scan_scratch_bytes(uint64_t n);
void launch_scan_excl(const uint32_t* in, uint64_t n, uint32_t* out, void* scratch, cudaStream_t s);
// count of kernels launched by these launchers (process-wide, for gpu_launches)
uint64_t launches();
void note_launch(uint64_t n = 1);

// ---- p2p.cu ----------------------------------------------------------------
// flags[kind][rank] = value on every rank (system-scope release after a fence)
void launch_p2p_signal(const P2PView& v, int kind, uint64_t value, cudaStream_t s);
// wait until flags[kind][s] >= target for all s < n (timeout -> *err)
void launch_p2p_wait(const uint64_t* flags, int kind, int n, uint64_t target, P2PErr* err,
                     cudaStream_t s);
// fold packed[*][b, e) in the reference order into out[b, e) (waits PACKED);
// max_ctas > 0 caps the grid (overlap with pack/unpack on other streams)
void launch_p2p_fold(const P2PView& v, float* out, uint64_t b, uint64_t e, const uint64_t* flags,
                     uint64_t target, P2PErr* err, int max_ctas, const P2PSig& sg, cudaStream_t s);
// out[j] = reduced[(j - P0) / Cb][j] for j in [b, e) (waits REDUCED)
void launch_p2p_gather(const P2PView& v, float* out, uint64_t b, uint64_t e, uint64_t P0, uint64_t Cb,
                       const uint64_t* flags, uint64_t target, P2PErr* err, int max_ctas,
                       const P2PSig& sg, cudaStream_t s);

// ---- prune.cu --------------------------------------------------------------
struct PruneWindow {
  uint32_t lo, hi;
};
struct PruneCounts {  // device-side accumulators (zeroed by the launcher)
  unsigned long long n_lt, n_eq_lo, n_eq_hi, n_mid;
};
struct BitmapCounts {  // zeroed by launch_prune_bitmap
  unsigned long long n_lt, n_eq;
  int changed, tie_mismatch;     // changed: a word bit outside the candidates
  unsigned long long n_cand_below;  // candidates with key < T (#(key < lo) = n_lt - this)
  unsigned long long n_cand;     // window candidates seen (may exceed cand.cap)
  int changed_cand, fix_changed;  // a candidate bit changed (bitmap pass / after a fix-up)
  int changed_tie, pad;           // a tie bit changed (before any tie fix-up)
};
// Window candidates of the bitmap pass (temporal reuse, prune.cu): elements
// with lo <= key <= hi and key != T are compacted as key[j], idx[j] | (the
// element's PREVIOUS mask bit << 31). lo > hi disables the window.
struct PruneCandBuf {
  uint32_t lo = 1, hi = 0;
  uint32_t* key = nullptr;
  uint32_t* idx = nullptr;
  uint64_t cap = 0;
  // histogram of the candidates' top digit (key - lo) >> hshift (<= 256
  // bins, zeroed by the launcher): the first radix digit of the moved
  // threshold's select comes for free with the pass
  uint32_t* hist = nullptr;
  int hshift = 0;
};
// 1 CTA: strided sample of keys, sorted; writes the [lo, hi] window.
void launch_prune_sample(const float* w, uint64_t len, uint64_t k, PruneWindow* win_dev,
                         cudaStream_t s);
// full read: counts below/at the window ends, compacts window-interior keys
void launch_prune_count(const float* w, uint64_t len, const PruneWindow* win_dev,
                        PruneCounts* counts_dev, uint32_t* cand, uint64_t cand_cap,
                        cudaStream_t s);
// histogram of digit [shift, shift+nbits) of key' = key - base over elements
// with (key' >> (shift+nbits)) == prefix. src: fp32 weights (from_float) or
// u32 keys. hist (1<<nbits u32) is zeroed by the launcher.
void launch_prune_hist(const void* src, int from_float, uint64_t n, uint32_t base, int shift,
                       int nbits, uint32_t prefix, uint32_t* hist, cudaStream_t s);
// Device-resident radix select: the digit prefix is read from sel->prefix
// (0 on the first pass), and a 1-CTA pick kernel consumes the histogram:
// d = first digit whose inclusive count reaches rem (the host loop of
// select_rank, run on the device), then rem -= counts below d, below += the
// same, prefix = prefix << nbits | d; err = 1 if the histogram holds < rem.
struct SelState {
  uint32_t prefix;
  int err;
  unsigned long long rem, below;
  unsigned long long eq;  // elements in the picked bin (after the last digit: #(key == result))
};
void launch_prune_hist_sel(const void* src, int from_float, uint64_t n, uint32_t base, int shift,
                           int nbits, int first, const SelState* sel, uint32_t* hist, cudaStream_t s);
void launch_prune_pick(const uint32_t* hist, int nbits, int first, uint64_t rank, SelState* sel,
                       cudaStream_t s);
// full read: words (written only where they change) + per-chunk kept counts;
// ties resolved against tie_prefix (per chunk) or all dropped if it is null;
// per-chunk tie counts -> ties_out (compared with ties_prev when given), tie
// bits of chunks with ties -> tie_words; global #(key<T), #(key==T).
void launch_prune_bitmap(const float* w, uint64_t len, uint32_t T, uint64_t r,
                         const uint32_t* tie_prefix, uint64_t* words, uint32_t* chunk_popc,
                         uint32_t* ties_out, const uint32_t* ties_prev, uint64_t* tie_words,
                         BitmapCounts* counts, cudaStream_t s, const PruneCandBuf& cand = PruneCandBuf{},
                         uint64_t* tie_old = nullptr);
// The moved threshold T' of the window path, resolved on the device from
// the select over the candidates (no host round trip before the fix-ups):
// T' = base + the select's value, c_lt' = c_base + #(candidates < T'),
// r' = k - c_lt', straddle = ties at T' split by r'.
struct WinSel {
  uint32_t T1;
  int straddle, err, pad;
  unsigned long long c_lt1, r1, eq1, below;
};
void launch_prune_win_final(const SelState* sel, uint32_t base, int bits, uint64_t ncand, uint64_t c_base,
                            uint64_t k, WinSel* ws, cudaStream_t s);
// one readback for the window path: {ws, *digest, *nnz, *fix_changed} -> out
struct WinReport {
  WinSel w;
  unsigned long long digest;
  uint32_t nnz;
  int fix_changed;
};
// Temporal reuse decided on the device: after the bitmap pass at the
// previous (T0, r0), gate = {changed, ok, digest}: ok when T0 is still the
// k-th key and no tie fix-up is needed (pv: the pass used the previous tie
// prefix -- exact unless r moved or the ties did; else ties all dropped --
// exact when r == #ties), changed when ok and a bit moved, digest when
// changed or force. The gate kernel writes {counts, gate} to `out`; the
// report kernel adds the offsets' total (nnz) and the digest when they ran.
struct HitReport {
  BitmapCounts bc;
  int gate[3], pad;
  unsigned long long digest;
  uint32_t nnz, pad2;
};
void launch_prune_hit_gate(const BitmapCounts* bc, uint64_t k, uint64_t r0, int pv, int force_digest, int* gate,
                           HitReport* out, cudaStream_t s);
void launch_prune_hit_report(const BitmapCounts* bc, const int* gate, const uint64_t* digest, const uint32_t* nnz,
                             HitReport* out, cudaStream_t s);
void launch_prune_win_report(const WinSel* ws, const uint64_t* digest, const uint32_t* nnz,
                             const int* fix_changed, WinReport* out, cudaStream_t s);
// Window fix-up once the true threshold T' of a moved mask is known (it lies
// in the window, T' != the pass's T): every candidate gets key > T' (ties at
// T' provisionally dropped; with `straddle` their bits go to tie_words and
// per-chunk counts to ties for the tie fix-up); words by 64-bit atomics,
// chunk_popc adjusted by the flips. tie_clear first zeroes the tie words of
// every chunk holding a T'-tie.
void launch_prune_cand_fix(const uint32_t* key, const uint32_t* idx, uint64_t n, const WinSel* ws,
                           uint64_t* words, uint32_t* chunk_popc, uint64_t* tie_words, uint32_t* ties,
                           int* changed, cudaStream_t s);
void launch_prune_cand_tieclear(const uint32_t* key, const uint32_t* idx, uint64_t n, const WinSel* ws,
                                uint64_t* tie_words, cudaStream_t s);
// *flag = 1 if a tie candidate's (key == T') final bit differs from its
// recorded previous bit (the fix-up checks the others into the same flag)
void launch_prune_cand_changed(const uint32_t* key, const uint32_t* idx, uint64_t n, const WinSel* ws,
                               const uint64_t* words, int* flag, cudaStream_t s);
// exact tie bits from the exact tie prefix; updates chunk_popc of tie chunks.
// Ties of global rank < r dropped (prune) or, keep_low, kept (TopK)
// tie_old (optional, the bitmap pass's previous tie bits): *changed = 1 if a
// tie bit ends different from it
// ws (optional): r = ws->r1, and nothing to do unless ws->straddle
void launch_prune_tiefix(uint64_t* words, uint64_t len, const uint64_t* tie_words,
                         const uint32_t* ties, const uint32_t* tie_prefix, uint64_t r,
                         uint32_t* chunk_popc, cudaStream_t s, int keep_low = 0,
                         const uint64_t* tie_old = nullptr, int* changed = nullptr,
                         const WinSel* ws = nullptr);
// TopK payload: the ascending indices of the set bits (u32), chunk offsets given
void launch_pack_index(uint64_t len, const uint64_t* words, const uint32_t* chunk_off,
                       uint32_t* idx, cudaStream_t s);
// acc[idx[j]] += double(val[j]) (unique idx per call); err |= 1 on idx >= len

// out[i] = float(acc[i] / n)
// sparse TopK accumulator: union bitmap of all ranks' indices, per-slot
// double sums (rank order = launch order), slot means -> packed for unpack
void launch_union_bits(const uint32_t* idx, uint64_t k, uint64_t len, uint64_t* words, int* err, cudaStream_t s);
void launch_scatter_add_slot(const uint32_t* idx, const float* val, uint64_t k, uint64_t len, const uint64_t* words,
                             const uint32_t* off, double* acc, cudaStream_t s);
void launch_slot_mean(const double* acc, const uint32_t* total, uint64_t max_slots, int n, float* packed,
                      cudaStream_t s);

// out[idx[j]] = val[j] over a zero-filled out; err |= 1 on idx >= len
void launch_scatter_f32(const uint32_t* idx, const float* val, uint64_t k, uint64_t len, float* out,
                        int* err, cudaStream_t s);

// ---- prune_seg.cu (per-layer mode, every layer at once) ---------------------
struct SegInfo {  // host-filled, one per layer [begin, end)
  unsigned long long begin, end, k;       // element range, drop count
  unsigned long long cand_off, cand_cap;  // the layer's window-candidate region
  int trivial;                            // 0 select, 1 keep all, 2 drop all
  int pad;
};
struct SegState {  // device-filled (the host seeds trivial layers)
  uint32_t lo, hi;  // sampled window of the k-th key
  uint32_t T;       // the layer's threshold key
  int mode;         // 0 resolved, 1 window missed (the host selects exactly)
  unsigned long long n_lt, n_eq_lo, n_eq_hi;  // counting pass
  unsigned long long c_lt, r;                 // #(key < T), ties dropped
  unsigned long long tie_base;                // ties before the layer's first element
  unsigned long long b_lt, b_eq;              // bitmap pass: #(key < T), #(key == T)
};
struct SegTile {  // a <= 64 Ki-element range inside one layer
  uint32_t seg, pad;
  unsigned long long begin, end;
};
void launch_seg_sample(const float* w, const SegInfo* info, SegState* st, uint32_t nseg, cudaStream_t s);
void launch_seg_count(const float* w, const SegInfo* info, SegState* st, const SegTile* tiles, uint32_t ntiles,
                      uint32_t* cand, unsigned long long* fill, cudaStream_t s);
void launch_seg_select(const SegInfo* info, SegState* st, uint32_t nseg, const uint32_t* cand,
                       const unsigned long long* fill, cudaStream_t s);
// words (ties provisionally dropped), tie words of chunks with ties,
// per-chunk tie counts and kept counts, per-layer b_lt / b_eq
void launch_seg_bitmap(const float* w, uint64_t len, const SegInfo* info, SegState* st, const uint32_t* chunk_seg,
                       uint64_t* words, uint64_t* tie_words, uint32_t* ties, uint32_t* chunk_popc, cudaStream_t s);
// per-layer temporal reuse: after a bitmap pass at the previous thresholds,
// every non-trivial layer whose T is still its k-th key (b_lt < k <= b_lt +
// b_eq) takes c_lt = b_lt, r = k - b_lt; any other sets *miss
void launch_seg_verify(const SegInfo* info, SegState* st, uint32_t nseg, int* miss, cudaStream_t s);
void launch_seg_tiebase(const SegInfo* info, SegState* st, uint32_t nseg, const uint64_t* tie_words,
                        const uint32_t* ties, const uint32_t* tie_prefix, cudaStream_t s);
void launch_seg_tiefix(uint64_t len, const SegInfo* info, const SegState* st, const uint32_t* chunk_seg,
                       uint64_t* words, const uint64_t* tie_words, const uint32_t* ties, const uint32_t* tie_prefix,
                       uint32_t* chunk_popc, cudaStream_t s);

// ---- ternary.cu -------------------------------------------------------------
// x[i] = x[i] / d (IEEE division; the gather paths' `sum / float(n)`)
void launch_div(float* x, uint64_t n, float d, cudaStream_t s);
// *out_bits = bits of max |v_i| over non-NaN v (0 for n = 0)
void launch_absmax(const float* v, uint64_t n, unsigned* out_bits, cudaStream_t s);
// signs[ceil(n/16)] u32: element i keeps sign(v_i) iff u_i < |v_i| / max,
// u_i the i-th SplitMix64 draw of `seed`
void launch_ternarize(const float* v, uint64_t n, const unsigned* smax_bits, uint64_t seed,
                      uint32_t* signs, cudaStream_t s);
// out[i] = float(sum_r double(scales[r*scale_stride]) * sign_r(i) / n), sign
// words of rank r at signs + r*sign_stride; decode errors OR-ed into *err
void launch_ternary_mean(const uint32_t* signs, uint64_t sign_stride, const float* scales,
                         uint64_t scale_stride, int n, uint64_t count, float* out, int* err,
                         cudaStream_t s);

// ---- f16wire.cu (reference binary16 conversions, codec.cpp:77-146) --------
void launch_f16_encode(const float* x, uint64_t n, uint16_t* out, cudaStream_t s);
// out[i] = encode(x[i] + decode(recv[i]))
void launch_f16_step(const float* x, const uint16_t* recv, uint64_t n, uint16_t* out, cudaStream_t s);
// out[j] = decode(gathered[((j / C) + n - 1) % n][j % C]) for j < count
void launch_f16_gather(const uint16_t* gathered, uint64_t count, int n, uint64_t C, float* out,
                       cudaStream_t s);
void launch_f16_roundtrip(const float* x, uint64_t n, float* out, cudaStream_t s);

// ---- digest.cu -------------------------------------------------------------
// FNV-1a-64 over the LE bytes of nwords words; scratch sized by
// digest_scratch_bytes(nwords). Result written to *out_dev.
size_t digest_scratch_bytes(uint64_t nwords);
void launch_digest(const uint64_t* words, uint64_t nwords, void* scratch, uint64_t* out_dev,
                   cudaStream_t s);

// ---- synth.cu --------------------------------------------------------------
void launch_synth(float* x, uint64_t len, uint64_t seed, uint64_t index_base, int recipe,
                  float scale, cudaStream_t s);

}  // namespace pactk
