// prune.cu -- global magnitude pruning (reference: sparsity.cpp:33-59).
//
// The reference stable-sorts an index array by |w| and drops the first k
// positions: the k smallest (|w_i|, i) pairs, ties at the threshold dropped
// lowest-index first. With key = bits(w) & 0x7fffffff (monotone in |w| for
// finite values, +0/-0 tie) that is exactly:
//
//   T = k-th smallest key,  c_lt = #(key < T),  r = k - c_lt  (1 <= r <= E)
//   bit_i = key_i > T  ||  (key_i == T  &&  tierank_i >= r)
//
// with E = #(key == T) and tierank_i = #{j < i : key_j == T}.
//
// Kernels (one warp owns one 1024-element chunk; persistent grids):
//   prune_sample   1 CTA: 16384 strided keys, register bitonic sort, a
//                  +-6 sigma window [lo, hi] around the k-th key's rank.
//   prune_count    full read: #(key<lo), #(key==lo), #(key==hi); keys strictly
//                  inside the window go to a small candidate buffer.
//   prune_hist     radix-select digits over the candidates (L2 resident) or,
//                  if the window missed, over the whole array.
//   prune_bitmap   full read: mask words with ties resolved against a given
//                  per-chunk tie prefix (or all ties dropped when r == E);
//                  records per-chunk tie counts, the tie bits, #(key<T),
//                  #(key==T), and whether any word changed.
//   prune_tiefix   only when ties straddle r: rewrites the tie bits from the
//                  exact prefix (reads the small tie bitmap, never w).
// Temporal reuse (C5 re-pruning): the previous call's (T, c_lt, tie prefix)
// is tried first; the bitmap pass verifies it from its own counts, so an
// unchanged threshold costs ONE read of w. On a miss the full path runs.
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

constexpr int kSample = 16384;
constexpr int kPruneWarps = 8;  // 256-thread CTAs for count / bitmap

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename K>
unsigned persistent_grid(K kernel, int threads, size_t smem, uint64_t work_units, int units_per_cta) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm <= 0) per_sm = 1;
  const uint64_t cap = (uint64_t)num_sms() * per_sm;
  const uint64_t need = (work_units + units_per_cta - 1) / units_per_cta;
  return (unsigned)(need < cap ? (need ? need : 1) : cap);
}

// load lane's 8 float4 slots of chunk c (keys), in-range mask per slot
__device__ __forceinline__ void load_chunk_keys(const float* __restrict__ w, uint64_t len, uint64_t c,
                                                bool vec_ok, uint32_t key[kVecPerLane][4],
                                                uint32_t inr[kVecPerLane]) {
  const int lane = threadIdx.x & 31;
  const uint64_t e0 = c * (uint64_t)kChunk + 4 * lane;
  float4 v[kVecPerLane];
#pragma unroll
  for (int j = 0; j < kVecPerLane; ++j) {
    const uint64_t ge = e0 + 128 * j;
    v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (vec_ok && ge + 4 <= len) {
      v[j] = ld_stream_f4(reinterpret_cast<const float4*>(w + ge));
      inr[j] = 0xF;
    } else {
      inr[j] = 0;
      for (int b = 0; b < 4; ++b)
        if (ge + b < len) {
          (&v[j].x)[b] = w[ge + b];
          inr[j] |= 1u << b;
        }
    }
  }
#pragma unroll
  for (int j = 0; j < kVecPerLane; ++j) {
    key[j][0] = mag_key(v[j].x);
    key[j][1] = mag_key(v[j].y);
    key[j][2] = mag_key(v[j].z);
    key[j][3] = mag_key(v[j].w);
  }
}

// ---------------------------------------------------------------- sample
// 16384 strided keys, 16 per thread in registers; the window ends are two
// order statistics of the sample, found by an in-CTA radix select (11/11/9
// bits: shared-memory histogram, block scan, pick the bucket holding the
// rank) -- no sort. (The first version bitonic-sorted the sample in one CTA:
// 130 us, the largest term of a first-time prune at C2.)
__device__ __forceinline__ uint32_t block1024_excl_scan(uint32_t v, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = scratch[lane];
    scratch[lane] = warp_incl_scan(x) - x;
  }
  __syncthreads();
  const uint32_t r = scratch[warp] + inc - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024, 1)
    prune_sample_kernel(const float* __restrict__ w, uint64_t len, uint64_t k,
                        PruneWindow* __restrict__ win) {
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t scratch[32];
  __shared__ uint32_t sh_prefix, sh_rank;
  const int t = threadIdx.x;
  uint32_t r[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const uint64_t i = (uint64_t)t * 16 + q;
    r[q] = mag_key(w[(i * len + len / 2) / kSample]);
  }
  const double p = (double)k / (double)len;
  const double center = ((double)k - 0.5) / (double)len * kSample;
  const double margin = 6.0 * sqrt(kSample * p * (1.0 - p)) + 8.0;
  const long lo_i = (long)floor(center - margin);
  const long hi_i = (long)ceil(center + margin);
  uint32_t res[2] = {0u, 0x7fffffffu};
  for (int which = 0; which < 2; ++which) {
    const long target = which ? hi_i : lo_i;
    if (which == 0 ? target <= 0 : target >= kSample - 1) continue;  // window open on that side
    uint32_t prefix = 0, pmask = 0, rank = (uint32_t)target;          // rank in the sorted sample
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      const int sh = pass == 0 ? 20 : (pass == 1 ? 9 : 0);
      const uint32_t nb = pass == 2 ? 512u : 2048u;
      hist[t] = 0;
      hist[t + 1024] = 0;
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if ((r[q] & pmask) == prefix) atomicAdd(&hist[(r[q] >> sh) & (nb - 1)], 1u);
      __syncthreads();
      const uint32_t a = hist[2 * t], b2 = hist[2 * t + 1];
      const uint32_t excl = block1024_excl_scan(a + b2, scratch);
      if (rank >= excl && rank < excl + a) {
        sh_prefix = prefix | ((uint32_t)(2 * t) << sh);
        sh_rank = rank - excl;
      } else if (rank >= excl + a && rank < excl + a + b2) {
        sh_prefix = prefix | ((uint32_t)(2 * t + 1) << sh);
        sh_rank = rank - excl - a;
      }
      __syncthreads();
      prefix = sh_prefix;
      rank = sh_rank;
      pmask |= (nb - 1) << sh;
      __syncthreads();
    }
    res[which] = prefix;
  }
  if (t == 0) *win = PruneWindow{res[0], res[1]};
}

// ----------------------------------------------------------------- count
__device__ __forceinline__ void flush_cands(uint32_t* buf, uint32_t fill, PruneCounts* counts,
                                            uint32_t* __restrict__ cand, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&counts->n_mid, (unsigned long long)fill);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (uint32_t i = lane; i < fill; i += 32)
    if (base + i < cap) cand[base + i] = buf[i];
  __syncwarp();
}

__global__ void __launch_bounds__(kPruneWarps * 32)
    prune_count_kernel(const float* __restrict__ w, uint64_t len, const PruneWindow* __restrict__ win,
                       PruneCounts* __restrict__ counts, uint32_t* __restrict__ cand,
                       uint64_t cap, uint64_t nchunks) {
  __shared__ uint32_t cbuf_all[kPruneWarps][kChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* buf = cbuf_all[warp];
  const uint32_t lo = win->lo, hi = win->hi;
  const bool vec_ok = (((uintptr_t)w) & 15) == 0;
  uint32_t c_lt = 0, c_eqlo = 0, c_eqhi = 0, fill = 0;
  const uint64_t nw_total = (uint64_t)gridDim.x * kPruneWarps;
  for (uint64_t c = (uint64_t)blockIdx.x * kPruneWarps + warp; c < nchunks; c += nw_total) {
    uint32_t key[kVecPerLane][4], inr[kVecPerLane];
    load_chunk_keys(w, len, c, vec_ok, key, inr);
    uint32_t nmid = 0;
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const bool in = (inr[j] >> b) & 1;
        const uint32_t kq = key[j][b];
        c_lt += in && kq < lo;
        c_eqlo += in && kq == lo;
        c_eqhi += in && kq == hi && hi != lo;
        nmid += in && kq > lo && kq < hi;
      }
    const uint32_t inc = warp_incl_scan(nmid);
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    if (tot == 0) continue;
    if (fill + tot > kChunk) {
      flush_cands(buf, fill, counts, cand, cap);
      fill = 0;
    }
    uint32_t o = fill + inc - nmid;
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t kq = key[j][b];
        if (((inr[j] >> b) & 1) && kq > lo && kq < hi) buf[o++] = kq;
      }
    __syncwarp();
    fill += tot;
  }
  if (fill) flush_cands(buf, fill, counts, cand, cap);
  c_lt = warp_sum(c_lt);
  c_eqlo = warp_sum(c_eqlo);
  c_eqhi = warp_sum(c_eqhi);
  if (lane == 0) {
    if (c_lt) atomicAdd(&counts->n_lt, (unsigned long long)c_lt);
    if (c_eqlo) atomicAdd(&counts->n_eq_lo, (unsigned long long)c_eqlo);
    if (c_eqhi) atomicAdd(&counts->n_eq_hi, (unsigned long long)c_eqhi);
  }
}

// ------------------------------------------------------------------ hist
template <bool kFloat>
__global__ void __launch_bounds__(256)
    prune_hist_kernel(const void* __restrict__ src, uint64_t n, uint32_t base, int shift, int nbits,
                      uint32_t prefix, uint32_t* __restrict__ ghist, const SelState* __restrict__ sel) {
  extern __shared__ uint32_t sh[];
  if (sel) prefix = sel->prefix;
  const int nb = 1 << nbits;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int hs = shift + nbits;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t raw = kFloat ? mag_key(static_cast<const float*>(src)[i])
                                : static_cast<const uint32_t*>(src)[i];
    const uint32_t key = raw - base;
    if (raw >= base && (uint32_t)((uint64_t)key >> hs) == prefix) {
      const uint32_t d = (key >> shift) & (uint32_t)(nb - 1);
      const unsigned act = __activemask();
      const unsigned peers = __match_any_sync(act, d);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh[d], __popc(peers));
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) atomicAdd(&ghist[b], sh[b]);
}

// 1 CTA of 1024 threads, bins 2t and 2t + 1 per thread (nbits <= 11): block
// exclusive scan of the counts, the one thread whose bins straddle rem
// updates the state. Same digit as select_rank's host loop (first bin whose
// inclusive count >= rem; bin 0 when rem == 0).
__global__ void __launch_bounds__(1024)
    prune_pick_kernel(const uint32_t* __restrict__ hist, int nbits, int first, uint64_t rank,
                      SelState* __restrict__ sel) {
  __shared__ unsigned long long wsum[32], s_total;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nb = 1 << nbits;
  const uint64_t a = 2 * t < nb ? hist[2 * t] : 0u, b = 2 * t + 1 < nb ? hist[2 * t + 1] : 0u;
  const uint64_t rem = first ? rank : sel->rem;
  const uint32_t prefix = first ? 0u : sel->prefix;
  const uint64_t below = first ? 0ull : sel->below;
  uint64_t inc = a + b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint64_t x = wsum[lane], xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    wsum[lane] = xi - x;
    if (lane == 31) s_total = xi;
  }
  __syncthreads();
  const uint64_t e0 = wsum[warp] + inc - (a + b), total = s_total;
  int d = -1;
  uint64_t eb = 0;
  if (rem == 0) {
    if (t == 0) d = 0;
  } else if (e0 < rem && rem <= e0 + a) {
    d = 2 * t;
    eb = e0;
  } else if (e0 + a < rem && rem <= e0 + a + b) {
    d = 2 * t + 1;
    eb = e0 + a;
  }
  if (d >= 0) {
    sel->prefix = (prefix << nbits) | (uint32_t)d;
    sel->rem = rem - eb;
    sel->below = below + eb;
    sel->eq = d == 2 * t ? a : b;
    if (first) sel->err = 0;
  }
  if (t == 0 && total < rem) sel->err = 1;
}

// ---------------------------------------------------------------- bitmap
// Lane-major chunk layout: lane l of the warp classifies the 32 consecutive
// elements [32l, 32l + 32) of its chunk, so its keep / tie bits ARE the
// 32-bit half 'l' of the chunk's 16 mask words (no cross-lane bit gather)
// and in-chunk tie ranks are one warp scan. The chunk is streamed into a
// per-warp cp.async ring with coalesced 16-byte copies; the shared-memory
// layout is XOR-swizzled so each lane's eight LDS.128 of its own 128 bytes
// are conflict-free (unit u of the chunk -> owner u/8, column u%8, stored at
// owner*8 + (column ^ (owner & 7))).
constexpr int kKeyStages = 2;
constexpr int kStageFloats = kChunk + 2 * kChunkWords;  // keys, then the 16 old mask words
constexpr int kCandBuf = 64;                            // per-warp window-candidate staging
constexpr int kCandHistBits = 8;                        // first select digit, counted by the pass
constexpr size_t bitmap_smem(int stages) {
  return (size_t)kPruneWarps * (stages * kStageFloats * sizeof(float) + 2 * kCandBuf * sizeof(uint32_t)) +
         (sizeof(uint32_t) << kCandHistBits) + (size_t)kPruneWarps * stages * sizeof(uint64_t);
}
constexpr size_t kBitmapSmem = bitmap_smem(kKeyStages);

__device__ __forceinline__ void chunk_issue(float* st, const float* __restrict__ w,
                                            const uint64_t* __restrict__ words, uint64_t c) {
  const int lane = threadIdx.x & 31;
  const float* src = w + c * (uint64_t)kChunk + 4 * lane;
#pragma unroll
  for (int j = 0; j < kVecPerLane; ++j) {
    const int u = 32 * j + lane, owner = u >> 3, col = u & 7;
    const uint32_t sa =
        (uint32_t)__cvta_generic_to_shared(st + 4 * (owner * 8 + (col ^ (owner & 7))));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 128 * j) : "memory");
  }
  if (lane < kChunkWords / 2) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st + kChunk + 4 * lane);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                 "l"(words + c * kChunkWords + 2 * lane)
                 : "memory");
  }
}

// Bulk (TMA engine) variant of the chunk load: lane 0 arms the stage's
// mbarrier with the byte count and issues two 1-D cp.async.bulk copies (the
// 4 KiB of weights and the 128 B of old mask words) into a LINEAR stage; the
// lanes wait on the mbarrier's phase. One instruction moves the chunk
// instead of 264 per-lane 16-byte cp.async.
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
}
__device__ __forceinline__ void chunk_issue_bulk(float* stg, uint64_t* mbar, const float* __restrict__ w,
                                                 const uint64_t* __restrict__ words, uint64_t c) {
  const uint32_t sm = (uint32_t)__cvta_generic_to_shared(stg);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the lanes' reads of this stage come first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(kChunk * 4 + kChunkWords * 8)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
               "l"(w + c * (uint64_t)kChunk), "r"(kChunk * 4), "r"(mb)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm + kChunk * 4),
               "l"(words + c * kChunkWords), "r"(kChunkWords * 8), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(mb), "r"(phase)
                 : "memory");
}

// staged window candidates of one warp -> the global list (one atomic per flush)
__device__ __forceinline__ void flush_pairs(const uint32_t* bk, const uint32_t* bi, uint32_t fill,
                                            unsigned long long* n_cand, const PruneCandBuf& cb) {
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(n_cand, (unsigned long long)fill);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (uint32_t i = lane; i < fill; i += 32)
    if (base + i < cb.cap) {
      cb.key[base + i] = bk[i];
      cb.idx[base + i] = bi[i];
    }
  __syncwarp();
}

template <bool kBulk, int kS>
__global__ void __launch_bounds__(kPruneWarps * 32)
    prune_bitmap_kernel(const float* __restrict__ w, uint64_t len, uint32_t T, uint64_t r,
                        const uint32_t* __restrict__ tie_prefix, uint64_t* __restrict__ words,
                        uint64_t nwords, uint32_t* __restrict__ chunk_popc,
                        uint32_t* __restrict__ ties_out, const uint32_t* __restrict__ ties_prev,
                        uint64_t* __restrict__ tie_words, uint64_t* __restrict__ tie_old,
                        BitmapCounts* __restrict__ counts, uint64_t nchunks, PruneCandBuf cb) {
  extern __shared__ __align__(16) float ring_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ring = ring_all + (size_t)warp * kS * kStageFloats;
  uint32_t* cbk = reinterpret_cast<uint32_t*>(ring_all + (size_t)kPruneWarps * kS * kStageFloats) +
                  warp * 2 * kCandBuf;
  uint32_t* cbi = cbk + kCandBuf;
  // CTA histogram of the candidates' top digit (warp-aggregated smem
  // atomics; a window whose lower end is crowded sends most to one bin),
  // added to the global one once at the end
  uint32_t* chist = reinterpret_cast<uint32_t*>(ring_all + (size_t)kPruneWarps * kS * kStageFloats) +
                    kPruneWarps * 2 * kCandBuf;
  if (cb.hist) {
    for (int b = threadIdx.x; b < (1 << kCandHistBits); b += blockDim.x) chist[b] = 0;
    __syncthreads();
  }
  // kBulk: one mbarrier per stage per warp, after the histogram
  uint64_t* mbars = reinterpret_cast<uint64_t*>(chist + (1 << kCandHistBits)) + warp * kS;
  uint32_t phases = 0;  // bit s: parity of stage s's next completion
  if constexpr (kBulk) {
    if (lane == 0) {
      for (int q = 0; q < kS; ++q) mbar_init(mbars + q);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  uint32_t* words32 = reinterpret_cast<uint32_t*>(words);
  uint32_t* tie32 = reinterpret_cast<uint32_t*>(tie_words);
  uint32_t* tie_old32 = reinterpret_cast<uint32_t*>(tie_old);
  const uint64_t nhalves = 2 * nwords;
  const bool vec_ok = (((uintptr_t)w) & 15) == 0;
  // the window always contains T (a disabled window is [T, T]): a lane
  // with no key inside it has no tie either, so its ">= T" mask is its
  // "> T" mask; only lanes touching the window rebuild both exactly
  const bool use_win = cb.lo <= cb.hi && cb.key != nullptr;
  const uint32_t wlo = use_win ? cb.lo : T, W = use_win ? cb.hi - cb.lo : 0u;
  // chunks streamed through the ring: whole 1024-element chunks of an
  // aligned vector (the ragged last chunk is read directly)
  auto full = [&](uint64_t c) { return vec_ok && (c + 1) * (uint64_t)kChunk <= len; };
  uint32_t c_lt = 0, c_eq = 0, c_below = 0, fill = 0;
  int changed = 0, changed_cand = 0, changed_tie = 0, mismatch = 0;
  const uint64_t nw_total = (uint64_t)gridDim.x * kPruneWarps;
  const uint64_t c0 = (uint64_t)blockIdx.x * kPruneWarps + warp;
#pragma unroll
  for (int s = 0; s < kS - 1; ++s) {
    const uint64_t cc = c0 + s * nw_total;
    if constexpr (kBulk) {
      if (lane == 0 && cc < nchunks && full(cc)) chunk_issue_bulk(ring + s * kStageFloats, mbars + s, w, words, cc);
    } else {
      if (cc < nchunks && full(cc)) chunk_issue(ring + s * kStageFloats, w, words, cc);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
  int slot = 0;
  for (uint64_t c = c0; c < nchunks; c += nw_total) {
    const int cur = slot;
    {
      const uint64_t cn = c + (kS - 1) * nw_total;
      const int sn = slot == 0 ? kS - 1 : slot - 1;
      __syncwarp();  // every lane is done reading stage sn (the previous chunk)
      if constexpr (kBulk) {
        if (lane == 0 && cn < nchunks && full(cn)) chunk_issue_bulk(ring + sn * kStageFloats, mbars + sn, w, words, cn);
        if (full(c)) {
          mbar_wait(mbars + cur, (phases >> cur) & 1u);
          phases ^= 1u << cur;
        }
      } else {
        if (cn < nchunks && full(cn)) chunk_issue(ring + sn * kStageFloats, w, words, cn);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(kS - 1) : "memory");
      }
      __syncwarp();  // lanes read stage cells other lanes' copies filled
    }
    const float* st = ring + slot * kStageFloats;
    slot = slot == kS - 1 ? 0 : slot + 1;
    const bool fc = full(c);
    const uint64_t e0 = c * (uint64_t)kChunk + 32 * lane;
    // per element: one compare against T (funnel-shifted sign) and the
    // running minimum of key - lo (unsigned: keys below lo wrap above W)
    uint32_t g = 0, mn = ~0u, inr = ~0u;
    if (fc) {
#pragma unroll
      for (int k = kVecPerLane - 1; k >= 0; --k) {  // elements 32*lane + 4k .. 4k+3
        // kBulk: linear stage, lane l reads its 16-byte cell (k + l) & 7 --
        // conflict-free -- and the rotated mask is turned back below
        const float4 v = kBulk ? *reinterpret_cast<const float4*>(st + 32 * lane + 4 * ((k + lane) & 7))
                               : *reinterpret_cast<const float4*>(st + 4 * (lane * 8 + (k ^ (lane & 7))));
        const uint32_t k3 = mag_key(v.w), k2 = mag_key(v.z), k1 = mag_key(v.y), k0 = mag_key(v.x);
        g = __funnelshift_l(T - k3, g, 1);
        g = __funnelshift_l(T - k2, g, 1);
        g = __funnelshift_l(T - k1, g, 1);
        g = __funnelshift_l(T - k0, g, 1);
        mn = min(mn, min(min(k3 - wlo, k2 - wlo), min(k1 - wlo, k0 - wlo)));
      }
      if constexpr (kBulk) g = __funnelshift_l(g, g, 4 * (lane & 7));  // cell (k + l) & 7 sat at bits 4k
    } else {
      inr = e0 >= len ? 0u : (len - e0 >= 32 ? ~0u : (1u << (len - e0)) - 1u);
      for (int i = 31; i >= 0; --i) {
        const uint32_t kq = e0 + i < len ? mag_key(w[e0 + i]) : 0u;
        g = __funnelshift_l(T - kq, g, 1);
        if (e0 + i < len) mn = min(mn, kq - wlo);
      }
    }
    g &= inr;
    uint32_t e = g, cand = 0;
    const uint64_t hi = c * 32 + lane;  // this lane's 32-bit half of the mask
    const uint32_t old = hi < nhalves ? (fc ? reinterpret_cast<const uint32_t*>(st + kChunk)[lane] : words32[hi]) : 0u;
    {
      // lanes whose keys touch the window, one at a time, by the whole warp:
      // lane j tests element j of lane l, ballots are lane l's exact masks
      uint32_t todo = __ballot_sync(0xffffffffu, mn <= W);
      while (todo) {
        const int l = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint64_t el0 = c * (uint64_t)kChunk + 32 * l;
        bool ok = true;
        uint32_t kq;
        if (fc) {
          kq = mag_key(kBulk ? st[32 * l + lane] : st[4 * (l * 8 + ((lane >> 2) ^ (l & 7))) + (lane & 3)]);
        } else {
          ok = el0 + lane < len;
          kq = ok ? mag_key(w[el0 + lane]) : 0u;
        }
        const uint32_t me = __ballot_sync(0xffffffffu, ok && kq >= T);
        const uint32_t mw = __ballot_sync(0xffffffffu, ok && kq != T && kq - wlo <= W);
        if (lane == l) {
          e = me;
          cand = use_win ? mw : 0u;
        }
        if (!use_win || !mw) continue;
        const uint32_t oldl = __shfl_sync(0xffffffffu, old, l);
        if (lane == 0) c_below += __popc(mw & ~me);  // #(key < lo) = #(key < T) - these
        const uint32_t nm = __popc(mw);
        if (fill + nm > (uint32_t)kCandBuf) {
          flush_pairs(cbk, cbi, fill, &counts->n_cand, cb);
          fill = 0;
        }
        if ((mw >> lane) & 1u) {
          const uint32_t pos = fill + __popc(mw & ((1u << lane) - 1u));
          cbk[pos] = kq;
          cbi[pos] = (uint32_t)(el0 + lane) | (((oldl >> lane) & 1u) << 31);
        }
        if (cb.hist && ((mw >> lane) & 1u)) {
          const uint32_t bin = (kq - wlo) >> cb.hshift;
          const unsigned peers = __match_any_sync(mw, bin);
          if (lane == __ffs(peers) - 1) atomicAdd(&chist[bin], (uint32_t)__popc(peers));
        }
        __syncwarp();
        fill += nm;
      }
    }
    const uint32_t eqm = e & ~g;
    c_lt += __popc(inr & ~e);
    const uint32_t ne = __popc(eqm);
    c_eq += ne;
    const uint32_t inc = warp_incl_scan(ne);
    const uint32_t E = __shfl_sync(0xffffffffu, inc, 31);
    uint32_t keep = g;
    if (E) {
      if (tie_prefix) {
        // ties of rank < r (index order) are dropped: the first D of this lane
        const uint64_t rk0 = (uint64_t)__ldg(tie_prefix + c) + inc - ne;
        uint32_t d = r > rk0 ? (r - rk0 < ne ? (uint32_t)(r - rk0) : ne) : 0u, x = eqm;
        for (; d; --d) x &= x - 1;
        keep |= x;
      }
      if (hi < nhalves) {
        tie32[hi] = eqm;
        if (tie_old32) tie_old32[hi] = old & eqm;  // previous bits of the ties: the fix-up's change test
      }
    }
    if (lane == 0) {
      ties_out[c] = E;
      if (ties_prev && ties_prev[c] != E) mismatch = 1;
    }
    if (hi < nhalves && old != keep) {
      words32[hi] = keep;
      if ((old ^ keep) & ~cand & ~eqm) changed = 1;
      if ((old ^ keep) & cand) changed_cand = 1;
      if ((old ^ keep) & eqm) changed_tie = 1;
    }
    const uint32_t pc = warp_sum((uint32_t)__popc(keep));
    if (lane == 0) chunk_popc[c] = pc;
  }
  if constexpr (kBulk) {  // retire the mbarriers (no copy is outstanding: every issued chunk was waited on)
    __syncwarp();
  }
  if (fill) flush_pairs(cbk, cbi, fill, &counts->n_cand, cb);
  if (cb.hist) {
    __syncthreads();
    for (int b = threadIdx.x; b < (1 << kCandHistBits); b += blockDim.x)
      if (chist[b]) atomicAdd(&cb.hist[b], chist[b]);
  }
  c_lt = warp_sum(c_lt);
  c_eq = warp_sum(c_eq);
  c_below = warp_sum(c_below);
  changed = __any_sync(0xffffffffu, changed);
  changed_cand = __any_sync(0xffffffffu, changed_cand);
  changed_tie = __any_sync(0xffffffffu, changed_tie);
  mismatch = __any_sync(0xffffffffu, mismatch);
  if (lane == 0) {
    if (c_lt) atomicAdd(&counts->n_lt, (unsigned long long)c_lt);
    if (c_eq) atomicAdd(&counts->n_eq, (unsigned long long)c_eq);
    if (c_below) atomicAdd(&counts->n_cand_below, (unsigned long long)c_below);  // candidates below T
    if (changed) atomicOr(&counts->changed, 1);
    if (changed_cand) atomicOr(&counts->changed_cand, 1);
    if (changed_tie) atomicOr(&counts->changed_tie, 1);
    if (mismatch) atomicOr(&counts->tie_mismatch, 1);
  }
}

// ------------------------------------------------------- window fix-up
// The pass's threshold T was stale, the true T' lies in the window: every
// candidate's bit is rewritten for T' (ties provisionally dropped, recorded
// for the tie fix-up when they straddle the rank r').
__global__ void prune_win_final_kernel(const SelState* __restrict__ sel, uint32_t base, int bits, uint64_t ncand,
                                       uint64_t c_base, uint64_t k, WinSel* __restrict__ ws) {
  WinSel o{};
  uint64_t below = 0, eq = ncand;
  uint32_t v = 0;
  if (bits > 0) {
    v = sel->prefix;
    below = sel->below;
    eq = sel->eq;
    o.err = sel->err;
  }
  o.T1 = base + v;
  o.below = below;
  o.eq1 = eq;
  o.c_lt1 = c_base + below;
  o.r1 = k - o.c_lt1;
  if (o.c_lt1 >= k || o.r1 > eq) o.err = 1;
  o.straddle = !o.err && o.r1 < eq;
  *ws = o;
}

__global__ void __launch_bounds__(256)
    prune_cand_tieclear_kernel(const uint32_t* __restrict__ key, const uint32_t* __restrict__ idx, uint64_t n,
                               const WinSel* __restrict__ ws, uint64_t* __restrict__ tie_words) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (!ws->straddle || j >= n || key[j] != ws->T1) return;
  const uint64_t c = (idx[j] & 0x7fffffffu) >> 10;
#pragma unroll
  for (int q = 0; q < kChunkWords; ++q) tie_words[c * kChunkWords + q] = 0ull;
}

__global__ void __launch_bounds__(256)
    prune_cand_fix_kernel(const uint32_t* __restrict__ key, const uint32_t* __restrict__ idx, uint64_t n,
                          const WinSel* __restrict__ ws, unsigned long long* __restrict__ words,
                          uint32_t* __restrict__ chunk_popc, unsigned long long* __restrict__ tie_words,
                          uint32_t* __restrict__ ties, int* __restrict__ changed) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t T = ws->T1;
  const int straddle = ws->straddle;
  bool ch = false;
  if (j < n) {
    const uint32_t kq = key[j], v = idx[j], ix = v & 0x7fffffffu;
    const bool keep = kq > T;
    const unsigned long long bit = 1ull << (ix & 63);
    const bool tie = kq == T && straddle;  // final bit decided by the tie fix-up
    if (tie) {
      atomicOr(&tie_words[ix >> 6], bit);
      atomicAdd(&ties[ix >> 10], 1u);
    }
    // only the bits between the pass's threshold and T' flip: test first,
    // atomics for the flips alone (other candidates of the word may flip too)
    if ((((words[ix >> 6] & bit) != 0) != keep) || tie) {
      const unsigned long long old = keep ? atomicOr(&words[ix >> 6], bit) : atomicAnd(&words[ix >> 6], ~bit);
      if (((old & bit) != 0) != keep) atomicAdd(&chunk_popc[ix >> 10], keep ? 1u : 0xffffffffu);
    }
    ch = !tie && keep != (bool)(v >> 31);
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

__global__ void __launch_bounds__(256)
    prune_cand_changed_kernel(const uint32_t* __restrict__ key, const uint32_t* __restrict__ idx, uint64_t n,
                              const WinSel* __restrict__ ws, const uint64_t* __restrict__ words,
                              int* __restrict__ flag) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (!ws->straddle) return;
  bool ch = false;
  if (j < n && key[j] == ws->T1) {  // the tie candidates (the others were checked by the fix-up)
    const uint32_t v = idx[j], ix = v & 0x7fffffffu;
    ch = ((words[ix >> 6] >> (ix & 63)) & 1u) != (v >> 31);
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *flag = 1;
}

// ----------------------------------------------------------------- tiefix
// Rewrite the tie bits of chunks with ties: the first D = clamp(r - prefix,
// 0, E) ties of the chunk (index order) are dropped, the rest kept -- or,
// keep_low (TopK, codec.cpp:147-172: ties select the lower index), the
// first D kept and the rest dropped.
__global__ void __launch_bounds__(256)
    prune_tiefix_kernel(uint64_t* __restrict__ words, uint64_t nwords,
                        const uint64_t* __restrict__ tie_words, const uint32_t* __restrict__ ties,
                        const uint32_t* __restrict__ tie_prefix, uint64_t r, int keep_low,
                        uint32_t* __restrict__ chunk_popc, uint64_t nchunks,
                        const uint64_t* __restrict__ tie_old, int* __restrict__ changed,
                        const WinSel* __restrict__ ws) {
  if (ws) {
    if (!ws->straddle) return;
    r = ws->r1;
  }
  // a warp scans the tie counts of 32 chunks at a time (one coalesced load)
  // and fixes only the chunks that hold ties: ties are rare except at key 0
  const int lane = threadIdx.x & 31;
  const uint64_t wg = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g0 = wg * 32; g0 < nchunks; g0 += nwarps * 32) {
    const uint32_t El = g0 + lane < nchunks ? ties[g0 + lane] : 0u;
    uint32_t todo = __ballot_sync(0xffffffffu, El != 0);
    while (todo) {
      const int bsel = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t c = g0 + bsel;
      const uint32_t E = __shfl_sync(0xffffffffu, El, bsel);
      const uint64_t pre = tie_prefix[c];
      const uint64_t D = r > pre ? (r - pre < E ? r - pre : E) : 0;
      const uint64_t wi = c * kChunkWords + lane;
      const bool valid = lane < kChunkWords && wi < nwords;
      const uint64_t tw = valid ? tie_words[wi] : 0ull;
      const uint32_t tc = (uint32_t)__popcll(tw);
      const uint32_t inc = warp_incl_scan(tc);
      const uint64_t excl = inc - tc;
      uint64_t d = D > excl ? D - excl : 0;
      if (d > tc) d = tc;
      uint64_t first = 0, x = tw;  // the chunk's first d ties of this word
      for (uint64_t q = 0; q < d; ++q) {
        const uint64_t bb = x & (~x + 1);
        first |= bb;
        x ^= bb;
      }
      uint32_t pc = 0;
      bool ch = false;
      if (valid) {
        // prune: the first ties (lowest indices) are dropped; TopK keeps them
        const uint64_t nw = (words[wi] & ~tw) | (keep_low ? first : (tw & ~first));
        words[wi] = nw;
        pc = (uint32_t)__popcll(nw);
        if (tie_old) ch = (nw & tw) != tie_old[wi];
      }
      if (tie_old && __any_sync(0xffffffffu, ch) && lane == 0) *changed = 1;
      pc = warp_sum(pc);
      if (lane == 0) chunk_popc[c] = pc;
    }
  }
}

}  // namespace

void launch_prune_sample(const float* w, uint64_t len, uint64_t k, PruneWindow* win_dev,
                         cudaStream_t s) {
  prune_sample_kernel<<<1, 1024, 0, s>>>(w, len, k, win_dev);
  note_launch();
}

void launch_prune_count(const float* w, uint64_t len, const PruneWindow* win_dev,
                        PruneCounts* counts_dev, uint32_t* cand, uint64_t cand_cap,
                        cudaStream_t s) {
  cudaMemsetAsync(counts_dev, 0, sizeof(PruneCounts), s);
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  static unsigned cap = 0;
  if (!cap) cap = persistent_grid(prune_count_kernel, kPruneWarps * 32, 0, ~0ull >> 8, kPruneWarps);
  const unsigned grid = (unsigned)((nc + kPruneWarps - 1) / kPruneWarps < cap ? (nc + kPruneWarps - 1) / kPruneWarps : cap);
  prune_count_kernel<<<grid ? grid : 1, kPruneWarps * 32, 0, s>>>(w, len, win_dev, counts_dev, cand,
                                                                  cand_cap, nc);
  note_launch();
}

void launch_prune_hist(const void* src, int from_float, uint64_t n, uint32_t base, int shift,
                       int nbits, uint32_t prefix, uint32_t* hist, cudaStream_t s) {
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) << nbits, s);
  uint64_t blocks = (n + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  const size_t smem = sizeof(uint32_t) << nbits;
  if (from_float)
    prune_hist_kernel<true><<<(unsigned)blocks, 256, smem, s>>>(src, n, base, shift, nbits, prefix,
                                                               hist, nullptr);
  else
    prune_hist_kernel<false><<<(unsigned)blocks, 256, smem, s>>>(src, n, base, shift, nbits,
                                                                prefix, hist, nullptr);
  note_launch();
}

void launch_prune_hist_sel(const void* src, int from_float, uint64_t n, uint32_t base, int shift,
                           int nbits, int first, const SelState* sel, uint32_t* hist, cudaStream_t s) {
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) << nbits, s);
  // candidate lists are small and L2 resident: few CTAs, so the per-CTA
  // histogram flushes (up to 2^nbits global atomics each) stay cheap
  uint64_t blocks = from_float ? (n + 255) / 256 : (n + 4095) / 4096;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  const size_t smem = sizeof(uint32_t) << nbits;
  const SelState* sp = first ? nullptr : sel;  // first pass: prefix 0
  if (from_float)
    prune_hist_kernel<true><<<(unsigned)blocks, 256, smem, s>>>(src, n, base, shift, nbits, 0u, hist, sp);
  else
    prune_hist_kernel<false><<<(unsigned)blocks, 256, smem, s>>>(src, n, base, shift, nbits, 0u, hist, sp);
  note_launch();
}

void launch_prune_pick(const uint32_t* hist, int nbits, int first, uint64_t rank, SelState* sel,
                       cudaStream_t s) {
  prune_pick_kernel<<<1, 1024, 0, s>>>(hist, nbits, first, rank, sel);
  note_launch();
}

void launch_prune_bitmap(const float* w, uint64_t len, uint32_t T, uint64_t r,
                         const uint32_t* tie_prefix, uint64_t* words, uint32_t* chunk_popc,
                         uint32_t* ties_out, const uint32_t* ties_prev, uint64_t* tie_words,
                         BitmapCounts* counts, cudaStream_t s, const PruneCandBuf& cand,
                         uint64_t* tie_old) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  cudaMemsetAsync(counts, 0, sizeof(BitmapCounts), s);
  if (cand.hist) cudaMemsetAsync(cand.hist, 0, sizeof(uint32_t) << kCandHistBits, s);
  if (!nc) return;
  // PACT_BITMAP_CPASYNC=1: the per-lane cp.async ring instead of the bulk
  // copies; PACT_BITMAP_STAGES=3: three bulk stages per warp (two chunks in
  // flight, 2 CTAs per SM instead of 3)
  static const bool bulk = getenv("PACT_BITMAP_CPASYNC") == nullptr;
  static const bool three = bulk && getenv("PACT_BITMAP_STAGES") && atoi(getenv("PACT_BITMAP_STAGES")) == 3;
  constexpr size_t kSmem3 = bitmap_smem(3);
  static DeviceCache<unsigned> cap;
  unsigned& cp = cap.get();
  if (!cp) {
    cudaFuncSetAttribute(prune_bitmap_kernel<true, kKeyStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBitmapSmem);
    cudaFuncSetAttribute(prune_bitmap_kernel<false, kKeyStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBitmapSmem);
    cudaFuncSetAttribute(prune_bitmap_kernel<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem3);
    cp = three ? persistent_grid(prune_bitmap_kernel<true, 3>, kPruneWarps * 32, kSmem3, ~0ull >> 8, kPruneWarps)
               : persistent_grid(prune_bitmap_kernel<true, kKeyStages>, kPruneWarps * 32, kBitmapSmem, ~0ull >> 8,
                                 kPruneWarps);
  }
  const uint64_t need = (nc + kPruneWarps - 1) / kPruneWarps;
  const unsigned grid = (unsigned)(need < cp ? need : cp);
  if (three)
    prune_bitmap_kernel<true, 3><<<grid, kPruneWarps * 32, kSmem3, s>>>(
        w, len, T, r, tie_prefix, words, (len + 63) / 64, chunk_popc, ties_out, ties_prev, tie_words, tie_old,
        counts, nc, cand);
  else if (bulk)
    prune_bitmap_kernel<true, kKeyStages><<<grid, kPruneWarps * 32, kBitmapSmem, s>>>(
        w, len, T, r, tie_prefix, words, (len + 63) / 64, chunk_popc, ties_out, ties_prev, tie_words, tie_old,
        counts, nc, cand);
  else
    prune_bitmap_kernel<false, kKeyStages><<<grid, kPruneWarps * 32, kBitmapSmem, s>>>(
        w, len, T, r, tie_prefix, words, (len + 63) / 64, chunk_popc, ties_out, ties_prev, tie_words, tie_old,
        counts, nc, cand);
  note_launch();
}

__global__ void prune_win_report_kernel(const WinSel* ws, const uint64_t* digest, const uint32_t* nnz,
                                        const int* fix_changed, WinReport* out) {
  WinReport r;
  r.w = *ws;
  r.digest = *digest;
  r.nnz = *nnz;
  r.fix_changed = *fix_changed;
  *out = r;
}

namespace {
__global__ void prune_hit_gate_kernel(const BitmapCounts* bc, uint64_t k, uint64_t r0, int pv, int force,
                                      int* gate, HitReport* out) {
  const unsigned long long n_lt = bc->n_lt, n_eq = bc->n_eq;
  const bool hit = n_lt < k && k <= n_lt + n_eq;
  const unsigned long long r = k - n_lt;
  const bool fix = pv ? (r != r0 || bc->tie_mismatch != 0) : (r < n_eq);
  const bool ok = hit && !fix;
  const bool chg = ok && (bc->changed | bc->changed_cand | bc->changed_tie) != 0;
  const int g[3] = {chg, ok, chg || (ok && force)};
  out->bc = *bc;
  for (int i = 0; i < 3; ++i) gate[i] = out->gate[i] = g[i];
  out->digest = 0ull;
  out->nnz = 0u;
}
__global__ void prune_hit_report_kernel(const BitmapCounts* bc, const int* gate, const uint64_t* digest,
                                        const uint32_t* nnz, HitReport* out) {
  out->bc = *bc;
  out->gate[0] = gate[0];
  out->gate[1] = gate[1];
  out->gate[2] = gate[2];
  out->digest = gate[2] ? *digest : 0ull;
  out->nnz = gate[0] ? *nnz : 0u;
}
}  // namespace

void launch_prune_hit_gate(const BitmapCounts* bc, uint64_t k, uint64_t r0, int pv, int force_digest, int* gate,
                           HitReport* out, cudaStream_t s) {
  prune_hit_gate_kernel<<<1, 1, 0, s>>>(bc, k, r0, pv, force_digest, gate, out);
  note_launch();
}
void launch_prune_hit_report(const BitmapCounts* bc, const int* gate, const uint64_t* digest, const uint32_t* nnz,
                             HitReport* out, cudaStream_t s) {
  prune_hit_report_kernel<<<1, 1, 0, s>>>(bc, gate, digest, nnz, out);
  note_launch();
}

void launch_prune_win_report(const WinSel* ws, const uint64_t* digest, const uint32_t* nnz,
                             const int* fix_changed, WinReport* out, cudaStream_t s) {
  prune_win_report_kernel<<<1, 1, 0, s>>>(ws, digest, nnz, fix_changed, out);
  note_launch();
}

void launch_prune_win_final(const SelState* sel, uint32_t base, int bits, uint64_t ncand, uint64_t c_base,
                            uint64_t k, WinSel* ws, cudaStream_t s) {
  prune_win_final_kernel<<<1, 1, 0, s>>>(sel, base, bits, ncand, c_base, k, ws);
  note_launch();
}

void launch_prune_cand_tieclear(const uint32_t* key, const uint32_t* idx, uint64_t n, const WinSel* ws,
                                uint64_t* tie_words, cudaStream_t s) {
  if (!n) return;
  prune_cand_tieclear_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(key, idx, n, ws, tie_words);
  note_launch();
}

void launch_prune_cand_fix(const uint32_t* key, const uint32_t* idx, uint64_t n, const WinSel* ws,
                           uint64_t* words, uint32_t* chunk_popc, uint64_t* tie_words, uint32_t* ties,
                           int* changed, cudaStream_t s) {
  if (!n) return;
  prune_cand_fix_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      key, idx, n, ws, reinterpret_cast<unsigned long long*>(words), chunk_popc,
      reinterpret_cast<unsigned long long*>(tie_words), ties, changed);
  note_launch();
}

void launch_prune_cand_changed(const uint32_t* key, const uint32_t* idx, uint64_t n, const WinSel* ws,
                               const uint64_t* words, int* flag, cudaStream_t s) {
  if (!n) return;
  prune_cand_changed_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(key, idx, n, ws, words, flag);
  note_launch();
}

void launch_prune_tiefix(uint64_t* words, uint64_t len, const uint64_t* tie_words,
                         const uint32_t* ties, const uint32_t* tie_prefix, uint64_t r,
                         uint32_t* chunk_popc, cudaStream_t s, int keep_low, const uint64_t* tie_old,
                         int* changed, const WinSel* ws) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  uint64_t blocks = (nc + 255) / 256;  // 8 warps x 32 chunks per CTA and pass
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  prune_tiefix_kernel<<<(unsigned)blocks, 256, 0, s>>>(words, (len + 63) / 64, tie_words, ties, tie_prefix, r,
                                                       keep_low, chunk_popc, nc, tie_old, changed, ws);
  note_launch();
}

}  // namespace pactk
