// prune_seg.cu -- per-layer magnitude pruning, every layer at once
// (north_star (1): "a per-layer k-th-magnitude threshold found by a
// histogram/radix-select kernel"). The reference rule
// (sparsity.cpp:33-59) applied to each layer slice [begin_s, end_s) with its
// own k_s = drop_count(ratio, len_s): keep all but the k_s smallest
// (|w|, index) of the slice.
//
// The global path's structure, batched over segments so the whole mask costs
// a fixed number of launches and two host round trips, whatever the number
// of layers (the first version looped over the layers on the host: ~300
// synchronisations for GPT-2-medium):
//   seg_sample   one CTA per layer: 65536 strided keys (the whole layer when
//                smaller -- then the window is the exact threshold), a
//                +-6 sigma window of the layer's k-th key by in-CTA radix
//                select.
//   seg_count    one full read, CTAs over (layer, 64 Ki-element) tiles:
//                per-layer counts below / at the window ends, the window
//                interior compacted into the layer's own candidate region.
//   seg_select   one CTA per layer: the exact k-th key from the counts and
//                an in-CTA radix select over the layer's candidates (L2).
//   seg_bitmap   one full read, warp per 1024-element chunk, lane-major like
//                prune_bitmap_kernel (prune.cu): bits key > T_s, ties at T_s
//                recorded (tie words, per-chunk counts) plus per-layer
//                counts that verify T_s.
//   seg_tiebase / seg_tiefix   ties of rank >= r_s = k_s - #(key < T_s)
//                within their layer are kept (index order), like the global
//                tie fix-up but with per-layer rank bases.
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

constexpr int kSegSample = 65536;       // sampled keys per layer (64 per thread)
constexpr int kSegSampleKeys = kSegSample / 1024;
constexpr int kSegWarps = 8;

__device__ __forceinline__ uint32_t block1024_excl_scan_u32(uint32_t v, uint32_t* scratch) {
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

// rank-th (0-based) smallest of the keys held by the CTA (nk per thread; 1024
// threads), by three smem-histogram digit passes (11/11/10 bits of 32-bit
// keys: the padding 0xffffffff sorts above every key)
template <int kN>
__device__ uint32_t cta_order_stat(const uint32_t (&r)[kN], uint32_t rank, uint32_t* hist, uint32_t* scratch,
                                   uint32_t* sh) {
  const int t = threadIdx.x;
  uint32_t prefix = 0, pmask = 0;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shf = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
    const uint32_t nb = pass == 2 ? 1024u : 2048u;
    hist[t] = 0;
    hist[t + 1024] = 0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kN; ++q)
      if ((r[q] & pmask) == prefix) atomicAdd(&hist[(r[q] >> shf) & (nb - 1)], 1u);
    __syncthreads();
    const uint32_t a = hist[2 * t], b2 = hist[2 * t + 1];
    const uint32_t excl = block1024_excl_scan_u32(a + b2, scratch);
    if (rank >= excl && rank < excl + a) {
      sh[0] = prefix | ((uint32_t)(2 * t) << shf);
      sh[1] = rank - excl;
    } else if (rank >= excl + a && rank < excl + a + b2) {
      sh[0] = prefix | ((uint32_t)(2 * t + 1) << shf);
      sh[1] = rank - excl - a;
    }
    __syncthreads();
    prefix = sh[0];
    rank = sh[1];
    pmask |= (nb - 1) << shf;
    __syncthreads();
  }
  return prefix;
}

__global__ void __launch_bounds__(1024, 1)
    seg_sample_kernel(const float* __restrict__ w, const SegInfo* __restrict__ info, SegState* __restrict__ st) {
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t scratch[32];
  __shared__ uint32_t sh[2];
  const int s = blockIdx.x;
  const SegInfo I = info[s];
  if (I.trivial) return;
  const uint64_t len = I.end - I.begin, k = I.k;
  const uint64_t S = len < (uint64_t)kSegSample ? len : (uint64_t)kSegSample;
  uint32_t r[kSegSampleKeys];
#pragma unroll
  for (int q = 0; q < kSegSampleKeys; ++q) {
    const uint64_t j = (uint64_t)q * 1024 + threadIdx.x;  // consecutive threads: consecutive samples
    r[q] = j < S ? mag_key(__ldg(w + I.begin + (j * len + len / 2) / S)) : 0xffffffffu;
  }
  uint32_t lo, hi;
  if (S == len) {  // the whole layer: its k-th smallest key exactly
    lo = hi = cta_order_stat(r, (uint32_t)(k - 1), hist, scratch, sh);
  } else {
    const double p = (double)k / (double)len;
    const double center = ((double)k - 0.5) / (double)len * (double)S;
    const double margin = 6.0 * sqrt((double)S * p * (1.0 - p)) + 8.0;
    const long lo_i = (long)floor(center - margin), hi_i = (long)ceil(center + margin);
    lo = lo_i <= 0 ? 0u : cta_order_stat(r, (uint32_t)lo_i, hist, scratch, sh);
    hi = hi_i >= (long)S - 1 ? 0x7fffffffu : cta_order_stat(r, (uint32_t)hi_i, hist, scratch, sh);
  }
  if (threadIdx.x == 0) {
    st[s].lo = lo;
    st[s].hi = hi;
  }
}

// ------------------------------------------------------------------ count
constexpr int kCntBuf = 512;  // per-warp candidate staging

__device__ __forceinline__ void seg_flush(uint32_t* buf, uint32_t fill, unsigned long long* seg_fill,
                                          uint32_t* __restrict__ region, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(seg_fill, (unsigned long long)fill);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (uint32_t i = lane; i < fill; i += 32)
    if (base + i < cap) region[base + i] = buf[i];
  __syncwarp();
}

__global__ void __launch_bounds__(kSegWarps * 32)
    seg_count_kernel(const float* __restrict__ w, const SegInfo* __restrict__ info, SegState* __restrict__ st,
                     const SegTile* __restrict__ tiles, uint32_t ntiles, uint32_t* __restrict__ cand,
                     unsigned long long* __restrict__ fill_seg) {
  __shared__ uint32_t buf_all[kSegWarps][kCntBuf];
  __shared__ unsigned long long red[kSegWarps][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* buf = buf_all[warp];
  for (uint32_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const SegTile tl = tiles[ti];
    const int s = (int)tl.seg;
    const uint32_t lo = st[s].lo, hi = st[s].hi;
    const SegInfo I = info[s];
    uint32_t* region = cand + I.cand_off;
    uint32_t c_lt = 0, c_eqlo = 0, c_eqhi = 0, fill = 0;
    auto one = [&](uint32_t kq, bool valid, uint32_t& nmid, uint32_t (&mk)[4], int slot) {
      c_lt += valid && kq < lo;
      c_eqlo += valid && kq == lo;
      c_eqhi += valid && kq == hi && hi != lo;
      const bool m = valid && kq > lo && kq < hi;
      mk[slot] = m ? kq : 0xffffffffu;
      nmid += m;
    };
    // float4 body over the 16-byte aligned part, scalars at the ends
    const uint64_t a = tl.begin, b = tl.end;
    const uint64_t a4 = (a + 3) & ~3ull, b4 = b & ~3ull;
    const uint64_t q0 = a4 < b4 ? a4 / 4 : 0, q1 = a4 < b4 ? b4 / 4 : 0;
    const uint64_t nv = q1 - q0;
    const uint64_t ns = (a4 < b4) ? (a4 - a) + (b - b4) : (b - a);  // scalar elements
    const uint64_t steps = (nv + blockDim.x - 1) / blockDim.x + (ns > 0 ? 1 : 0);
    for (uint64_t it = 0; it < steps; ++it) {
      uint32_t mk[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
      uint32_t nmid = 0;
      if (it < (nv + blockDim.x - 1) / blockDim.x) {
        const uint64_t q = q0 + it * blockDim.x + threadIdx.x;
        const bool v = q < q1;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v) x = ld_stream_f4(reinterpret_cast<const float4*>(w) + q);
        one(mag_key(x.x), v, nmid, mk, 0);
        one(mag_key(x.y), v, nmid, mk, 1);
        one(mag_key(x.z), v, nmid, mk, 2);
        one(mag_key(x.w), v, nmid, mk, 3);
      } else {  // the scalar head / tail, at most 6 elements
        const uint64_t j = threadIdx.x;
        uint64_t e = 0;
        bool v = false;
        if (a4 < b4) {
          if (j < a4 - a) {
            e = a + j;
            v = true;
          } else if (j - (a4 - a) < b - b4) {
            e = b4 + (j - (a4 - a));
            v = true;
          }
        } else if (j < b - a) {
          e = a + j;
          v = true;
        }
        one(v ? mag_key(w[e]) : 0u, v, nmid, mk, 0);
      }
      const uint32_t inc = warp_incl_scan(nmid);
      const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
      if (tot) {
        if (fill + tot > kCntBuf) {
          seg_flush(buf, fill, &fill_seg[s], region, I.cand_cap);
          fill = 0;
        }
        uint32_t o = fill + inc - nmid;
#pragma unroll
        for (int z = 0; z < 4; ++z)
          if (mk[z] != 0xffffffffu) buf[o++] = mk[z];
        __syncwarp();
        fill += tot;
      }
    }
    if (fill) seg_flush(buf, fill, &fill_seg[s], region, I.cand_cap);
    const uint32_t l0 = warp_sum(c_lt), l1 = warp_sum(c_eqlo), l2 = warp_sum(c_eqhi);
    if (lane == 0) {
      red[warp][0] = l0;
      red[warp][1] = l1;
      red[warp][2] = l2;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      unsigned long long t = 0;
      for (int q = 0; q < kSegWarps; ++q) t += red[q][threadIdx.x];
      if (t) {
        unsigned long long* dst = threadIdx.x == 0 ? &st[s].n_lt : (threadIdx.x == 1 ? &st[s].n_eq_lo : &st[s].n_eq_hi);
        atomicAdd(dst, t);
      }
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------- select
// one CTA per layer: T_s and #(key < T_s) from the counts, the k-th key from
// the layer's candidates when it lies inside the window (11-bit digit passes
// over the candidates, L2 resident), a fallback flag otherwise
__global__ void __launch_bounds__(1024, 1)
    seg_select_kernel(const SegInfo* __restrict__ info, SegState* __restrict__ st,
                      const uint32_t* __restrict__ cand, const unsigned long long* __restrict__ fill_seg) {
  __shared__ uint32_t hist[2048];
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long sh_rem, sh_below;
  __shared__ uint32_t sh_prefix;
  const int s = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const SegInfo I = info[s];
  if (I.trivial) return;
  SegState* S = &st[s];
  const uint32_t lo = S->lo, hi = S->hi;
  const uint64_t n_lt = S->n_lt, lo_end = n_lt + S->n_eq_lo;
  const uint64_t n_mid = fill_seg[s], mid_end = lo_end + n_mid, hi_end = mid_end + S->n_eq_hi;
  const uint64_t k = I.k;
  if (k <= n_lt || k > hi_end || n_mid > I.cand_cap) {  // the sampled window missed: the host resolves it
    if (t == 0) S->mode = 1;
    return;
  }
  uint32_t T;
  uint64_t c_lt;
  if (k <= lo_end) {
    T = lo;
    c_lt = n_lt;
  } else if (k > mid_end) {
    T = hi;
    c_lt = mid_end;
  } else {
    const uint32_t* src = cand + I.cand_off;
    const uint32_t base = lo + 1;
    const uint32_t span = hi - lo - 2;  // key - base <= span
    const int bits = span ? 32 - __clz(span) : 0;
    uint64_t rem = k - lo_end, below = 0;
    uint32_t prefix = 0;
    for (int hb = bits; hb > 0;) {
      const int nb = hb < 11 ? hb : 11;
      const int shf = hb - nb;
      hist[t] = 0;
      hist[t + 1024] = 0;
      __syncthreads();
      for (uint64_t i = t; i < n_mid; i += 1024) {
        const uint32_t kk = src[i] - base;
        if ((uint32_t)((uint64_t)kk >> (shf + nb)) == prefix) atomicAdd(&hist[(kk >> shf) & ((1u << nb) - 1)], 1u);
      }
      __syncthreads();
      const uint64_t x = (2 * t < (1 << nb) ? hist[2 * t] : 0u), y = (2 * t + 1 < (1 << nb) ? hist[2 * t + 1] : 0u);
      uint64_t inc = x + y;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      if (warp == 0) {
        const uint64_t v = wsum[lane];
        uint64_t vi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t u = __shfl_up_sync(0xffffffffu, vi, o);
          if (lane >= o) vi += u;
        }
        wsum[lane] = vi - v;
      }
      __syncthreads();
      const uint64_t e0 = wsum[warp] + inc - (x + y);
      if (e0 < rem && rem <= e0 + x) {
        sh_prefix = (prefix << nb) | (uint32_t)(2 * t);
        sh_rem = rem - e0;
        sh_below = below + e0;
      } else if (e0 + x < rem && rem <= e0 + x + y) {
        sh_prefix = (prefix << nb) | (uint32_t)(2 * t + 1);
        sh_rem = rem - e0 - x;
        sh_below = below + e0 + x;
      }
      __syncthreads();
      prefix = sh_prefix;
      rem = sh_rem;
      below = sh_below;
      hb = shf;
      __syncthreads();
    }
    T = base + prefix;
    c_lt = lo_end + below;
  }
  if (t == 0) {
    S->T = T;
    S->c_lt = c_lt;
    S->r = k - c_lt;
    S->mode = 0;
  }
}

// ----------------------------------------------------------------- bitmap
constexpr int kSbStages = 2;
constexpr int kSbStageFloats = kChunk;
constexpr size_t kSegBitmapSmem = (size_t)kSegWarps * kSbStages * kSbStageFloats * sizeof(float);

__device__ __forceinline__ void seg_chunk_issue(float* stg, const float* __restrict__ w, uint64_t c) {
  const int lane = threadIdx.x & 31;
  const float* src = w + c * (uint64_t)kChunk + 4 * lane;
#pragma unroll
  for (int j = 0; j < kVecPerLane; ++j) {
    const int u = 32 * j + lane, owner = u >> 3, col = u & 7;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(stg + 4 * (owner * 8 + (col ^ (owner & 7))));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 128 * j) : "memory");
  }
}

// the layer holding element e, walking forward from a layer at or before it
__device__ __forceinline__ uint32_t seg_walk(const SegInfo* __restrict__ info, uint32_t s, uint64_t e) {
  while (e >= info[s].end) ++s;
  return s;
}

// per-warp accumulation of a layer's counts, flushed on a change of layer
struct SegAcc {
  uint32_t s = 0xffffffffu;
  unsigned long long lt = 0, eq = 0;
};
__device__ __forceinline__ void seg_acc_flush(SegAcc& a, SegState* st) {
  if (a.s != 0xffffffffu && (a.lt | a.eq)) {
    if (a.lt) atomicAdd(&st[a.s].b_lt, a.lt);
    if (a.eq) atomicAdd(&st[a.s].b_eq, a.eq);
  }
  a.lt = a.eq = 0;
}

__global__ void __launch_bounds__(kSegWarps * 32)
    seg_bitmap_kernel(const float* __restrict__ w, uint64_t len, const SegInfo* __restrict__ info,
                      SegState* __restrict__ st, const uint32_t* __restrict__ chunk_seg,
                      uint64_t* __restrict__ words, uint64_t nwords, uint64_t* __restrict__ tie_words,
                      uint32_t* __restrict__ ties, uint32_t* __restrict__ chunk_popc, uint64_t nchunks) {
  extern __shared__ __align__(16) float sring_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ring = sring_all + (size_t)warp * kSbStages * kSbStageFloats;
  uint32_t* words32 = reinterpret_cast<uint32_t*>(words);
  uint32_t* tie32 = reinterpret_cast<uint32_t*>(tie_words);
  const uint64_t nhalves = 2 * nwords;
  const bool vec_ok = (((uintptr_t)w) & 15) == 0;
  auto full = [&](uint64_t c) { return vec_ok && (c + 1) * (uint64_t)kChunk <= len; };
  const uint64_t nw_total = (uint64_t)gridDim.x * kSegWarps;
  const uint64_t c0 = (uint64_t)blockIdx.x * kSegWarps + warp;
  SegAcc acc;  // lane 0's
  if (c0 < nchunks && full(c0)) seg_chunk_issue(ring, w, c0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int slot = 0;
  for (uint64_t c = c0; c < nchunks; c += nw_total) {
    {
      const uint64_t cn = c + nw_total;
      __syncwarp();
      if (cn < nchunks && full(cn)) seg_chunk_issue(ring + (slot ^ 1) * kSbStageFloats, w, cn);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
    }
    const float* stg = ring + slot * kSbStageFloats;
    slot ^= 1;
    const bool fc = full(c);
    const uint64_t e0 = c * (uint64_t)kChunk + 32 * lane;
    const uint32_t inr = e0 >= len ? 0u : (len - e0 >= 32 ? ~0u : (1u << (len - e0)) - 1u);
    // this lane's layer (one layer for all 32 elements: the common case)
    const uint32_t sc = chunk_seg[c];
    const uint32_t s = e0 < len ? seg_walk(info, sc, e0) : sc;
    const uint64_t last = e0 + 31 < len ? e0 + 31 : len - 1;
    const bool uni = e0 >= len || last < info[s].end;
    uint32_t g = 0, e = 0;
    if (uni && fc) {
      const uint32_t T = st[s].T;
#pragma unroll
      for (int k = kVecPerLane - 1; k >= 0; --k) {
        const float4 v = *reinterpret_cast<const float4*>(stg + 4 * (lane * 8 + (k ^ (lane & 7))));
        const uint32_t k3 = mag_key(v.w), k2 = mag_key(v.z), k1 = mag_key(v.y), k0 = mag_key(v.x);
        g = __funnelshift_l(T - k3, g, 1);
        e = __funnelshift_l(T - 1u - k3, e, 1);
        g = __funnelshift_l(T - k2, g, 1);
        e = __funnelshift_l(T - 1u - k2, e, 1);
        g = __funnelshift_l(T - k1, g, 1);
        e = __funnelshift_l(T - 1u - k1, e, 1);
        g = __funnelshift_l(T - k0, g, 1);
        e = __funnelshift_l(T - 1u - k0, e, 1);
      }
    } else {  // layer boundary inside the lane's 32 elements, or the ragged end
      uint32_t ss = s;
      for (int i = 0; i < 32; ++i) {
        const uint64_t ei = e0 + i;
        if (ei >= len) break;
        ss = seg_walk(info, ss, ei);
        const uint32_t T = st[ss].T;
        const uint32_t kq = mag_key(fc ? stg[4 * (lane * 8 + ((i >> 2) ^ (lane & 7))) + (i & 3)] : w[ei]);
        g |= (uint32_t)(kq > T) << i;
        e |= (uint32_t)(kq >= T) << i;
      }
    }
    g &= inr;
    e &= inr;
    const uint32_t eqm = e & ~g;
    // per-layer verification counts: #(key < T_s), #(key == T_s)
    {
      const uint32_t lt = __popc(inr & ~e), eq = __popc(eqm);
      const uint32_t s_lane0 = __shfl_sync(0xffffffffu, s, 0);  // every lane takes part in the shuffle
      const bool warp_uni = __all_sync(0xffffffffu, uni && (e0 >= len || s == s_lane0));
      if (warp_uni) {
        const uint32_t slt = warp_sum(lt), seq = warp_sum(eq);
        if (lane == 0) {
          if (acc.s != s) {
            seg_acc_flush(acc, st);
            acc.s = s;
          }
          acc.lt += slt;
          acc.eq += seq;
        }
      } else {  // mixed layers in this chunk: per element, straight to the layer counters
        for (int i = 0; i < 32; ++i) {
          if (!((inr >> i) & 1u)) break;
          const uint32_t si = seg_walk(info, s, e0 + i);
          if (!((e >> i) & 1u)) atomicAdd(&st[si].b_lt, 1ull);
          else if ((eqm >> i) & 1u) atomicAdd(&st[si].b_eq, 1ull);
        }
      }
    }
    const uint32_t E = warp_sum((uint32_t)__popc(eqm));
    const uint64_t hi2 = c * 32 + lane;
    if (E && hi2 < nhalves) tie32[hi2] = eqm;
    if (hi2 < nhalves) words32[hi2] = g;  // ties provisionally dropped
    const uint32_t pc = warp_sum((uint32_t)__popc(g));
    if (lane == 0) {
      ties[c] = E;
      chunk_popc[c] = pc;
    }
  }
  if (lane == 0) seg_acc_flush(acc, st);
}

// ties before each layer's first element (ranks are counted within a layer)
__global__ void seg_tiebase_kernel(const SegInfo* __restrict__ info, SegState* __restrict__ st, uint32_t nseg,
                                   const uint64_t* __restrict__ tie_words, const uint32_t* __restrict__ ties,
                                   const uint32_t* __restrict__ tie_prefix) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const uint64_t b = info[s].begin, c = b >> 10;
  uint64_t base = tie_prefix[c];
  if (ties[c]) {  // tie words are only written for chunks with ties
    const uint64_t w0 = c * kChunkWords, wb = b >> 6;
    for (uint64_t q = w0; q < wb; ++q) base += __popcll(tie_words[q]);
    if (b & 63) base += __popcll(tie_words[wb] & ((1ull << (b & 63)) - 1ull));
  }
  st[s].tie_base = base;
}

// keep tie j of layer s iff its rank among the layer's ties (index order)
// is >= r_s; a warp scans the tie counts of 32 chunks, fixes those with ties
__global__ void __launch_bounds__(256)
    seg_tiefix_kernel(const SegInfo* __restrict__ info, const SegState* __restrict__ st,
                      const uint32_t* __restrict__ chunk_seg, uint64_t* __restrict__ words, uint64_t nwords,
                      const uint64_t* __restrict__ tie_words, const uint32_t* __restrict__ ties,
                      const uint32_t* __restrict__ tie_prefix, uint32_t* __restrict__ chunk_popc,
                      uint64_t nchunks) {
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
      const uint64_t wi = c * kChunkWords + lane;
      const bool valid = lane < kChunkWords && wi < nwords;
      const uint64_t tw = valid ? tie_words[wi] : 0ull;
      const uint32_t tc = (uint32_t)__popcll(tw);
      const uint32_t ex = warp_incl_scan(tc) - tc;
      uint64_t keep = 0, x = tw;
      uint32_t s = chunk_seg[c], seen = 0;
      while (x) {
        const int bb = __ffsll((long long)x) - 1;
        x &= x - 1;
        const uint64_t ei = wi * 64 + bb;
        s = seg_walk(info, s, ei);
        const uint64_t rank = (uint64_t)tie_prefix[c] + ex + seen - st[s].tie_base;
        if (rank >= st[s].r) keep |= 1ull << bb;
        ++seen;
      }
      uint32_t pc = 0;
      if (valid) {
        const uint64_t nw = words[wi] | keep;
        words[wi] = nw;
        pc = (uint32_t)__popcll(nw);
      }
      pc = warp_sum(pc);
      if (lane == 0) chunk_popc[c] = pc;
    }
  }
}

int sms_seg() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

void launch_seg_sample(const float* w, const SegInfo* info, SegState* st, uint32_t nseg, cudaStream_t s) {
  if (!nseg) return;
  seg_sample_kernel<<<nseg, 1024, 0, s>>>(w, info, st);
  note_launch();
}

void launch_seg_count(const float* w, const SegInfo* info, SegState* st, const SegTile* tiles, uint32_t ntiles,
                      uint32_t* cand, unsigned long long* fill, cudaStream_t s) {
  if (!ntiles) return;
  static DeviceCache<int> cc;
  int& cap = cc.get();
  if (!cap) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, seg_count_kernel, kSegWarps * 32, 0);
    cap = sms_seg() * (per > 0 ? per : 1);
  }
  seg_count_kernel<<<ntiles < (uint32_t)cap ? ntiles : (uint32_t)cap, kSegWarps * 32, 0, s>>>(w, info, st, tiles,
                                                                                             ntiles, cand, fill);
  note_launch();
}

void launch_seg_select(const SegInfo* info, SegState* st, uint32_t nseg, const uint32_t* cand,
                       const unsigned long long* fill, cudaStream_t s) {
  if (!nseg) return;
  seg_select_kernel<<<nseg, 1024, 0, s>>>(info, st, cand, fill);
  note_launch();
}

void launch_seg_bitmap(const float* w, uint64_t len, const SegInfo* info, SegState* st, const uint32_t* chunk_seg,
                       uint64_t* words, uint64_t* tie_words, uint32_t* ties, uint32_t* chunk_popc, cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  static DeviceCache<int> cc;
  int& cap = cc.get();
  if (!cap) {
    cudaFuncSetAttribute(seg_bitmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSegBitmapSmem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, seg_bitmap_kernel, kSegWarps * 32, kSegBitmapSmem);
    cap = sms_seg() * (per > 0 ? per : 1);
  }
  const uint64_t need = (nc + kSegWarps - 1) / kSegWarps;
  seg_bitmap_kernel<<<(unsigned)(need < (uint64_t)cap ? need : (uint64_t)cap), kSegWarps * 32, kSegBitmapSmem, s>>>(
      w, len, info, st, chunk_seg, words, (len + 63) / 64, tie_words, ties, chunk_popc, nc);
  note_launch();
}

void launch_seg_tiebase(const SegInfo* info, SegState* st, uint32_t nseg, const uint64_t* tie_words,
                        const uint32_t* ties, const uint32_t* tie_prefix, cudaStream_t s) {
  if (!nseg) return;
  seg_tiebase_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(info, st, nseg, tie_words, ties, tie_prefix);
  note_launch();
}

namespace {
__global__ void seg_verify_kernel(const SegInfo* __restrict__ info, SegState* __restrict__ st, uint32_t nseg,
                                  int* __restrict__ miss) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nseg; q += gridDim.x * blockDim.x) {
    if (info[q].trivial) continue;
    const unsigned long long k = info[q].k, lt = st[q].b_lt, eq = st[q].b_eq;
    if (lt < k && k <= lt + eq) {
      st[q].c_lt = lt;
      st[q].r = k - lt;
    } else {
      atomicExch(miss, 1);
    }
  }
}
}  // namespace

void launch_seg_verify(const SegInfo* info, SegState* st, uint32_t nseg, int* miss, cudaStream_t s) {
  if (!nseg) return;
  seg_verify_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(info, st, nseg, miss);
  note_launch();
}

void launch_seg_tiefix(uint64_t len, const SegInfo* info, const SegState* st, const uint32_t* chunk_seg,
                       uint64_t* words, const uint64_t* tie_words, const uint32_t* ties, const uint32_t* tie_prefix,
                       uint32_t* chunk_popc, cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  uint64_t blocks = (nc + 255) / 256;
  const uint64_t cap = (uint64_t)sms_seg() * 8;
  if (blocks > cap) blocks = cap;
  seg_tiefix_kernel<<<(unsigned)blocks, 256, 0, s>>>(info, st, chunk_seg, words, (len + 63) / 64, tie_words, ties,
                                                     tie_prefix, chunk_popc, nc);
  note_launch();
}

}  // namespace pactk
