// prune.cu -- global magnitude pruning (reference: sparsity.cpp:33-59).
//
// The reference stable-sorts an index array by |w| and drops the first k
// positions: the k smallest (|w_i|, i) pairs, ties at the threshold dropped
// lowest-index first. With key = bits(w) & 0x7fffffff (monotone in |w| for
// finite values, +0/-0 tie) that is:
//
//   T    = k-th smallest key,  c_lt = #(key < T),  r = k - c_lt
//   bit_i = key_i > T  ||  (key_i == T  &&  tierank_i >= r)
//
// where tierank_i = #{j < i : key_j == T}. The selection of T is
// sample-guided so the dense array is streamed only twice:
//   1. prune_sample  (1 CTA): 16384 strided keys, bitonic-sorted in smem;
//      a [lo, hi] window of +-6 sigma around the expected rank of the k-th key.
//   2. prune_count   (full read): #(key<lo), #(key==lo), #(key==hi), and the
//      window-interior keys compacted to a small candidate buffer.
//   3. prune_hist    (only if T is strictly inside the window): radix-select
//      digits over the candidate buffer (L2 resident).
//   4. prune_bitmap  (full read): mask words + per-tile kept counts; the
//      tie ranks come from a decoupled look-back over per-tile tie counts.
// If the window misses (sample unrepresentative) or the candidate buffer
// overflows, step 3 runs over the full array instead (3 digit passes); the
// result is identical, only slower.
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

constexpr int kSample = 16384;

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

// ---------------------------------------------------------------- sample
__global__ void __launch_bounds__(1024, 1)
    prune_sample_kernel(const float* __restrict__ w, uint64_t len, uint64_t k,
                        PruneWindow* __restrict__ win) {
  extern __shared__ uint32_t s[];
  const int tid = threadIdx.x;
  for (int i = tid; i < kSample; i += 1024) {
    const uint64_t idx = ((uint64_t)i * len + len / 2) / kSample;  // < len
    s[i] = mag_key(w[idx]);
  }
  __syncthreads();
  for (int kk = 2; kk <= kSample; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < kSample; i += 1024) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = s[i], b = s[ixj];
          const bool asc = (i & kk) == 0;
          if ((a > b) == asc) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    const double p = (double)k / (double)len;
    const double center = ((double)k - 0.5) / (double)len * kSample;
    const double margin = 6.0 * sqrt(kSample * p * (1.0 - p)) + 8.0;
    const long lo_i = (long)floor(center - margin);
    const long hi_i = (long)ceil(center + margin);
    PruneWindow out;
    out.lo = lo_i <= 0 ? 0u : s[lo_i];
    out.hi = hi_i >= kSample - 1 ? 0x7fffffffu : s[hi_i];
    *win = out;
  }
}

// ----------------------------------------------------------------- count
__global__ void __launch_bounds__(kThreads)
    prune_count_kernel(const float* __restrict__ w, uint64_t len, const PruneWindow* __restrict__ win,
                       PruneCounts* __restrict__ counts, uint32_t* __restrict__ cand,
                       uint64_t cap, uint64_t ntiles) {
  __shared__ unsigned long long scratch[kThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x;
  const uint32_t lo = win->lo, hi = win->hi;
  const bool vec_ok = (((uintptr_t)w) & 15) == 0;
  uint32_t c_lt = 0, c_eqlo = 0, c_eqhi = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t e0 = t * (uint64_t)kTile;
    uint32_t key[kVecPerThread * 4];
    uint32_t inr = 0;  // in-range bits
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const uint64_t ge = e0 + (uint64_t)(j * kThreads + tid) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vec_ok && ge + 4 <= len) {
        v = ld_stream_f4(reinterpret_cast<const float4*>(w + ge));
        inr |= 0xFu << (4 * j);
      } else {
        for (int b = 0; b < 4; ++b)
          if (ge + b < len) {
            (&v.x)[b] = w[ge + b];
            inr |= 1u << (4 * j + b);
          }
      }
      key[4 * j + 0] = mag_key(v.x);
      key[4 * j + 1] = mag_key(v.y);
      key[4 * j + 2] = mag_key(v.z);
      key[4 * j + 3] = mag_key(v.w);
    }
    uint32_t mid = 0;
#pragma unroll
    for (int q = 0; q < kVecPerThread * 4; ++q) {
      const bool in = (inr >> q) & 1;
      const uint32_t kq = key[q];
      c_lt += in && kq < lo;
      c_eqlo += in && kq == lo;
      c_eqhi += in && kq == hi && hi != lo;
      if (in && kq > lo && kq < hi) mid |= 1u << q;
    }
    unsigned long long tot;
    const unsigned long long off = block_excl_scan<unsigned long long>(__popc(mid), scratch, &tot);
    if (tot) {
      if (tid == 0) s_base = atomicAdd(&counts->n_mid, tot);
      __syncthreads();
      unsigned long long o = s_base + off;
      for (int q = 0; q < kVecPerThread * 4; ++q)
        if ((mid >> q) & 1) {
          if (o < cap) cand[o] = key[q];
          ++o;
        }
      __syncthreads();
    }
  }
  unsigned long long tot;
  block_excl_scan<unsigned long long>(c_lt, scratch, &tot);
  if (tid == 0 && tot) atomicAdd(&counts->n_lt, tot);
  block_excl_scan<unsigned long long>(c_eqlo, scratch, &tot);
  if (tid == 0 && tot) atomicAdd(&counts->n_eq_lo, tot);
  block_excl_scan<unsigned long long>(c_eqhi, scratch, &tot);
  if (tid == 0 && tot) atomicAdd(&counts->n_eq_hi, tot);
}

// ------------------------------------------------------------------ hist
template <bool kFloat>
__global__ void __launch_bounds__(256)
    prune_hist_kernel(const void* __restrict__ src, uint64_t n, uint32_t base, int shift, int nbits,
                      uint32_t prefix, uint32_t* __restrict__ ghist) {
  extern __shared__ uint32_t sh[];
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

// ---------------------------------------------------------------- bitmap
constexpr uint64_t kStAgg = 1ull << 62;
constexpr uint64_t kStIncl = 2ull << 62;
constexpr uint64_t kStMask = 3ull << 62;

__global__ void __launch_bounds__(kThreads, 4)
    prune_bitmap_kernel(const float* __restrict__ w, uint64_t len, uint32_t T, uint64_t r,
                        uint64_t* __restrict__ words, uint64_t nwords,
                        uint32_t* __restrict__ tile_popc, int* __restrict__ changed,
                        uint64_t* __restrict__ state, unsigned* __restrict__ tile_counter) {
  __shared__ unsigned long long scratch[kThreads / 32 + 1];
  __shared__ uint64_t sw[kTileWords];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_before;
  __shared__ uint32_t s_pc[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint64_t t = s_tile;
  const uint64_t e0 = t * (uint64_t)kTile;
  const bool vec_ok = (((uintptr_t)w) & 15) == 0;

  uint32_t gt = 0, eq = 0;  // bit q = 4*j + b
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    const uint64_t ge = e0 + (uint64_t)(j * kThreads + tid) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t inr = 0;
    if (vec_ok && ge + 4 <= len) {
      v = ld_stream_f4(reinterpret_cast<const float4*>(w + ge));
      inr = 0xF;
    } else {
      for (int b = 0; b < 4; ++b)
        if (ge + b < len) {
          (&v.x)[b] = w[ge + b];
          inr |= 1u << b;
        }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t kq = mag_key((&v.x)[b]);
      if ((inr >> b) & 1) {
        gt |= (uint32_t)(kq > T) << (4 * j + b);
        eq |= (uint32_t)(kq == T) << (4 * j + b);
      }
    }
  }
  // tie counts per float4 slot j, packed in 16-bit lanes of a u64, scanned
  // in (j, tid) order = element order within the tile
  unsigned long long packed_cnt = 0;
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j)
    packed_cnt |= (unsigned long long)__popc((eq >> (4 * j)) & 0xF) << (16 * j);
  unsigned long long tot;
  const unsigned long long excl = block_excl_scan<unsigned long long>(packed_cnt, scratch, &tot);
  uint32_t slot_base[kVecPerThread];
  uint32_t run = 0;
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    slot_base[j] = run + (uint32_t)((excl >> (16 * j)) & 0xFFFF);
    run += (uint32_t)((tot >> (16 * j)) & 0xFFFF);
  }
  const uint64_t E = run;  // ties in this tile

  // decoupled look-back over the tie counts (plain sum; identity = 0)
  if (warp == 0) {
    uint64_t before = 0;
    if (t == 0) {
      if (lane == 0) st_relaxed_u64(state, kStIncl | E);
    } else {
      if (lane == 0) st_relaxed_u64(state + t, kStAgg | E);
      int64_t base = (int64_t)t - 1;
      while (true) {
        const int64_t p = base - lane;
        uint64_t s = p >= 0 ? ld_relaxed_u64(state + p) : kStIncl;
        while (__any_sync(0xffffffffu, (s & kStMask) == 0)) {
          if ((s & kStMask) == 0) s = ld_relaxed_u64(state + p);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, (s & kStMask) == kStIncl);
        const int L = incl ? __ffs(incl) - 1 : 31;
        uint64_t v = lane <= L ? (s & ~kStMask) : 0ull;
        v = warp_sum(v);
        before += v;
        if (incl) break;
        base -= 32;
      }
      if (lane == 0) st_relaxed_u64(state + t, kStIncl | (before + E));
    }
    if (lane == 0) s_before = before;
  }
  __syncthreads();
  const uint64_t before = s_before;

  // final bits: keep = key > T || (key == T && tierank >= r)
  uint32_t keep = gt;
  if (eq) {
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      uint32_t rk = slot_base[j];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = 4 * j + b;
        if ((eq >> q) & 1) {
          if (before + rk >= r) keep |= 1u << q;
          ++rk;
        }
      }
    }
  }
  // assemble words: slot j of lane l covers word 16j + 2*warp + (l >= 16),
  // nibble 4*(l & 15)
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    uint32_t x = ((keep >> (4 * j)) & 0xFu) << (4 * (lane & 7));
    x |= __shfl_xor_sync(0xffffffffu, x, 1);
    x |= __shfl_xor_sync(0xffffffffu, x, 2);
    x |= __shfl_xor_sync(0xffffffffu, x, 4);
    const uint32_t hi32 = __shfl_down_sync(0xffffffffu, x, 8);
    if ((lane & 15) == 0) sw[16 * j + 2 * warp + (lane >> 4)] = (uint64_t)x | ((uint64_t)hi32 << 32);
  }
  __syncthreads();
  if (tid < kTileWords) {
    const uint64_t wi = t * kTileWords + tid;
    const uint64_t nwv = sw[tid];
    uint32_t pc = 0;
    int diff = 0;
    if (wi < nwords) {
      diff = words[wi] != nwv;
      words[wi] = nwv;
      pc = __popcll(nwv);
    }
    pc = warp_sum(pc);
    diff = __any_sync(0xffffffffu, diff);
    if (lane == 0) {
      s_pc[warp] = pc;
      if (diff) atomicOr(changed, 1);
    }
  }
  __syncthreads();
  if (tid == 0) tile_popc[t] = s_pc[0] + s_pc[1];
}

}  // namespace

void launch_prune_sample(const float* w, uint64_t len, uint64_t k, PruneWindow* win_dev,
                         cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prune_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSample * 4);
    attr = true;
  }
  prune_sample_kernel<<<1, 1024, kSample * 4, s>>>(w, len, k, win_dev);
  note_launch();
}

void launch_prune_count(const float* w, uint64_t len, const PruneWindow* win_dev,
                        PruneCounts* counts_dev, uint32_t* cand, uint64_t cand_cap,
                        cudaStream_t s) {
  cudaMemsetAsync(counts_dev, 0, sizeof(PruneCounts), s);
  const uint64_t nt = (len + kTile - 1) / kTile;
  const uint64_t cap = (uint64_t)num_sms() * 6;
  prune_count_kernel<<<(unsigned)(nt < cap ? nt : cap), kThreads, 0, s>>>(w, len, win_dev,
                                                                        counts_dev, cand, cand_cap,
                                                                        nt);
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
                                                               hist);
  else
    prune_hist_kernel<false><<<(unsigned)blocks, 256, smem, s>>>(src, n, base, shift, nbits,
                                                                prefix, hist);
  note_launch();
}

void launch_prune_bitmap(const float* w, uint64_t len, uint32_t T, uint64_t r, uint64_t* words,
                         uint32_t* tile_popc, int* changed, uint64_t* ws_state, cudaStream_t s) {
  const uint64_t nt = (len + kTile - 1) / kTile;
  cudaMemsetAsync(ws_state, 0, nt * sizeof(uint64_t) + sizeof(unsigned), s);
  cudaMemsetAsync(changed, 0, sizeof(int), s);
  prune_bitmap_kernel<<<(unsigned)nt, kThreads, 0, s>>>(
      w, len, T, r, words, (len + 63) / 64, tile_popc, changed, ws_state,
      reinterpret_cast<unsigned*>(ws_state + nt));
  note_launch();
}

}  // namespace pactk
