// codec.cu -- mask-indexed stream compaction (pack), scatter-expand (unpack,
// optionally fused with to_mean and the masked SGD step), GSE, and the
// mask bookkeeping kernels (fill, tile popcounts, exclusive scan).
//
// Reference semantics: codec.cpp:14-38 (pack/unpack), sparsity.cpp:112-119
// (GSE), trainer.cpp:202-214 and 268-273 (to_mean + sgd_step), tensor.cpp
// 83-129 (mask layout, nnz).
//
// Layout: the gradient is split into 4096-element tiles (64 mask words). A
// mask carries tile_off[t] = kept elements before tile t, so every tile's
// packed range is known up front and tiles are independent: pack/unpack are
// one streaming pass with no inter-CTA communication. Each thread owns four
// float4 slots of the tile (coalesced 128-bit accesses), reads its 4-bit mask
// nibble per slot and skips the load entirely when the nibble is zero (pack
// and GSE only fetch the 32-byte sectors that hold kept values). Compacted
// values are staged in shared memory and written out as one contiguous,
// coalesced run per tile.
#include <cstdio>

#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

unsigned long long g_launches = 0;

int grid_for(uint64_t tiles, int per_sm) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const uint64_t cap = (uint64_t)sms * per_sm;
  return (int)(tiles < cap ? tiles : cap);
}

// ------------------------------------------------------------------ pack
__global__ void __launch_bounds__(kThreads, 6)
    pack_kernel(const float* __restrict__ g, uint64_t len, const uint64_t* __restrict__ words,
                uint64_t nwords, const uint32_t* __restrict__ tile_off, float* __restrict__ packed,
                uint64_t tb, uint64_t te) {
  __shared__ uint64_t sw[kTileWords];
  __shared__ uint32_t wpre[kTileWords + 1];
  __shared__ float stage[kTile];
  const int tid = threadIdx.x;
  const bool vec_ok = (((uintptr_t)g) & 15) == 0;
  for (uint64_t t = tb + blockIdx.x; t < te; t += gridDim.x) {
    load_tile_words(words, nwords, t, sw, wpre);
    const uint64_t e0 = t * (uint64_t)kTile;
    float4 v[kVecPerThread];
    uint32_t nib[kVecPerThread];
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const int e = (j * kThreads + tid) * 4;
      nib[j] = nibble_at(sw, e);
      v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (nib[j]) {
        const uint64_t ge = e0 + e;
        if (vec_ok && ge + 4 <= len) {
          v[j] = ld_stream_f4(reinterpret_cast<const float4*>(g + ge));
        } else {  // unaligned base or ragged tail: only kept (hence in-range) lanes
          if (nib[j] & 1) v[j].x = g[ge];
          if (nib[j] & 2) v[j].y = g[ge + 1];
          if (nib[j] & 4) v[j].z = g[ge + 2];
          if (nib[j] & 8) v[j].w = g[ge + 3];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      if (!nib[j]) continue;
      const int e = (j * kThreads + tid) * 4;
      uint32_t pos = rank_before(sw, wpre, e);
      if (nib[j] & 1) stage[pos++] = v[j].x;
      if (nib[j] & 2) stage[pos++] = v[j].y;
      if (nib[j] & 4) stage[pos++] = v[j].z;
      if (nib[j] & 8) stage[pos++] = v[j].w;
    }
    __syncthreads();
    const uint32_t cnt = wpre[kTileWords];
    float* dst = packed + tile_off[t];
    for (uint32_t i = tid; i < cnt; i += kThreads) dst[i] = stage[i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- unpack
// kSgd: fused to_mean (scale) + masked SGD on weights; grad_out optional.
template <bool kSgd>
__global__ void __launch_bounds__(kThreads, 8)
    unpack_kernel(const float* __restrict__ packed, uint64_t len, const uint64_t* __restrict__ words,
                  uint64_t nwords, const uint32_t* __restrict__ tile_off, float scale, int do_scale,
                  float* __restrict__ out, float lr, float* __restrict__ weights, uint64_t tb,
                  uint64_t te) {
  __shared__ uint64_t sw[kTileWords];
  __shared__ uint32_t wpre[kTileWords + 1];
  __shared__ float stage[kTile];
  const int tid = threadIdx.x;
  const bool vec_ok = ((((uintptr_t)out) | (kSgd ? (uintptr_t)weights : 0)) & 15) == 0;
  for (uint64_t t = tb + blockIdx.x; t < te; t += gridDim.x) {
    load_tile_words(words, nwords, t, sw, wpre);
    const uint32_t cnt = wpre[kTileWords];
    const float* src = packed + tile_off[t];
    for (uint32_t i = tid; i < cnt; i += kThreads) stage[i] = src[i];
    __syncthreads();
    const uint64_t e0 = t * (uint64_t)kTile;
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const int e = (j * kThreads + tid) * 4;
      const uint64_t ge = e0 + e;
      if (ge >= len) continue;
      const uint32_t nib = nibble_at(sw, e);
      uint32_t pos = nib ? rank_before(sw, wpre, e) : 0;
      float o[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (nib & (1u << b)) {
          const float x = stage[pos++];
          o[b] = do_scale ? __fmul_rn(x, scale) : x;
        } else {
          o[b] = 0.0f;
        }
      }
      const bool full = vec_ok && ge + 4 <= len;
      if (!kSgd || out != nullptr) {
        if (full) {
          st_stream_f4(reinterpret_cast<float4*>(out + ge), make_float4(o[0], o[1], o[2], o[3]));
        } else {
          for (int b = 0; b < 4 && ge + b < len; ++b) out[ge + b] = o[b];
        }
      }
      if (kSgd) {
        float p[4];
        if (full) {
          const float4 w4 = *reinterpret_cast<const float4*>(weights + ge);
          p[0] = w4.x, p[1] = w4.y, p[2] = w4.z, p[3] = w4.w;
        } else {
          for (int b = 0; b < 4; ++b) p[b] = ge + b < len ? weights[ge + b] : 0.f;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b)  // trainer.cpp:208-212, no FMA contraction
          p[b] = (nib & (1u << b)) ? __fsub_rn(p[b], __fmul_rn(lr, o[b])) : 0.0f;
        if (full) {
          *reinterpret_cast<float4*>(weights + ge) = make_float4(p[0], p[1], p[2], p[3]);
        } else {
          for (int b = 0; b < 4 && ge + b < len; ++b) weights[ge + b] = p[b];
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------- GSE
__global__ void __launch_bounds__(kThreads, 8)
    gse_kernel(const float* g, uint64_t len, const uint64_t* __restrict__ words, uint64_t nwords,
               float* out, uint64_t ntiles) {  // out may alias g (in-place GSE)
  __shared__ uint64_t sw[kTileWords];
  const int tid = threadIdx.x;
  const bool vec_ok = ((((uintptr_t)g) | ((uintptr_t)out)) & 15) == 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (tid < kTileWords) {
      const uint64_t wi = t * kTileWords + tid;
      sw[tid] = wi < nwords ? __ldg(words + wi) : 0ull;
    }
    __syncthreads();
    const uint64_t e0 = t * (uint64_t)kTile;
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const int e = (j * kThreads + tid) * 4;
      const uint64_t ge = e0 + e;
      if (ge >= len) continue;
      const uint32_t nib = nibble_at(sw, e);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vec_ok && ge + 4 <= len) {
        if (nib) {
          v = ld_stream_f4(reinterpret_cast<const float4*>(g + ge));
          if (!(nib & 1)) v.x = 0.f;
          if (!(nib & 2)) v.y = 0.f;
          if (!(nib & 4)) v.z = 0.f;
          if (!(nib & 8)) v.w = 0.f;
        }
        st_stream_f4(reinterpret_cast<float4*>(out + ge), v);
      } else {
        for (int b = 0; b < 4 && ge + b < len; ++b) out[ge + b] = (nib >> b) & 1 ? g[ge + b] : 0.0f;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- mask bookkeeping
__global__ void mask_fill_kernel(uint64_t* words, uint64_t nwords, uint64_t len, int keep,
                                 uint32_t* tile_off, uint64_t ntiles) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nwords; i += stride) {
    uint64_t w = keep ? ~0ull : 0ull;
    if (keep && i == nwords - 1 && (len & 63)) w = (1ull << (len & 63)) - 1ull;
    words[i] = w;
  }
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= ntiles; t += stride) {
    const uint64_t e = t * (uint64_t)kTile;
    tile_off[t] = keep ? (uint32_t)(e < len ? e : len) : 0u;
  }
}

__global__ void clear_tail_kernel(uint64_t* words, uint64_t len) {
  const uint64_t last = (len - 1) >> 6;
  words[last] &= (1ull << (len & 63)) - 1ull;
}

// one warp per tile: popcount of its 64 words
__global__ void tile_popc_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                                 uint32_t* __restrict__ tile_popc, uint64_t ntiles) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ntiles) return;
  const uint64_t w0 = warp * kTileWords + 2 * lane;
  uint32_t c = 0;
  if (w0 < nwords) c += __popcll(words[w0]);
  if (w0 + 1 < nwords) c += __popcll(words[w0 + 1]);
  c = warp_sum(c);
  if (lane == 0) tile_popc[warp] = c;
}

// single-CTA exclusive scan, 1024 threads x 8 items per chunk
__global__ void __launch_bounds__(1024) scan_excl_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                         uint32_t* __restrict__ out) {
  __shared__ uint32_t warp_tot[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t carry = 0;
  for (uint64_t base = 0; base < n; base += 8192) {
    uint32_t v[8];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t idx = base + (uint64_t)tid * 8 + i;
      v[i] = idx < n ? in[idx] : 0u;
      s += v[i];
    }
    const uint32_t inc = warp_incl_scan(s);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = warp_tot[lane];
      const uint32_t xi = warp_incl_scan(x);
      warp_tot[lane] = xi - x;
      if (lane == 31) warp_tot[32] = xi;
    }
    __syncthreads();
    uint32_t run = carry + warp_tot[warp] + inc - s;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t idx = base + (uint64_t)tid * 8 + i;
      if (idx < n) out[idx] = run;
      run += v[i];
    }
    carry += warp_tot[32];
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
}

// out[i] = in[i] * scale (dense-fallback epilogue of to_mean, trainer.cpp:268-273)
__global__ void __launch_bounds__(256) scale_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    uint64_t len, float scale) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += stride)
    out[i] = __fmul_rn(in[i], scale);
}

}  // namespace

uint64_t launches() { return g_launches; }
void note_launch(uint64_t n) { g_launches += n; }

void launch_pack(const float* g, uint64_t len, const uint64_t* words, const uint32_t* tile_off,
                 float* packed, uint64_t tb, uint64_t te, cudaStream_t s) {
  if (te <= tb) return;
  pack_kernel<<<grid_for(te - tb, 8), kThreads, 0, s>>>(g, len, words, (len + 63) / 64, tile_off,
                                                        packed, tb, te);
  note_launch();
}

void launch_unpack(const float* packed, uint64_t len, const uint64_t* words,
                   const uint32_t* tile_off, float scale, int do_scale, float* out, uint64_t tb,
                   uint64_t te, cudaStream_t s) {
  if (te <= tb) return;
  unpack_kernel<false><<<grid_for(te - tb, 8), kThreads, 0, s>>>(
      packed, len, words, (len + 63) / 64, tile_off, scale, do_scale, out, 0.f, nullptr, tb, te);
  note_launch();
}

void launch_unpack_sgd(const float* packed, uint64_t len, const uint64_t* words,
                       const uint32_t* tile_off, float scale, int do_scale, float lr,
                       float* grad_out, float* weights, cudaStream_t s) {
  const uint64_t nt = (len + kTile - 1) / kTile;
  if (!nt) return;
  unpack_kernel<true><<<grid_for(nt, 8), kThreads, 0, s>>>(packed, len, words, (len + 63) / 64,
                                                           tile_off, scale, do_scale, grad_out, lr,
                                                           weights, 0, nt);
  note_launch();
}

void launch_gse(const float* g, uint64_t len, const uint64_t* words, float* out, cudaStream_t s) {
  const uint64_t nt = (len + kTile - 1) / kTile;
  if (!nt) return;
  gse_kernel<<<grid_for(nt, 8), kThreads, 0, s>>>(g, len, words, (len + 63) / 64, out, nt);
  note_launch();
}

void launch_mask_fill(uint64_t* words, uint64_t len, int keep, uint32_t* tile_off, cudaStream_t s) {
  const uint64_t nw = (len + 63) / 64, nt = (len + kTile - 1) / kTile;
  const uint64_t work = nw > nt + 1 ? nw : nt + 1;
  int grid = (int)((work + 255) / 256);
  if (grid > 4096) grid = 4096;
  mask_fill_kernel<<<grid, 256, 0, s>>>(words, nw, len, keep, tile_off, nt);
  note_launch();
}

void launch_clear_tail(uint64_t* words, uint64_t len, cudaStream_t s) {
  if (!len || !(len & 63)) return;
  clear_tail_kernel<<<1, 1, 0, s>>>(words, len);
  note_launch();
}

void launch_tile_popc(const uint64_t* words, uint64_t len, uint32_t* tile_popc, cudaStream_t s) {
  const uint64_t nt = (len + kTile - 1) / kTile;
  if (!nt) return;
  tile_popc_kernel<<<(unsigned)((nt * 32 + 255) / 256), 256, 0, s>>>(words, (len + 63) / 64,
                                                                    tile_popc, nt);
  note_launch();
}

void launch_scan_excl(const uint32_t* in, uint64_t n, uint32_t* out, cudaStream_t s) {
  scan_excl_kernel<<<1, 1024, 0, s>>>(in, n, out);
  note_launch();
}

void launch_scale(const float* in, float* out, uint64_t len, float scale, cudaStream_t s) {
  if (!len) return;
  uint64_t blocks = (len + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  scale_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, len, scale);
  note_launch();
}

}  // namespace pactk
