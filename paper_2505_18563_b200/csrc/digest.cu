// digest.cu -- exact FNV-1a-64 of a mask on the GPU (reference:
// tensor.cpp:11-19 fnv1a64 over the little-endian word bytes, 122-128).
//
// FNV-1a is a serial chain h <- (h ^ b) * P mod 2^64 (P = 0x100000001b3).
// Three facts make it parallel without changing a bit of the result:
//  (1) h ^ b only touches the low byte s of h, and the low byte of a product
//      only depends on the low bytes of its factors, so the low-byte sequence
//      is an automaton s <- ((s ^ b) * 0xb3) & 0xff driven by the bytes.
//  (2) That automaton is triangular: the low nibble t of s evolves on its own,
//      t <- ((t ^ b_lo) * 3) & 15 (0xb3 = 3 mod 16), and once the low-nibble
//      trajectory is known the high nibble u evolves as
//      u <- ((u ^ b_hi) * 3 + K) & 15 with K = ((t ^ b_lo) * 0xb3 >> 4) & 15.
//      So a segment's transition needs two 16-entry maps (low nibble, then
//      high nibble given the true low-nibble start), not one 256-entry map:
//      32 automaton states per byte instead of 256.
//  (3) With the low-byte trajectory fixed, h ^ b == h + d(s, b), so a segment
//      is the affine map h -> P^L * h + (g_L - s0 * P^L), g_L = the FNV chain
//      of the segment started from the value s0; affine maps compose.
// Each thread owns a 128-byte segment, a CTA a tile of 256 segments. Three
// kernels, one per fact; each composes its per-thread maps into a tile map
// (warp shuffles + 8 warp totals) and the last CTA to finish scans the tile
// maps (the classic last-block pattern), so a digest is 3 kernels and a
// 16-byte memset. Maps are held "byte form": 16 bytes in a uint4, byte i =
// image of input i; four inputs are advanced per 32-bit ALU op (8-bit lanes,
// values < 64, no carries between lanes) and maps compose with byte_perm.
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr int kDThreads = 256;             // segments per tile
constexpr int kSegWords = 16;              // 128 bytes per segment (thread)
constexpr int kTileWordsD = kDThreads * kSegWords;

__host__ __device__ inline uint64_t pow_p(uint64_t e) {
  uint64_t r = 1, b = kFnvPrime;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

struct Aff {
  uint64_t a, c;
};
// apply f first, then g
__device__ __forceinline__ Aff aff_compose(Aff f, Aff g) { return {g.a * f.a, g.a * f.c + g.c}; }

__device__ __forceinline__ uint4 map_identity() {
  return make_uint4(0x03020100u, 0x07060504u, 0x0b0a0908u, 0x0f0e0d0cu);
}
// four 4-bit indices (bytes of fb) looked up in the 16-byte table g
__device__ __forceinline__ uint32_t lut4(uint32_t fb, const uint4& g) {
  uint32_t s = fb & 0x07070707u;
  s = (s | (s >> 4)) & 0x00ff00ffu;
  s = (s | (s >> 8)) & 0x0000ffffu;
  const uint32_t lo = __byte_perm(g.x, g.y, s), hi = __byte_perm(g.z, g.w, s);
  const uint32_t m = ((fb >> 3) & 0x01010101u) * 0xffu;
  return (lo & ~m) | (hi & m);
}
// apply f first, then g
__device__ __forceinline__ uint4 map_compose(const uint4& f, const uint4& g) {
  return make_uint4(lut4(f.x, g), lut4(f.y, g), lut4(f.z, g), lut4(f.w, g));
}
__device__ __forceinline__ uint32_t map_apply(const uint4& f, uint32_t v) {
  const uint32_t r = v < 8 ? (v < 4 ? f.x : f.y) : (v < 12 ? f.z : f.w);
  return (r >> (8 * (v & 3))) & 0xffu;
}
__device__ __forceinline__ uint4 shfl_up4(const uint4& v, int o) {
  return make_uint4(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o),
                    __shfl_up_sync(0xffffffffu, v.z, o), __shfl_up_sync(0xffffffffu, v.w, o));
}
__device__ __forceinline__ uint4 warp_scan_map(uint4 m) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint4 y = shfl_up4(m, o);
    if (lane >= o) m = map_compose(y, m);
  }
  return m;
}
__device__ __forceinline__ Aff warp_scan_aff(Aff m) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Aff y{__shfl_up_sync(0xffffffffu, m.a, o), __shfl_up_sync(0xffffffffu, m.c, o)};
    if (lane >= o) m = aff_compose(y, m);
  }
  return m;
}

// Tile-level: returns this thread's incoming value given the tile's incoming
// value `tin` (thread 0's), and writes the tile map (all 256 composed) to
// *tile_map when tile_map != null. sh: 8 maps + 8 values of shared scratch.
struct MapScratch {
  uint4 warp_tot[kDThreads / 32];
  uint32_t warp_in[kDThreads / 32];
};
__device__ __forceinline__ uint4 tile_reduce_map(uint4 m, MapScratch& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint4 inc = warp_scan_map(m);
  if (lane == 31) sh.warp_tot[warp] = inc;
  __syncthreads();
  uint4 agg = sh.warp_tot[0];
  if (threadIdx.x == 0)
    for (int w = 1; w < kDThreads / 32; ++w) agg = map_compose(agg, sh.warp_tot[w]);
  __syncthreads();
  return agg;  // valid in thread 0
}
__device__ __forceinline__ uint32_t tile_scan_map(uint4 m, uint32_t tin, MapScratch& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint4 inc = warp_scan_map(m);
  if (lane == 31) sh.warp_tot[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t v = tin;
    for (int w = 0; w < kDThreads / 32; ++w) {
      sh.warp_in[w] = v;
      v = map_apply(sh.warp_tot[w], v);
    }
  }
  __syncthreads();
  const uint4 ex = shfl_up4(inc, 1);
  const uint32_t win = sh.warp_in[warp];
  const uint32_t r = lane == 0 ? win : map_apply(ex, win);
  __syncthreads();
  return r;
}

__device__ __forceinline__ bool last_block(unsigned* cnt) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}
__device__ __forceinline__ uint4 ldcg4(const uint4* p) { return __ldcg(p); }

// last CTA: incoming value of every tile from the tile maps (in order)
__device__ void scan_tiles(const uint4* tile_map, uint32_t* tile_in, uint32_t ntiles, uint32_t start,
                           MapScratch& sh) {
  const uint32_t q = (ntiles + kDThreads - 1) / kDThreads;
  const uint32_t t0 = threadIdx.x * q, t1 = min(ntiles, t0 + q);
  uint4 m = map_identity();
  for (uint32_t t = t0; t < t1; ++t) m = map_compose(m, ldcg4(tile_map + t));
  uint32_t v = tile_scan_map(m, start, sh);
  for (uint32_t t = t0; t < t1; ++t) {
    tile_in[t] = v;
    v = map_apply(ldcg4(tile_map + t), v);
  }
}

// the thread's whole segment in registers before the serial chain: 8
// independent 16-byte loads in flight instead of one 8-byte load per step
struct SegRegs {
  uint2 w[kSegWords];
};
__device__ __forceinline__ void load_seg(const uint64_t* __restrict__ words, uint64_t seg, int nw, SegRegs& r) {
  const uint64_t* src = words + seg * kSegWords;
  if (nw == kSegWords) {
#pragma unroll
    for (int i = 0; i < kSegWords / 2; ++i) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + i);
      r.w[2 * i] = make_uint2(v.x, v.y);
      r.w[2 * i + 1] = make_uint2(v.z, v.w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSegWords; ++i)
      r.w[i] = i < nw ? __ldg(reinterpret_cast<const uint2*>(src) + i) : make_uint2(0u, 0u);
  }
}

__device__ __forceinline__ int seg_words(uint64_t nwords, uint64_t seg) {
  const uint64_t w0 = seg * kSegWords;
  return w0 >= nwords ? 0 : (int)min((uint64_t)kSegWords, nwords - w0);
}

// (1) low-nibble maps of every segment; tile maps; last CTA: tile starts
__global__ void __launch_bounds__(kDThreads)
    digest_low_kernel(const uint64_t* __restrict__ words, uint64_t nwords, uint4* __restrict__ seg_low,
                      uint4* __restrict__ tile_low, uint32_t* __restrict__ tile_tin, unsigned* cnt) {
  __shared__ MapScratch sh;
  const uint64_t seg = (uint64_t)blockIdx.x * kDThreads + threadIdx.x;
  const int nw = seg_words(nwords, seg);
  SegRegs sr;
  load_seg(words, seg, nw, sr);
  uint4 x = map_identity();
#pragma unroll
  for (int i = 0; i < kSegWords; ++i) {
    if (i >= nw) break;
    const uint2 wv = sr.w[i];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w32 = h ? wv.y : wv.x;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t B = __byte_perm(w32, 0u, b * 0x1111u) & 0x0f0f0f0fu;
        x.x = ((x.x & 0x0f0f0f0fu) ^ B) * 3u;
        x.y = ((x.y & 0x0f0f0f0fu) ^ B) * 3u;
        x.z = ((x.z & 0x0f0f0f0fu) ^ B) * 3u;
        x.w = ((x.w & 0x0f0f0f0fu) ^ B) * 3u;
      }
    }
  }
  x = make_uint4(x.x & 0x0f0f0f0fu, x.y & 0x0f0f0f0fu, x.z & 0x0f0f0f0fu, x.w & 0x0f0f0f0fu);
  seg_low[seg] = x;
  const uint4 agg = tile_reduce_map(x, sh);
  if (threadIdx.x == 0) tile_low[blockIdx.x] = agg;
  if (last_block(cnt)) {
    scan_tiles(tile_low, tile_tin, gridDim.x, (uint32_t)(kFnvBasis & 0xf), sh);
    if (threadIdx.x == 0) *cnt = 0;
  }
}

// (2) each segment's true low-nibble start, then its high-nibble map
__global__ void __launch_bounds__(kDThreads)
    digest_high_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                       const uint4* __restrict__ seg_low, const uint32_t* __restrict__ tile_tin,
                       uint4* __restrict__ seg_high, uint8_t* __restrict__ seg_tin,
                       uint4* __restrict__ tile_high, uint32_t* __restrict__ tile_hin, unsigned* cnt) {
  __shared__ MapScratch sh;
  const uint64_t seg = (uint64_t)blockIdx.x * kDThreads + threadIdx.x;
  const int nw = seg_words(nwords, seg);
  const uint32_t tin = tile_scan_map(seg_low[seg], tile_tin[blockIdx.x], sh);
  seg_tin[seg] = (uint8_t)tin;
  SegRegs sr;
  load_seg(words, seg, nw, sr);
  uint4 x = map_identity();
  uint32_t t = tin;
#pragma unroll
  for (int i = 0; i < kSegWords; ++i) {
    if (i >= nw) break;
    const uint2 wv = sr.w[i];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w32 = h ? wv.y : wv.x;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t by = (w32 >> (8 * b)) & 0xffu;
        const uint32_t p = (t ^ (by & 0xfu)) * 0xb3u;
        t = p & 0xfu;
        const uint32_t K = ((p >> 4) & 0xfu) * 0x01010101u;
        const uint32_t B = (__byte_perm(w32, 0u, b * 0x1111u) >> 4) & 0x0f0f0f0fu;
        x.x = ((x.x & 0x0f0f0f0fu) ^ B) * 3u + K;
        x.y = ((x.y & 0x0f0f0f0fu) ^ B) * 3u + K;
        x.z = ((x.z & 0x0f0f0f0fu) ^ B) * 3u + K;
        x.w = ((x.w & 0x0f0f0f0fu) ^ B) * 3u + K;
      }
    }
  }
  x = make_uint4(x.x & 0x0f0f0f0fu, x.y & 0x0f0f0f0fu, x.z & 0x0f0f0f0fu, x.w & 0x0f0f0f0fu);
  seg_high[seg] = x;
  const uint4 agg = tile_reduce_map(x, sh);
  if (threadIdx.x == 0) tile_high[blockIdx.x] = agg;
  if (last_block(cnt)) {
    scan_tiles(tile_high, tile_hin, gridDim.x, (uint32_t)((kFnvBasis >> 4) & 0xf), sh);
    if (threadIdx.x == 0) *cnt = 0;
  }
}

// (3) each segment's true start byte, its affine map; last CTA folds them
__global__ void __launch_bounds__(kDThreads)
    digest_affine_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                         const uint4* __restrict__ seg_high, const uint8_t* __restrict__ seg_tin,
                         const uint32_t* __restrict__ tile_hin, Aff* __restrict__ tile_aff,
                         uint64_t p_full, unsigned* cnt, uint64_t* __restrict__ out) {
  __shared__ MapScratch sh;
  __shared__ Aff warp_aff[kDThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t seg = (uint64_t)blockIdx.x * kDThreads + threadIdx.x;
  const int nw = seg_words(nwords, seg);
  const uint32_t hin = tile_scan_map(seg_high[seg], tile_hin[blockIdx.x], sh);
  const uint64_t s0 = (uint64_t)((hin << 4) | seg_tin[seg]);
  SegRegs sr;
  load_seg(words, seg, nw, sr);
  uint64_t h = s0;
#pragma unroll
  for (int i = 0; i < kSegWords; ++i) {
    if (i >= nw) break;
    const uint2 wv = sr.w[i];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      h ^= ((b < 4 ? wv.x : wv.y) >> (8 * (b & 3))) & 0xffu;
      h *= kFnvPrime;
    }
  }
  const uint64_t A = nw == kSegWords ? p_full : pow_p(8ull * (uint64_t)nw);
  Aff a{A, h - s0 * A};
  a = warp_scan_aff(a);
  if (lane == 31) warp_aff[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    Aff t = warp_aff[0];
    for (int w = 1; w < kDThreads / 32; ++w) t = aff_compose(t, warp_aff[w]);
    tile_aff[blockIdx.x] = t;
  }
  if (last_block(cnt)) {
    const uint32_t nt = gridDim.x;
    const uint32_t q = (nt + kDThreads - 1) / kDThreads;
    const uint32_t t0 = threadIdx.x * q, t1 = min(nt, t0 + q);
    Aff m{1, 0};
    for (uint32_t t = t0; t < t1; ++t) {
      const Aff y{__ldcg(&tile_aff[t].a), __ldcg(&tile_aff[t].c)};
      m = aff_compose(m, y);
    }
    m = warp_scan_aff(m);
    __syncthreads();
    if (lane == 31) warp_aff[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      Aff t = warp_aff[0];
      for (int w = 1; w < kDThreads / 32; ++w) t = aff_compose(t, warp_aff[w]);
      *out = t.a * kFnvBasis + t.c;
      *cnt = 0;
    }
  }
}

struct DigestLayout {
  uint64_t ntiles, nseg;
  size_t o_tile_low, o_tile_high, o_tile_aff, o_tile_tin, o_tile_hin, o_seg_low, o_seg_high, o_seg_tin,
      total;
};
DigestLayout digest_layout(uint64_t nwords) {
  DigestLayout L{};
  L.ntiles = (nwords + kTileWordsD - 1) / kTileWordsD;
  L.nseg = L.ntiles * kDThreads;
  size_t o = 64;  // counters
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o = (o + bytes + 63) & ~size_t(63);
    return r;
  };
  L.o_tile_low = take(L.ntiles * 16);
  L.o_tile_high = take(L.ntiles * 16);
  L.o_tile_aff = take(L.ntiles * sizeof(Aff));
  L.o_tile_tin = take(L.ntiles * 4);
  L.o_tile_hin = take(L.ntiles * 4);
  L.o_seg_low = take(L.nseg * 16);
  L.o_seg_high = take(L.nseg * 16);
  L.o_seg_tin = take(L.nseg);
  L.total = o;
  return L;
}

}  // namespace

size_t digest_scratch_bytes(uint64_t nwords) { return digest_layout(nwords).total; }

void launch_digest(const uint64_t* words, uint64_t nwords, void* scratch, uint64_t* out_dev,
                   cudaStream_t s) {
  if (nwords == 0) {  // fnv1a64 of zero bytes is the offset basis
    static const uint64_t basis = kFnvBasis;
    cudaMemcpyAsync(out_dev, &basis, 8, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    return;
  }
  const DigestLayout L = digest_layout(nwords);
  char* b = static_cast<char*>(scratch);
  unsigned* cnt = reinterpret_cast<unsigned*>(b);
  auto u4 = [&](size_t o) { return reinterpret_cast<uint4*>(b + o); };
  auto u32p = [&](size_t o) { return reinterpret_cast<uint32_t*>(b + o); };
  cudaMemsetAsync(cnt, 0, 16, s);
  const unsigned grid = (unsigned)L.ntiles;
  digest_low_kernel<<<grid, kDThreads, 0, s>>>(words, nwords, u4(L.o_seg_low), u4(L.o_tile_low),
                                               u32p(L.o_tile_tin), cnt);
  digest_high_kernel<<<grid, kDThreads, 0, s>>>(words, nwords, u4(L.o_seg_low), u32p(L.o_tile_tin),
                                                u4(L.o_seg_high),
                                                reinterpret_cast<uint8_t*>(b + L.o_seg_tin),
                                                u4(L.o_tile_high), u32p(L.o_tile_hin), cnt + 1);
  digest_affine_kernel<<<grid, kDThreads, 0, s>>>(
      words, nwords, u4(L.o_seg_high), reinterpret_cast<const uint8_t*>(b + L.o_seg_tin),
      u32p(L.o_tile_hin), reinterpret_cast<Aff*>(b + L.o_tile_aff), pow_p(8ull * kSegWords), cnt + 2,
      out_dev);
  note_launch(3);
}

}  // namespace pactk
