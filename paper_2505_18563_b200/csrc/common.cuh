// common.cuh -- device helpers shared by the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pactk {

constexpr int kTile = 4096;            // elements per mask tile (= PACT_TILE)
constexpr int kTileWords = kTile / 64; // 64 words
constexpr int kThreads = 256;          // CTA size of the streaming kernels
constexpr int kVecPerThread = kTile / (4 * kThreads);  // 4 float4 per thread

// |w| ordering of finite floats == unsigned ordering of bits & 0x7fffffff
// (+0.0 and -0.0 tie, as fabs does). sparsity.cpp:48-54.
__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7fffffffu; }

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// streaming (evict-first) 128-bit load: the dense gradient is touched once
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream_f4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float f4_get(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// 4-bit slice of the tile mask covering elements [e, e+4) (e multiple of 4)
__device__ __forceinline__ uint32_t nibble_at(const uint64_t* sw, int e) {
  return (uint32_t)(sw[e >> 6] >> (e & 63)) & 0xFu;
}
// kept elements of the tile strictly before element e
__device__ __forceinline__ uint32_t rank_before(const uint64_t* sw, const uint32_t* wpre, int e) {
  const uint64_t below = (e & 63) ? (sw[e >> 6] & ((1ull << (e & 63)) - 1ull)) : 0ull;
  return wpre[e >> 6] + (uint32_t)__popcll(below);
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan for kThreads threads; returns exclusive prefix,
// *total receives the block total. scratch: >= kThreads/32 + 1 elements.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* scratch, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nw = kThreads / 32;
  T inc = warp_incl_scan(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < nw ? scratch[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) scratch[lane] = si - s;
    if (lane == nw - 1) scratch[nw] = si;
  }
  __syncthreads();
  T r = scratch[warp] + inc - v;
  *total = scratch[nw];
  __syncthreads();
  return r;
}

// Load the 64 words of tile t and their exclusive popcount prefix into smem.
// Must be called by all threads; ends with a barrier.
__device__ __forceinline__ void load_tile_words(const uint64_t* __restrict__ words, uint64_t nwords,
                                                uint64_t t, uint64_t* sw, uint32_t* wpre) {
  const int tid = threadIdx.x;
  if (tid < kTileWords) {
    const uint64_t wi = t * kTileWords + tid;
    sw[tid] = wi < nwords ? __ldg(words + wi) : 0ull;
  }
  __syncthreads();
  if (tid < 32) {
    const uint32_t c0 = __popcll(sw[2 * tid]), c1 = __popcll(sw[2 * tid + 1]);
    const uint32_t s = c0 + c1;
    const uint32_t inc = warp_incl_scan(s);
    wpre[2 * tid] = inc - s;
    wpre[2 * tid + 1] = inc - s + c0;
    if (tid == 31) wpre[64] = inc;
  }
  __syncthreads();
}

}  // namespace pactk
