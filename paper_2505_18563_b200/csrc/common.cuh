// common.cuh -- device helpers shared by the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pactk {

// Host-side launcher caches (occupancy grids, dynamic-smem opt-ins) are per
// DEVICE: one process may drive several GPUs (thread per GPU), and
// cudaFuncSetAttribute applies to the current device's context only.
template <typename T>
struct DeviceCache {
  T v[64] = {};
  T& get() {
    int d = 0;
    cudaGetDevice(&d);
    return v[d & 63];
  }
};

// Offset granularity of a mask: one warp work unit of pack/unpack.
constexpr int kChunk = 1024;             // elements (= PACT_TILE)
constexpr int kChunkWords = kChunk / 64; // 16 words
constexpr int kVecPerLane = kChunk / (4 * 32);  // 8 float4 per lane

// CTA tile of the prune kernels (4 chunks).
constexpr int kTile = 4096;
constexpr int kTileWords = kTile / 64;
constexpr int kThreads = 256;
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

// streaming (evict-first) 128-bit accesses: the dense gradient is touched once
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
__device__ __forceinline__ uint64_t ld_nc_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
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

// A warp's view of one 1024-element chunk: lane l < 16 holds word l and its
// exclusive popcount prefix; lane l's j-th float4 slot covers elements
// 128*j + 4*l .. +3, i.e. nibble 4*(l&15) of word 2*j + (l>>4).
struct ChunkMask {
  uint64_t w;      // lane's own word (lanes 0..15)
  uint32_t excl;   // exclusive prefix of popcounts (lanes 0..15)
  uint32_t total;  // kept elements in the chunk (all lanes)
};

__device__ __forceinline__ ChunkMask load_chunk_mask(const uint64_t* __restrict__ words,
                                                     uint64_t nwords, uint64_t c) {
  const int lane = threadIdx.x & 31;
  ChunkMask m;
  const uint64_t wi = c * kChunkWords + lane;
  m.w = (lane < kChunkWords && wi < nwords) ? ld_nc_u64(words + wi) : 0ull;
  const uint32_t pc = (uint32_t)__popcll(m.w);
  const uint32_t inc = warp_incl_scan(pc);
  m.excl = inc - pc;
  m.total = __shfl_sync(0xffffffffu, inc, 31);
  return m;
}

// nibble and in-chunk rank of lane's slot j
__device__ __forceinline__ void slot_of(const ChunkMask& m, int j, uint32_t& nib, uint32_t& pos) {
  const int lane = threadIdx.x & 31;
  const int wi = 2 * j + (lane >> 4);
  const uint64_t w = __shfl_sync(0xffffffffu, m.w, wi);
  const uint32_t ex = __shfl_sync(0xffffffffu, m.excl, wi);
  const int sh = 4 * (lane & 15);
  nib = (uint32_t)(w >> sh) & 0xFu;
  pos = ex + (uint32_t)__popcll(sh ? (w & ((1ull << sh) - 1ull)) : 0ull);
}

}  // namespace pactk
