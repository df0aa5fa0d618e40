// topk.cu -- TopK payload kernels.
//
// Reference: topk_select / topk_densify (codec.cpp:147-182) and the mean in
// topk_allgather_aggregate (collective.cpp:370-390). The selection itself
// reuses the prune machinery (radix select of the threshold + bitmap +
// tie fix-up with the lower-index-first tie rule, prune.cu); here are the
// payload kernels around it:
//  * pack_index: ascending indices of the selected bits (the values come
//    from pack_lm_kernel over the same mask);
//  * union_bits / scatter_add_slot / slot_mean: the per-index double
//    accumulator over ranks in rank order, then float(acc / n), kept only
//    for the union of the ranks' indices (the unpack kernel expands it);
//  * scatter_f32: topk_densify (zeros elsewhere, out-of-range -> error).
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

// warp per 1024-element chunk; lane l owns the 32-bit half l of the chunk's
// 16 words, so its indices are consecutive from chunk_off[c] + (excl scan).
__global__ void __launch_bounds__(256)
    pack_index_kernel(uint64_t len, const uint32_t* __restrict__ words32,
                      const uint32_t* __restrict__ chunk_off, uint32_t* __restrict__ idx,
                      uint64_t nchunks) {
  const int lane = threadIdx.x & 31;
  const uint64_t nhalves = 2 * ((len + 63) / 64);
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nw) {
    const uint64_t h = c * 32 + lane;
    uint32_t bits = h < nhalves ? words32[h] : 0u;
    const uint32_t cnt = __popc(bits);
    uint32_t pos = chunk_off[c] + warp_incl_scan(cnt) - cnt;
    const uint32_t base = (uint32_t)(h * 32);
    while (bits) {
      const int b = __ffs(bits) - 1;
      idx[pos++] = base + (uint32_t)b;
      bits &= bits - 1;
    }
  }
}

__global__ void scatter_f32_kernel(const uint32_t* __restrict__ idx, const float* __restrict__ val,
                                   uint64_t k, uint64_t len, float* __restrict__ out, int* __restrict__ err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k; j += stride) {
    const uint32_t i = idx[j];
    if (i >= len)
      atomicOr(err, 1);
    else
      out[i] = val[j];
  }
}

// ---- sparse accumulator over the union of the ranks' selections
// U = OR of every rank's index set (bit i of words[i >> 6]); validates ranges
__global__ void union_bits_kernel(const uint32_t* __restrict__ idx, uint64_t k, uint64_t len,
                                  unsigned long long* __restrict__ words, int* __restrict__ err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k; j += stride) {
    const uint32_t i = idx[j];
    if (i >= len) {
      atomicOr(err, 1);
      continue;
    }
    atomicOr(words + (i >> 6), 1ull << (i & 63));
  }
}

// slot of index i in U: kept elements of U before i (chunk offset + the
// popcounts of the chunk's earlier words and of word i>>6 below bit i)
__device__ __forceinline__ uint32_t union_slot(const uint64_t* __restrict__ words, const uint32_t* __restrict__ off,
                                               uint32_t i) {
  const uint32_t c = i >> 10, w = i >> 6;
  uint32_t s = off[c];
  for (uint32_t q = c << 4; q < w; ++q) s += __popcll(words[q]);
  return s + __popcll(words[w] & ((1ull << (i & 63)) - 1ull));
}

// acc[slot(i)] += (double)val -- one rank's list (indices unique), ranks in
// order on the stream: the reference's per-index double accumulation order
__global__ void scatter_add_slot_kernel(const uint32_t* __restrict__ idx, const float* __restrict__ val, uint64_t k,
                                        uint64_t len, const uint64_t* __restrict__ words,
                                        const uint32_t* __restrict__ off, double* __restrict__ acc) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k; j += stride) {
    const uint32_t i = idx[j];
    if (i < len) acc[union_slot(words, off, i)] += (double)val[j];
  }
}

// packed[s] = float(acc[s] / n) for s < |U| (= off[nchunks])
__global__ void slot_mean_kernel(const double* __restrict__ acc, const uint32_t* __restrict__ total, int n,
                                 float* __restrict__ packed) {
  const uint64_t m = *total, stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < m; s += stride)
    packed[s] = (float)(acc[s] / (double)n);
}

unsigned grid_of(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (unsigned)(g > 4736 ? 4736 : (g ? g : 1));
}

}  // namespace

void launch_pack_index(uint64_t len, const uint64_t* words, const uint32_t* chunk_off, uint32_t* idx,
                       cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  uint64_t grid = (nc * 32 + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  pack_index_kernel<<<(unsigned)grid, 256, 0, s>>>(len, reinterpret_cast<const uint32_t*>(words),
                                                   chunk_off, idx, nc);
  note_launch();
}

void launch_union_bits(const uint32_t* idx, uint64_t k, uint64_t len, uint64_t* words, int* err, cudaStream_t s) {
  if (!k) return;
  union_bits_kernel<<<grid_of(k), 256, 0, s>>>(idx, k, len, reinterpret_cast<unsigned long long*>(words), err);
  note_launch();
}

void launch_scatter_add_slot(const uint32_t* idx, const float* val, uint64_t k, uint64_t len, const uint64_t* words,
                             const uint32_t* off, double* acc, cudaStream_t s) {
  if (!k) return;
  scatter_add_slot_kernel<<<grid_of(k), 256, 0, s>>>(idx, val, k, len, words, off, acc);
  note_launch();
}

void launch_slot_mean(const double* acc, const uint32_t* total, uint64_t max_slots, int n, float* packed,
                      cudaStream_t s) {
  if (!max_slots) return;
  slot_mean_kernel<<<grid_of(max_slots), 256, 0, s>>>(acc, total, n, packed);
  note_launch();
}

void launch_scatter_f32(const uint32_t* idx, const float* val, uint64_t k, uint64_t len, float* out,
                        int* err, cudaStream_t s) {
  if (!k) return;
  scatter_f32_kernel<<<grid_of(k), 256, 0, s>>>(idx, val, k, len, out, err);
  note_launch();
}

}  // namespace pactk
