// digest.cu -- exact FNV-1a-64 of a mask on the GPU (reference:
// tensor.cpp:11-19 fnv1a64 over the little-endian word bytes, 122-128).
//
// FNV-1a is a serial chain h <- (h ^ b) * P mod 2^64. Two facts make it
// parallel without changing a bit of the result:
//  (1) h ^ b only touches the low byte s of h, and the low byte of a product
//      only depends on the low bytes of its factors, so the sequence of low
//      bytes is a 256-state automaton  s <- ((s ^ b) * 0xb3) & 0xff  (0xb3 =
//      P mod 256). Each 2 KiB segment's transition map (256 entries) is
//      computed independently; composing the maps yields every segment's
//      true starting low byte.
//  (2) With the low-byte trajectory fixed, h ^ b == h + d(s, b), so a segment
//      is the affine map h -> P^L * h + (g_L - s0 * P^L), where g_L is the
//      FNV chain of the segment started from the value s0 itself. Affine maps
//      compose associatively, so the per-segment results fold in a tree.
// Work: 256 x bytes automaton steps (2 states per thread in 16-bit lanes)
// plus one ordinary FNV pass; computed only when a mask changes.
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr int kSegWords = 256;  // 2 KiB of mask bytes per segment
constexpr int kGroup = 128;     // segments per group

__host__ __device__ inline uint64_t pow_p(uint64_t e) {
  uint64_t r = 1, b = kFnvPrime;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

struct Affine {
  uint64_t a, c;
};
// apply f first, then g
__device__ inline Affine compose(Affine f, Affine g) { return {g.a * f.a, g.a * f.c + g.c}; }

// (A) per-segment low-byte transition maps, two states per thread
__global__ void __launch_bounds__(128)
    digest_maps_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                       uint8_t* __restrict__ maps) {
  __shared__ uint64_t sw[kSegWords];
  const uint64_t seg = blockIdx.x;
  const uint64_t w0 = seg * kSegWords;
  const int nw = (int)min((uint64_t)kSegWords, nwords - w0);
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sw[i] = words[w0 + i];
  __syncthreads();
  const uint32_t s0 = 2 * threadIdx.x, s1 = s0 + 1;
  uint32_t x = s0 | (s1 << 16);
  for (int i = 0; i < nw; ++i) {
    const uint64_t wv = sw[i];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t by = (uint32_t)(wv >> (8 * b)) & 0xffu;
      x = ((x ^ (by * 0x10001u)) * 0xb3u) & 0x00ff00ffu;
    }
  }
  maps[seg * 256 + s0] = (uint8_t)(x & 0xff);
  maps[seg * 256 + s1] = (uint8_t)(x >> 16);
}

// (B) compose the maps of each group of kGroup segments
__global__ void __launch_bounds__(256)
    digest_group_kernel(const uint8_t* __restrict__ maps, uint64_t nseg, uint8_t* __restrict__ gmaps) {
  __shared__ uint8_t sm[kGroup * 256];
  const uint64_t g = blockIdx.x;
  const uint64_t s_begin = g * kGroup;
  const int ns = (int)min((uint64_t)kGroup, nseg - s_begin);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(maps + s_begin * 256);
  uint32_t* dst = reinterpret_cast<uint32_t*>(sm);
  for (int i = threadIdx.x; i < ns * 64; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  uint32_t st = threadIdx.x;
  for (int j = 0; j < ns; ++j) st = sm[j * 256 + st];
  gmaps[g * 256 + threadIdx.x] = (uint8_t)st;
}

// (C) sequential walk over the group maps -> true start low byte per group
__global__ void digest_group_starts_kernel(const uint8_t* __restrict__ gmaps, uint64_t ngroups,
                                           uint8_t* __restrict__ gstart) {
  extern __shared__ uint8_t sg[];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(gmaps);
  uint32_t* dst = reinterpret_cast<uint32_t*>(sg);
  for (uint64_t i = threadIdx.x; i < ngroups * 64; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t st = (uint32_t)(kFnvBasis & 0xff);
    for (uint64_t g = 0; g < ngroups; ++g) {
      gstart[g] = (uint8_t)st;
      st = sg[g * 256 + st];
    }
  }
}

// (D) per group: segment start bytes, per-segment chain from s0, affine fold
__global__ void __launch_bounds__(kGroup)
    digest_affine_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                         const uint8_t* __restrict__ maps, uint64_t nseg,
                         const uint8_t* __restrict__ gstart, uint64_t p_full, uint64_t p_last,
                         Affine* __restrict__ gaff) {
  __shared__ uint8_t sm[kGroup * 256];
  __shared__ uint8_t s_start[kGroup];
  __shared__ Affine s_aff[kGroup];
  const uint64_t g = blockIdx.x;
  const uint64_t s_begin = g * kGroup;
  const int ns = (int)min((uint64_t)kGroup, nseg - s_begin);
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(maps + s_begin * 256);
    uint32_t* dst = reinterpret_cast<uint32_t*>(sm);
    for (int i = threadIdx.x; i < ns * 64; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t st = gstart[g];
    for (int j = 0; j < ns; ++j) {
      s_start[j] = (uint8_t)st;
      st = sm[j * 256 + st];
    }
  }
  __syncthreads();
  const int j = threadIdx.x;
  Affine a{1, 0};
  if (j < ns) {
    const uint64_t seg = s_begin + j;
    const uint64_t w0 = seg * kSegWords;
    const int nw = (int)min((uint64_t)kSegWords, nwords - w0);
    const uint64_t s0 = s_start[j];
    uint64_t h = s0;
    for (int i = 0; i < nw; ++i) {
      const uint64_t wv = __ldg(words + w0 + i);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        h ^= (wv >> (8 * b)) & 0xffu;
        h *= kFnvPrime;
      }
    }
    const uint64_t A = (nw == kSegWords) ? p_full : p_last;
    a = {A, h - s0 * A};
  }
  s_aff[j] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    Affine acc{1, 0};
    for (int q = 0; q < ns; ++q) acc = compose(acc, s_aff[q]);
    gaff[g] = acc;
  }
}

// (E) fold the group affines starting from the offset basis
__global__ void digest_final_kernel(const Affine* __restrict__ gaff, uint64_t ngroups,
                                    uint64_t* __restrict__ out) {
  uint64_t h = kFnvBasis;
  for (uint64_t g = 0; g < ngroups; ++g) h = gaff[g].a * h + gaff[g].c;
  *out = h;
}

}  // namespace

size_t digest_scratch_bytes(uint64_t nwords) {
  const uint64_t nseg = (nwords + kSegWords - 1) / kSegWords;
  const uint64_t ng = (nseg + kGroup - 1) / kGroup;
  return nseg * 256 + ng * 256 + ng + 16 + ng * sizeof(Affine) + 64;
}

void launch_digest(const uint64_t* words, uint64_t nwords, void* scratch, uint64_t* out_dev,
                   cudaStream_t s) {
  if (nwords == 0) {  // fnv1a64 of zero bytes is the offset basis
    const uint64_t basis = kFnvBasis;
    cudaMemcpyAsync(out_dev, &basis, 8, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    return;
  }
  const uint64_t nseg = (nwords + kSegWords - 1) / kSegWords;
  const uint64_t ng = (nseg + kGroup - 1) / kGroup;
  uint8_t* maps = static_cast<uint8_t*>(scratch);
  uint8_t* gmaps = maps + nseg * 256;
  uint8_t* gstart = gmaps + ng * 256;
  uintptr_t ap = reinterpret_cast<uintptr_t>(gstart + ng);
  ap = (ap + 15) & ~uintptr_t(15);
  Affine* gaff = reinterpret_cast<Affine*>(ap);
  const uint64_t last_words = nwords - (nseg - 1) * kSegWords;
  digest_maps_kernel<<<(unsigned)nseg, 128, 0, s>>>(words, nwords, maps);
  digest_group_kernel<<<(unsigned)ng, 256, 0, s>>>(maps, nseg, gmaps);
  const size_t smem = ng * 256;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(digest_group_starts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  digest_group_starts_kernel<<<1, 256, smem, s>>>(gmaps, ng, gstart);
  digest_affine_kernel<<<(unsigned)ng, kGroup, 0, s>>>(words, nwords, maps, nseg, gstart,
                                                       pow_p(8ull * kSegWords),
                                                       pow_p(8ull * last_words), gaff);
  digest_final_kernel<<<1, 1, 0, s>>>(gaff, ng, out_dev);
  note_launch(5);
}

}  // namespace pactk
