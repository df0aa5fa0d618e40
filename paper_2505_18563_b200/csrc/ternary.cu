// ternary.cu -- stochastic ternarization of the packed gradient and the
// decode-and-average of n ranks' ternary frames.
//
// Reference: ternarize / deternarize / sign_at (codec.cpp:40-75), the wire
// layout of the signs (codec.hpp:73-78: 2 bits per element, 00 = 0, 01 = +1,
// 10 = -1, 11 reserved, element i at byte i >> 2, bits 2 (i & 3)), the
// decode checks (codec.cpp:313-343) and the aggregation in
// ternary_allgather_aggregate (collective.cpp:311-368: per element a double
// accumulator over ranks in rank order, then float(acc / n)).
//
// The one deliberate difference: the reference draws u_i from a sequential
// mt19937_64 stream; here u_i is the i-th output of a SplitMix64 stream with
// the same seed (x_i = seed + (i + 1) * golden, output = mix(x_i)), so every
// element's draw is computed independently. The acceptance test is the
// reference's: unbiasedness within 3 standard errors (test_codec.cpp:109-125)
// and exact results whenever no draw matters (|g_i| in {0, max}).
//
// Layout on the device: signs are u32 words (16 elements each, the same
// bytes as the reference's sign bytes read little-endian); the per-rank
// block of the all-gather is [signs: W = ceil(count/16) u32][scale bits]
// [3 pad], stride W + 4 words (16-byte aligned blocks).
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:16-21 (splitmix64 finaliser)
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// max |v_i| as float bits (non-negative floats order like their bits); NaNs
// are skipped, as std::max(s, NaN) keeps s (codec.cpp:55)
__global__ void __launch_bounds__(256) absmax_kernel(const float* __restrict__ v, uint64_t n,
                                                     unsigned* __restrict__ out) {
  unsigned m = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (((uintptr_t)v) & 15) == 0;
  const uint64_t n4 = vec ? n / 4 : 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 x = ld_stream_f4(reinterpret_cast<const float4*>(v) + i);
    const unsigned a = __float_as_uint(x.x) & 0x7fffffffu, b = __float_as_uint(x.y) & 0x7fffffffu,
                   c = __float_as_uint(x.z) & 0x7fffffffu, d = __float_as_uint(x.w) & 0x7fffffffu;
    m = max(m, a <= 0x7f800000u ? a : 0u);
    m = max(m, b <= 0x7f800000u ? b : 0u);
    m = max(m, c <= 0x7f800000u ? c : 0u);
    m = max(m, d <= 0x7f800000u ? d : 0u);
  }
  for (uint64_t i = 4 * n4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned a = __float_as_uint(v[i]) & 0x7fffffffu;
    m = max(m, a <= 0x7f800000u ? a : 0u);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ unsigned wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, wm[w]);
    if (m) atomicMax(out, m);
  }
}

// thread per 16 elements -> one u32 of sign pairs (codec.cpp:58-64)
__global__ void __launch_bounds__(256)
    ternarize_kernel(const float* __restrict__ v, uint64_t n, const unsigned* __restrict__ smax,
                     uint64_t seed, uint32_t* __restrict__ signs, uint64_t nwords) {
  const float s = __uint_as_float(*smax);
  const double sd = (double)s;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    uint32_t out = 0;
    if (s != 0.0f) {
      const uint64_t i0 = w * 16;
#pragma unroll 4
      for (int j = 0; j < 16; ++j) {
        const uint64_t i = i0 + j;
        if (i >= n) break;
        const float g = v[i];
        const double keep_p = (double)fabsf(g) / sd;
        const double u = (double)(mix64(seed + (i + 1) * kGolden) >> 11) * 0x1.0p-53;
        if (u < keep_p) out |= (g > 0.0f ? 1u : 2u) << (2 * j);
      }
    }
    signs[w] = out;
  }
}

// mean over n rank blocks: out[i] = float((sum_r double(scale_r) * sign_r(i)) / n)
// (collective.cpp:355-360), with decode_ternary's checks (codec.cpp:324-340):
// err |= 1 reserved pattern 11, 2 sign bits past count, 4 bad scale,
// 8 zero scale with a non-zero sign
__global__ void __launch_bounds__(256)
    ternary_mean_kernel(const uint32_t* __restrict__ signs, uint64_t sign_stride,
                        const float* __restrict__ scales, uint64_t scale_stride, int n, uint64_t count,
                        float* __restrict__ out, int* __restrict__ err) {
  const uint64_t nwords = (count + 15) / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  int e = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    const uint64_t i0 = w * 16;
    const int valid = count - i0 >= 16 ? 16 : (int)(count - i0);
    for (int r = 0; r < n; ++r) {
      const float sc = scales[r * scale_stride];
      const uint32_t x = signs[r * sign_stride + w];
      if (!(sc >= 0.0f) || isinf(sc)) e |= 4;
      if (x & (x >> 1) & 0x55555555u) e |= 1;
      if (valid < 16 && (x >> (2 * valid))) e |= 2;
      if (sc == 0.0f && x) e |= 8;
      const double sd = (double)sc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t p = (x >> (2 * j)) & 3u;
        acc[j] += sd * (p == 1u ? 1.0 : (p == 2u ? -1.0 : 0.0));
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < valid) out[i0 + j] = (float)(acc[j] / (double)n);
  }
  if (e) atomicOr(err, e);
}

__global__ void div_kernel(float* __restrict__ x, uint64_t n, float d) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    x[i] = __fdiv_rn(x[i], d);
}

}  // namespace

void launch_div(float* x, uint64_t n, float d, cudaStream_t s) {
  if (!n) return;
  uint64_t grid = (n + 255) / 256;
  if (grid > 4736) grid = 4736;
  div_kernel<<<(unsigned)grid, 256, 0, s>>>(x, n, d);
  note_launch();
}

void launch_absmax(const float* v, uint64_t n, unsigned* out_bits, cudaStream_t s) {
  cudaMemsetAsync(out_bits, 0, 4, s);
  if (!n) return;
  uint64_t grid = (n / 4 + 255) / 256 + 1;
  if (grid > 1184) grid = 1184;
  absmax_kernel<<<(unsigned)grid, 256, 0, s>>>(v, n, out_bits);
  note_launch();
}

void launch_ternarize(const float* v, uint64_t n, const unsigned* smax_bits, uint64_t seed,
                      uint32_t* signs, cudaStream_t s) {
  const uint64_t nw = (n + 15) / 16;
  if (!nw) return;
  uint64_t grid = (nw + 255) / 256;
  if (grid > 4736) grid = 4736;
  ternarize_kernel<<<(unsigned)grid, 256, 0, s>>>(v, n, smax_bits, seed, signs, nw);
  note_launch();
}

void launch_ternary_mean(const uint32_t* signs, uint64_t sign_stride, const float* scales,
                         uint64_t scale_stride, int n, uint64_t count, float* out, int* err,
                         cudaStream_t s) {
  const uint64_t nw = (count + 15) / 16;
  if (!nw) return;
  uint64_t grid = (nw + 255) / 256;
  if (grid > 4736) grid = 4736;
  ternary_mean_kernel<<<(unsigned)grid, 256, 0, s>>>(signs, sign_stride, scales, scale_stride, n, count,
                                                     out, err);
  note_launch();
}

}  // namespace pactk
