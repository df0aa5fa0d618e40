// synth.cu -- synthetic weights / gradients.
//
// x[i] = recipe(splitmix64(seed ^ (index_base + i))) * scale with integer
// hashing (rng.hpp:15-20) and round-to-nearest int->float conversions only,
// so the host twin (paper_2505_18563_b200/synth.py) reproduces every bit.
//   0 W-ties   : ((m >> 40) - 2^23) * 2^-23          24-bit grid, many ties
//   1 W-real   : (int32)(m >> 32) * 2^-31            31-bit, few ties
//   2 G-dyadic : ((m % (2^21+1)) - 2^20) * 2^-20     sums of <= 8 exact
//   3 G-full   : ((m >> 39) - 2^24) * 2^-24          partial sums round
#include "common.cuh"
#include "launch.h"

namespace pactk {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <int kRecipe>
__device__ __forceinline__ float synth_one(uint64_t m, float scale) {
  float v;
  if (kRecipe == 0) {
    v = __fmul_rn(__int2float_rn((int)(m >> 40) - (1 << 23)), 0x1p-23f);
  } else if (kRecipe == 1) {
    v = __fmul_rn(__int2float_rn((int)(uint32_t)(m >> 32)), 0x1p-31f);
  } else if (kRecipe == 2) {
    v = __fmul_rn(__int2float_rn((int)(m % ((1ull << 21) + 1)) - (1 << 20)), 0x1p-20f);
  } else {
    v = __fmul_rn(__int2float_rn((int)(m >> 39) - (1 << 24)), 0x1p-24f);
  }
  return __fmul_rn(v, scale);
}

template <int kRecipe>
__global__ void __launch_bounds__(256)
    synth_kernel(float* __restrict__ x, uint64_t len, uint64_t seed, uint64_t base, float scale) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += stride)
    x[i] = synth_one<kRecipe>(splitmix64(seed ^ (base + i)), scale);
}

}  // namespace

void launch_synth(float* x, uint64_t len, uint64_t seed, uint64_t index_base, int recipe,
                  float scale, cudaStream_t s) {
  if (!len) return;
  uint64_t blocks = (len + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  switch (recipe) {
    case 0: synth_kernel<0><<<(unsigned)blocks, 256, 0, s>>>(x, len, seed, index_base, scale); break;
    case 1: synth_kernel<1><<<(unsigned)blocks, 256, 0, s>>>(x, len, seed, index_base, scale); break;
    case 2: synth_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(x, len, seed, index_base, scale); break;
    default: synth_kernel<3><<<(unsigned)blocks, 256, 0, s>>>(x, len, seed, index_base, scale); break;
  }
  note_launch();
}

}  // namespace pactk
