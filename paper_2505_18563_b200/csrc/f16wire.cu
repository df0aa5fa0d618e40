// f16wire.cu -- binary16 wire for the ring all-reduce.
//
// Reference: float_to_half / half_to_float (codec.cpp:77-140: hand-rolled
// round-to-nearest-even, overflow and +-Inf clamp to +-65504, NaN -> signed
// quiet NaN 0x7e00, subnormals rounded RNE), fp16_roundtrip (codec.cpp:
// 142-146) and F16Wire (collective.cpp:133-163): every ring hop re-rounds
// the partial sum to binary16 before it leaves, the receiver adds it to its
// own fp32 value, and the chunk owner rounds the final sum once more so the
// all-gather copies identical bits. The conversions here are the same bit
// manipulations, not the hardware cvt (whose overflow goes to Inf).
//
// Kernels: seed (first hop: encode own chunk), step (p = x + decode(recv);
// encode p), gather (decode the owners' final chunks into the output).
#include <cuda_fp16.h>

#include "common.cuh"
#include "launch.h"

namespace pactk {

__device__ __forceinline__ uint16_t f2h_ref(float v) {  // codec.cpp:79-111
  const uint32_t bits = __float_as_uint(v);
  const uint32_t sign = (bits >> 16) & 0x8000u;
  const int32_t exp = (int32_t)((bits >> 23) & 0xffu) - 127;
  uint32_t mant = bits & 0x7fffffu;
  if (exp == 128) return (uint16_t)(sign | (mant ? 0x7e00u : 0x7bffu));
  if (exp > 15) return (uint16_t)(sign | 0x7bffu);
  if (exp >= -14) {
    uint32_t m = mant >> 13;
    const uint32_t rest = mant & 0x1fffu;
    if (rest > 0x1000u || (rest == 0x1000u && (m & 1u))) ++m;
    const uint32_t h = ((uint32_t)(exp + 15) << 10) + m;
    return (uint16_t)(sign | (h >= 0x7c00u ? 0x7bffu : h));
  }
  if (exp >= -25) {
    mant |= 0x800000u;
    const int shift = -exp - 14 + 13;  // 14..24
    uint32_t m = mant >> shift;
    const uint32_t cut = mant & ((1u << shift) - 1u);
    const uint32_t half_ulp = 1u << (shift - 1);
    if (cut > half_ulp || (cut == half_ulp && (m & 1u))) ++m;
    return (uint16_t)(sign | m);
  }
  return (uint16_t)sign;
}

__device__ __forceinline__ float h2f_ref(uint16_t h) {  // codec.cpp:113-140
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1fu;
  const uint32_t mant = h & 0x3ffu;
  uint32_t bits;
  if (exp == 0) {
    if (mant == 0) {
      bits = sign;
    } else {  // subnormal: normalise (leading-zero count instead of the loop)
      const int lz = __clz(mant) - 21;  // shifts until bit 10 is set
      const uint32_t m = mant << lz;
      bits = sign | ((uint32_t)(1 - lz + 112) << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (mant << 13);
  } else {
    bits = sign | ((exp + 112) << 23) | (mant << 13);
  }
  return __uint_as_float(bits);
}

namespace {

__global__ void f16_encode_kernel(const float* __restrict__ x, uint64_t n, uint16_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = f2h_ref(x[i]);
}

// p = x + decode(recv) (F16Wire::accumulate: chunk[i] += decode_one), then
// the next hop's payload encode(p) -- or, on the last hop, the owner's
// prepare_owned rounding (the same encode)
__global__ void f16_step_kernel(const float* __restrict__ x, const uint16_t* __restrict__ recv, uint64_t n,
                                uint16_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = f2h_ref(__fadd_rn(x[i], h2f_ref(recv[i])));
}

// out[j] = decode(gathered[owner(c)][j - begin(c)]), owner(c) = c - 1 mod n
// (position p ends the reduce-scatter owning chunk p + 1)
__global__ void f16_gather_kernel(const uint16_t* __restrict__ gathered, uint64_t count, int n, uint64_t C,
                                  float* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count; j += stride) {
    const uint64_t c = j / C;
    const int owner = (int)((c + n - 1) % n);
    out[j] = h2f_ref(gathered[(uint64_t)owner * C + (j - c * C)]);
  }
}

__global__ void f16_roundtrip_kernel(const float* __restrict__ x, uint64_t n, float* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = h2f_ref(f2h_ref(x[i]));
}

unsigned grid_of(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (unsigned)(g > 4736 ? 4736 : (g ? g : 1));
}

}  // namespace

void launch_f16_encode(const float* x, uint64_t n, uint16_t* out, cudaStream_t s) {
  if (!n) return;
  f16_encode_kernel<<<grid_of(n), 256, 0, s>>>(x, n, out);
  note_launch();
}
void launch_f16_step(const float* x, const uint16_t* recv, uint64_t n, uint16_t* out, cudaStream_t s) {
  if (!n) return;
  f16_step_kernel<<<grid_of(n), 256, 0, s>>>(x, recv, n, out);
  note_launch();
}
void launch_f16_gather(const uint16_t* gathered, uint64_t count, int n, uint64_t C, float* out,
                       cudaStream_t s) {
  if (!count) return;
  f16_gather_kernel<<<grid_of(count), 256, 0, s>>>(gathered, count, n, C, out);
  note_launch();
}
void launch_f16_roundtrip(const float* x, uint64_t n, float* out, cudaStream_t s) {
  if (!n) return;
  f16_roundtrip_kernel<<<grid_of(n), 256, 0, s>>>(x, n, out);
  note_launch();
}

}  // namespace pactk
