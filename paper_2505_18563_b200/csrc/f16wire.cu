// f16wire.cu -- binary16 wire for the ring all-reduce.
//
// Reference: float_to_half / half_to_float (codec.cpp:77-140: hand-rolled
// round-to-nearest-even, overflow and +-Inf clamp to +-65504, NaN -> signed
// quiet NaN 0x7e00, subnormals rounded RNE), fp16_roundtrip (codec.cpp:
// 142-146) and F16Wire (collective.cpp:133-163): every ring hop re-rounds
// the partial sum to binary16 before it leaves, the receiver adds it to its
// own fp32 value, and the chunk owner rounds the final sum once more so the
// all-gather copies identical bits. The conversions use the hardware cvt
// (cvt.rn.f16.f32 / cvt.f32.f16) with the reference's special-value rules
// patched on top (overflow clamps instead of going to Inf, NaN canonical).
//
// Kernels: seed (first hop: encode own chunk), step (p = x + decode(recv);
// encode p), gather (decode the owners' final chunks into the output).
#include <cuda_fp16.h>

#include "common.cuh"
#include "launch.h"

namespace pactk {

// The reference's conversions (codec.cpp:79-140) are RNE with three
// departures from IEEE, so the hardware cvt does the rounding (normals and
// subnormals alike: RNE at 2^-24 granularity, flush below 2^-25 to signed
// zero, exactly as codec.cpp:100-110's shift-and-round) and only the
// specials are patched: overflow (a rounded result >= 0x7c00, including
// +-Inf inputs) clamps to +-65504 (codec.cpp:86-88, 96), NaN becomes the
// input-signed quiet NaN 0x7e00 (codec.cpp:85).
__device__ __forceinline__ uint16_t f2h_ref(float v) {
  const uint16_t sign = (uint16_t)((__float_as_uint(v) >> 16) & 0x8000u);
  uint16_t h = __half_as_ushort(__float2half_rn(v));
  if ((h & 0x7fffu) >= 0x7c00u) h = sign | ((v != v) ? 0x7e00u : 0x7bffu);
  return h;
}

// Every binary16 value is exactly representable in fp32, so the hardware cvt
// is the reference's decode (codec.cpp:113-140) except for NaN payloads,
// which the reference carries through (mant << 13) and the cvt canonicalises.
__device__ __forceinline__ float h2f_ref(uint16_t h) {
  if ((h & 0x7c00u) == 0x7c00u)
    return __uint_as_float(((uint32_t)(h & 0x8000u) << 16) | 0x7f800000u | ((uint32_t)(h & 0x3ffu) << 13));
  return __half2float(__ushort_as_half(h));
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
