// p2p.cu -- NVLink peer-memory allreduce of the packed gradient (the B200
// replacement of ring_allreduce on the packed path; reference:
// collective.cpp:165-216 and 269-309).
//
// Every rank owns one CUDA-IPC-exported "symmetric" buffer: a flag array that
// peers write into, its packed gradient and a reduced-chunk region (both
// double-buffered by step parity). With the reference's ChunkMap(M, n)
// (C = ceil(M/n)) every element of chunk c is folded in the reference's order
// (((x_c + x_{c+1}) + ...) + x_{c-1}), so the result is BIT-IDENTICAL to the
// reference ring for every n (NCCL's order is unspecified; the reference ring
// is order-free only at n = 2).
//
//   one-shot (n == 2): every rank folds all M values, pulling the peer's
//     packed buffer over NVLink (M remote reads per rank, one barrier).
//   two-shot (n > 2): rank c folds chunk c (reduce-scatter by pulls), then
//     every rank pulls the other reduced chunks from their owners
//     (all-gather); 2(n-1)/n * M remote reads per rank, two barriers.
// Pulls, not pushes: measured on this pool (tools/nvlink_probe.cu) peer
// float4 loads reach 741 GB/s, aligned float4 stores 696 GB/s, but stores at
// an arbitrary 4-byte offset (compacted runs) only 413 GB/s. All streams are
// 16-byte aligned float4 at the same index in source and destination, with
// several loads in flight per thread; remote reads use ld.global.cg (no stale
// L1 lines across steps).
//
// Ordering: producer kernels complete; a 1-warp signal kernel fences at
// system scope and stores the step number into every peer's flag slot with
// st.release.sys; consumers spin on their local flags with ld.acquire.sys,
// bounded by a 10 s globaltimer timeout that raises a device error flag
// instead of hanging.
#include "common.cuh"
#include "launch.h"
#include "p2p_sync.cuh"

namespace pactk {

namespace {

using namespace p2psync;

__global__ void p2p_signal_kernel(P2PView v, int kind, uint64_t value) {
  const int lane = threadIdx.x;
  __threadfence_system();
  if (lane < v.n) st_release_sys(v.flags[lane] + kind * kP2PMaxRanks + v.rank, value);
}

__global__ void p2p_wait_kernel(const uint64_t* flags, int kind, int n, uint64_t target, P2PErr* err) {
  block_wait_flags(flags, kind, n, target, err);
}

__device__ __forceinline__ float4 ldcg4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}

// fold element i of chunk c: ((x_c + x_{c+1}) + ...) + x_{c-1}
__device__ __forceinline__ float fold1(const P2PView& v, uint32_t c, uint64_t i) {
  float acc = __ldcg(v.packed[c] + i);
  for (int s = 1; s < v.n; ++s) {
    int r = (int)c + s;
    if (r >= v.n) r -= v.n;
    acc = __fadd_rn(acc, __ldcg(v.packed[r] + i));
  }
  return acc;
}

// Fold packed[*][b, e) into out[b, e), reference order per element. A float4
// inside one chunk folds as a vector; chunk-straddling vectors and ragged
// ends go element by element.
__device__ void fold_range(const P2PView& v, float* __restrict__ out, uint64_t b, uint64_t e) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t vb = (b + 3) & ~3ull, ve = e & ~3ull;
  if (vb >= ve) {
    for (uint64_t i = b + gt; i < e; i += stride) out[i] = fold1(v, (uint32_t)(i / v.C), i);
    return;
  }
  for (uint64_t i = b + gt; i < vb; i += stride) out[i] = fold1(v, (uint32_t)(i / v.C), i);
  for (uint64_t i = ve + gt; i < e; i += stride) out[i] = fold1(v, (uint32_t)(i / v.C), i);
  constexpr int kU = 2;  // float4 per thread per iteration, x n sources in flight
  const uint64_t qe = ve / 4;
  for (uint64_t q = vb / 4 + gt; q < qe; q += stride * kU) {
    float4 acc[kU];
    uint32_t c0[kU];
    bool same[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t qq = q + u * stride;
      same[u] = false;
      c0[u] = 0;
      if (qq >= qe) continue;
      const uint64_t i = 4 * qq;
      c0[u] = (uint32_t)(i / v.C);
      same[u] = (uint32_t)((i + 3) / v.C) == c0[u];
      if (same[u]) acc[u] = ldcg4(v.packed[c0[u]] + i);
    }
#pragma unroll
    for (int s = 1; s < kP2PMaxRanks; ++s) {
      if (s >= v.n) break;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!same[u]) continue;
        int r = (int)c0[u] + s;
        if (r >= v.n) r -= v.n;
        const float4 x = ldcg4(v.packed[r] + 4 * (q + u * stride));
        acc[u].x = __fadd_rn(acc[u].x, x.x);
        acc[u].y = __fadd_rn(acc[u].y, x.y);
        acc[u].z = __fadd_rn(acc[u].z, x.z);
        acc[u].w = __fadd_rn(acc[u].w, x.w);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t qq = q + u * stride;
      if (qq >= qe) continue;
      const uint64_t i = 4 * qq;
      if (same[u]) {
        *reinterpret_cast<float4*>(out + i) = acc[u];
      } else {
        for (int k = 0; k < 4; ++k) out[i + k] = fold1(v, (uint32_t)((i + k) / v.C), i + k);
      }
    }
  }
}

// one-shot (whole vector) or the owner's chunk (two-shot reduce-scatter)
__global__ void __launch_bounds__(256)
    p2p_fold_kernel(P2PView v, float* __restrict__ out, uint64_t b, uint64_t e, const uint64_t* flags,
                    uint64_t target, P2PErr* err, P2PSig sg) {
  entry_signal(v, sg);  // this rank's packed buffer is complete (the producer ran before)
  if (!block_wait_flags(flags, kP2PPacked, v.n, target, err)) return;
  fold_range(v, out, b, e);
  exit_signal(v, sg);
}

// two-shot all-gather of [b, e): out[j] = reduced[owner(j)][j] (same
// absolute index), owner(j) = (j - P0) / Cb (the bucket's ownership split;
// the fold ORDER always follows the global ChunkMap, so buckets stay exact)
__device__ void gather_range(const P2PView& v, float* __restrict__ out, uint64_t b, uint64_t e,
                             uint64_t P0, uint64_t Cb);

__global__ void __launch_bounds__(256)
    p2p_gather_kernel(P2PView v, float* __restrict__ out, uint64_t b, uint64_t e, uint64_t P0,
                      uint64_t Cb, const uint64_t* flags, uint64_t target, P2PErr* err, P2PSig sg) {
  entry_signal(v, sg);
  if (!block_wait_flags(flags, kP2PReduced, v.n, target, err)) return;
  gather_range(v, out, b, e, P0, Cb);
  exit_signal(v, sg);
}

__device__ void gather_range(const P2PView& v, float* __restrict__ out, uint64_t b, uint64_t e,
                             uint64_t P0, uint64_t Cb) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t vb = (b + 3) & ~3ull, ve = e & ~3ull;
  auto one = [&](uint64_t i) { out[i] = __ldcg(v.reduced[(i - P0) / Cb] + i); };
  if (vb >= ve) {
    for (uint64_t i = b + gt; i < e; i += stride) one(i);
    return;
  }
  for (uint64_t i = b + gt; i < vb; i += stride) one(i);
  for (uint64_t i = ve + gt; i < e; i += stride) one(i);
  const uint64_t qe = ve / 4;
  for (uint64_t q = vb / 4 + gt; q < qe; q += 2 * stride) {
    float4 x[2];
    bool ok[2], same[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t qq = q + u * stride;
      ok[u] = qq < qe;
      same[u] = false;
      if (!ok[u]) continue;
      const uint64_t i = 4 * qq;
      const uint64_t c = (i - P0) / Cb;
      same[u] = (i + 3 - P0) / Cb == c;
      if (same[u]) x[u] = ldcg4(v.reduced[c] + i);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      const uint64_t i = 4 * (q + u * stride);
      if (same[u])
        *reinterpret_cast<float4*>(out + i) = x[u];
      else
        for (int k = 0; k < 4; ++k) one(i + k);
    }
  }
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

unsigned stream_grid(uint64_t elems, int max_ctas) {
  // consumers spin at entry: keep every CTA resident (<= 8 x 256 per SM), and
  // at most max_ctas when the exchange overlaps pack/unpack on other streams
  uint64_t blocks = (elems / 4 + 255) / 256;
  uint64_t cap = (uint64_t)sms() * 8;
  if (max_ctas > 0 && (uint64_t)max_ctas < cap) cap = (uint64_t)max_ctas;
  if (blocks > cap) blocks = cap;
  return (unsigned)(blocks ? blocks : 1);
}

}  // namespace

void launch_p2p_signal(const P2PView& v, int kind, uint64_t value, cudaStream_t s) {
  p2p_signal_kernel<<<1, 32, 0, s>>>(v, kind, value);
  note_launch();
}

void launch_p2p_wait(const uint64_t* flags, int kind, int n, uint64_t target, P2PErr* err,
                     cudaStream_t s) {
  p2p_wait_kernel<<<1, 32, 0, s>>>(flags, kind, n, target, err);
  note_launch();
}

void launch_p2p_fold(const P2PView& v, float* out, uint64_t b, uint64_t e, const uint64_t* flags,
                     uint64_t target, P2PErr* err, int max_ctas, const P2PSig& sg, cudaStream_t s) {
  p2p_fold_kernel<<<stream_grid(e > b ? e - b : 0, max_ctas), 256, 0, s>>>(v, out, b, e, flags,
                                                                          target, err, sg);
  note_launch();
}

void launch_p2p_gather(const P2PView& v, float* out, uint64_t b, uint64_t e, uint64_t P0, uint64_t Cb,
                       const uint64_t* flags, uint64_t target, P2PErr* err, int max_ctas,
                       const P2PSig& sg, cudaStream_t s) {
  p2p_gather_kernel<<<stream_grid(e > b ? e - b : 0, max_ctas), 256, 0, s>>>(v, out, b, e, P0, Cb,
                                                                            flags, target, err, sg);
  note_launch();
}

}  // namespace pactk
