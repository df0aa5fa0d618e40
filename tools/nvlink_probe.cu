// nvlink_probe.cu -- measure GPU0 <-> GPU1 peer-memory access patterns
// (design evidence for p2p.cu). Single process, peer access enabled.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                     \
      return 1;                                                           \
    }                                                                     \
  } while (0)

__global__ void rd4(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
}
__global__ void wr4(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void wr1(const float* __restrict__ src, float* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
// 4 consecutive floats per thread as scalar stores (strided warp instructions)
__global__ void wr1x4(const float* __restrict__ src, float* __restrict__ dst, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    dst[4 * i] = v.x;
    dst[4 * i + 1] = v.y;
    dst[4 * i + 2] = v.z;
    dst[4 * i + 3] = v.w;
  }
}
// contiguous 4-byte stores at a +1 element misalignment (runs of arbitrary offset)
__global__ void wr1_off(const float* __restrict__ src, float* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i + 1] = src[i];
}

// one-shot fold pattern of p2p.cu: out = local + remote (float4)
__global__ void fold2(const float4* __restrict__ loc, const float4* __restrict__ rem, float4* __restrict__ out,
                      size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = __ldcg(loc + i), b = __ldcg(rem + i);
    out[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
}

// smem-staged bulk copy / bulk reduce-add to a (peer) global buffer: 4 KiB
// per warp-iteration, issued by lane 0 (the n = 2 reduce-push candidate)
// one-way push of `seg` floats per bulk op (each warp: load a segment into
// smem, bulk-copy it to the peer at the same offset; two smem slots so a
// segment's copy drains while the next one loads -- the pack's pattern)
__global__ void bulk_push_seg(const float* __restrict__ src, float* __restrict__ dst, size_t n, int seg) {
  __shared__ __align__(128) float st[4][2][1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int slot = 0;
  for (size_t c = (size_t)blockIdx.x * 4 + warp; c * seg < n; c += (size_t)gridDim.x * 4) {
    float* b = st[warp][slot];
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    for (int i = lane; i < seg / 4; i += 32)
      reinterpret_cast<float4*>(b)[i] = reinterpret_cast<const float4*>(src + c * seg)[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(b);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                   " cp.async.bulk.commit_group;" ::"l"(dst + c * seg), "r"(sa), "r"(seg * 4) : "memory");
    }
    slot ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <bool kReduce>
__global__ void bulk_push(const float* __restrict__ src, float* __restrict__ dst, size_t n) {
  __shared__ __align__(128) float st[8][1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* b = st[warp];
  for (size_t c = (size_t)blockIdx.x * 8 + warp; c * 1024 < n; c += (size_t)gridDim.x * 8) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    for (int i = lane; i < 256; i += 32)
      reinterpret_cast<float4*>(b)[i] = reinterpret_cast<const float4*>(src + c * 1024)[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(b);
      if (kReduce)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 4096;\n"
                     " cp.async.bulk.commit_group;" ::"l"(dst + c * 1024), "r"(sa) : "memory");
      else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;\n"
                     " cp.async.bulk.commit_group;" ::"l"(dst + c * 1024), "r"(sa) : "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 1;
  }
  const size_t bytes = 256ull << 20, n = bytes / 4;
  float *a0, *b0, *a1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&a1, bytes + 64));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes + 64));
  CK(cudaMalloc(&b0, bytes + 64));
  CK(cudaMemset(a0, 1, bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8, blk = 256;
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-44s %8.1f GB/s  (%.1f us for %zu MB)\n", name, bytes / (best * 1e-3) / 1e9, best * 1e3,
           bytes >> 20);
  };
  run("local copy float4 (HBM r+w, r counted)", [&] { rd4<<<grid, blk>>>((float4*)a0, (float4*)b0, n / 4); });
  run("remote READ float4 ld.cg  (GPU1 -> GPU0)", [&] { rd4<<<grid, blk>>>((float4*)a1, (float4*)b0, n / 4); });
  run("remote WRITE float4        (GPU0 -> GPU1)", [&] { wr4<<<grid, blk>>>((float4*)a0, (float4*)a1, n / 4); });
  run("remote WRITE f32 coalesced (GPU0 -> GPU1)", [&] { wr1<<<grid, blk>>>(a0, a1, n); });
  // one-way bulk pushes by op size (the pack pushes ~400-byte runs)
  for (int seg : {100, 256, 1024})
    for (int g : {148 * 4, 148 * 6}) {
      char nm[96];
      snprintf(nm, sizeof nm, "bulk push %5d B ops, %d CTAs x 4 warps", seg * 4, g);
      run(nm, [&] { bulk_push_seg<<<g, 128>>>(a0, a1, n, seg); });
    }
  // how few SMs saturate a one-way NVLink push (float4 stores, 256 MB)
  for (int g : {8, 16, 32, 64})
    for (int per : {1, 4}) {
      char nm[96];
      snprintf(nm, sizeof nm, "remote WRITE float4, %d SMs x %d CTAs", g, per);
      run(nm, [&] { wr4<<<g * per, 1024 / per, 0>>>((float4*)a0, (float4*)a1, n / 4); });
    }
  run("remote WRITE f32 x4/thread strided", [&] { wr1x4<<<grid, blk>>>(a0, a1, n / 4); });
  run("remote WRITE f32 coalesced, +4B offset", [&] { wr1_off<<<grid, blk>>>(a0, a1, n); });
  run("cudaMemcpyPeer GPU0 -> GPU1", [&] { cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes); });
  run("fold local+remote -> local (remote bytes)", [&] { fold2<<<grid, blk>>>((float4*)a0, (float4*)a1, (float4*)b0, n / 4); });
  for (size_t mb : {4, 20, 64}) {
    const size_t nn = (mb << 20) / 16;
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0);
      fold2<<<grid, blk>>>((float4*)a0, (float4*)a1, (float4*)b0, nn);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    float best_r = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0);
      rd4<<<grid, blk>>>((float4*)a1, (float4*)b0, nn);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best_r = ms < best_r ? ms : best_r;
    }
    printf("%3zu MB: fold %7.1f us (%6.1f GB/s remote), remote read %7.1f us (%6.1f GB/s)\n", mb, best * 1e3,
           (mb << 20) / (best * 1e-3) / 1e9, best_r * 1e3, (mb << 20) / (best_r * 1e-3) / 1e9);
  }
  // both GPUs fold at once (each reads the other: the one-shot exchange)
  {
    float *b1, *o1;
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaMalloc(&b1, bytes + 64));
    CK(cudaMalloc(&o1, bytes + 64));
    cudaStream_t s0, s1;
    cudaEvent_t f0, f1, g0, g1;
    cudaStreamCreate(&s1);
    cudaEventCreate(&f1);
    cudaEventCreate(&g1);
    CK(cudaSetDevice(0));
    cudaStreamCreate(&s0);
    cudaEventCreate(&f0);
    cudaEventCreate(&g0);
    for (size_t mb : {4, 20, 64}) {
      const size_t nn = (mb << 20) / 16;
      float best0 = 1e9, best1 = 1e9;
      for (int it = 0; it < 10; ++it) {
        CK(cudaSetDevice(0));
        cudaDeviceSynchronize();
        CK(cudaSetDevice(1));
        cudaDeviceSynchronize();
        CK(cudaSetDevice(0));
        cudaEventRecord(f0, s0);
        fold2<<<grid, blk, 0, s0>>>((float4*)a0, (float4*)b1, (float4*)b0, nn);
        cudaEventRecord(g0, s0);
        CK(cudaSetDevice(1));
        cudaEventRecord(f1, s1);
        fold2<<<grid, blk, 0, s1>>>((float4*)b1, (float4*)a0, (float4*)o1, nn);
        cudaEventRecord(g1, s1);
        cudaEventSynchronize(g1);
        CK(cudaSetDevice(0));
        cudaEventSynchronize(g0);
        float m0, m1;
        cudaEventElapsedTime(&m0, f0, g0);
        CK(cudaSetDevice(1));
        cudaEventElapsedTime(&m1, f1, g1);
        CK(cudaSetDevice(0));
        best0 = m0 < best0 ? m0 : best0;
        best1 = m1 < best1 ? m1 : best1;
      }
      printf("%3zu MB: bidirectional fold GPU0 %7.1f us, GPU1 %7.1f us (%6.1f GB/s remote each)\n", mb,
             best0 * 1e3, best1 * 1e3, (mb << 20) / (best0 * 1e-3) / 1e9);
    }
  }
  // both GPUs WRITE into each other at once (the n = 2 push exchange),
  // 20 MiB each way, at several grid sizes; then the copy engines
  {
    float *r0, *r1, *l1;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&r1, bytes + 64));
    CK(cudaMalloc(&l1, bytes + 64));
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&r0, bytes + 64));
    cudaStream_t s0, s1;
    cudaEvent_t f0, f1, g0, g1;
    CK(cudaSetDevice(1));
    cudaStreamCreate(&s1);
    cudaEventCreate(&f1);
    cudaEventCreate(&g1);
    CK(cudaSetDevice(0));
    cudaStreamCreate(&s0);
    cudaEventCreate(&f0);
    cudaEventCreate(&g0);
    for (size_t mb_ : {(size_t)20, (size_t)128})
    for (int mode = 0; mode < 5; ++mode) {
      const size_t mb = mb_, nn = (mb << 20) / 16;
      const int grids[4] = {148, 296, 592, 1184};
      float best0 = 1e9, best1 = 1e9;
      for (int it = 0; it < 10; ++it) {
        CK(cudaSetDevice(0));
        cudaDeviceSynchronize();
        CK(cudaSetDevice(1));
        cudaDeviceSynchronize();
        CK(cudaSetDevice(0));
        cudaEventRecord(f0, s0);
        if (mode < 4) wr4<<<grids[mode], blk, 0, s0>>>((float4*)a0, (float4*)r1, nn);
        else cudaMemcpyPeerAsync(r1, 1, a0, 0, mb << 20, s0);
        cudaEventRecord(g0, s0);
        CK(cudaSetDevice(1));
        cudaEventRecord(f1, s1);
        if (mode < 4) wr4<<<grids[mode], blk, 0, s1>>>((float4*)l1, (float4*)r0, nn);
        else cudaMemcpyPeerAsync(r0, 0, l1, 1, mb << 20, s1);
        cudaEventRecord(g1, s1);
        cudaEventSynchronize(g1);
        CK(cudaSetDevice(0));
        cudaEventSynchronize(g0);
        float m0, m1;
        cudaEventElapsedTime(&m0, f0, g0);
        CK(cudaSetDevice(1));
        cudaEventElapsedTime(&m1, f1, g1);
        CK(cudaSetDevice(0));
        best0 = m0 < best0 ? m0 : best0;
        best1 = m1 < best1 ? m1 : best1;
      }
      printf("%3zu MB bidirectional %s (grid %d): GPU0 %7.1f us, GPU1 %7.1f us (%6.1f GB/s each way)\n", mb,
             mode < 4 ? "WRITE float4" : "cudaMemcpyPeer", mode < 4 ? grids[mode] : 0, best0 * 1e3, best1 * 1e3,
             (mb << 20) / (best0 * 1e-3) / 1e9);
    }
    const size_t mb = 20, nn = (mb << 20) / 16;
    // bulk copy / bulk reduce-add, both directions at once; then check the sums
    for (int red = 0; red < 2; ++red) {
      float best0 = 1e9;
      for (int it = 0; it < 10; ++it) {
        CK(cudaSetDevice(0));
        cudaDeviceSynchronize();
        CK(cudaSetDevice(1));
        cudaDeviceSynchronize();
        CK(cudaSetDevice(0));
        cudaEventRecord(f0, s0);
        if (red) bulk_push<true><<<148 * 2, 256, 0, s0>>>(a0, r1, nn * 4);
        else bulk_push<false><<<148 * 2, 256, 0, s0>>>(a0, r1, nn * 4);
        cudaEventRecord(g0, s0);
        CK(cudaSetDevice(1));
        if (red) bulk_push<true><<<148 * 2, 256, 0, s1>>>(l1, r0, nn * 4);
        else bulk_push<false><<<148 * 2, 256, 0, s1>>>(l1, r0, nn * 4);
        cudaStreamSynchronize(s1);
        CK(cudaSetDevice(0));
        cudaEventSynchronize(g0);
        float m0;
        cudaEventElapsedTime(&m0, f0, g0);
        best0 = m0 < best0 ? m0 : best0;
      }
      CK(cudaGetLastError());
      printf("%3zu MB bidirectional bulk %s: %7.1f us (%6.1f GB/s each way)\n", mb, red ? "REDUCE-ADD" : "copy",
             best0 * 1e3, (mb << 20) / (best0 * 1e-3) / 1e9);
    }
    {  // correctness of the remote reduce-add: r1 = 1.0 + sum of pushes
      CK(cudaSetDevice(0));
      float* h = (float*)malloc(16 * 4);
      std::vector<float> ones(nn * 4, 1.0f), twos(nn * 4, 2.0f);
      CK(cudaMemcpy(a0, twos.data(), nn * 16, cudaMemcpyHostToDevice));
      CK(cudaSetDevice(1));
      CK(cudaMemcpy(r1, ones.data(), nn * 16, cudaMemcpyHostToDevice));
      CK(cudaSetDevice(0));
      bulk_push<true><<<148 * 2, 256, 0, s0>>>(a0, r1, nn * 4);
      CK(cudaStreamSynchronize(s0));
      CK(cudaSetDevice(1));
      CK(cudaMemcpy(h, r1 + 12345, 16 * 4, cudaMemcpyDeviceToHost));
      printf("remote reduce-add check: %s (r1[12345] = %.1f, want 3.0)\n", h[0] == 3.0f ? "OK" : "WRONG", h[0]);
      CK(cudaSetDevice(0));
      free(h);
    }
  }
  return 0;
}
