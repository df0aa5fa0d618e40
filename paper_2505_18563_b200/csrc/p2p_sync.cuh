// p2p_sync.cuh -- device-side flag protocol of the NVLink P2P exchange,
// shared by the exchange kernels (p2p.cu) and the unpack kernels that consume
// peer memory directly (codec.cu).
#pragma once

#include "common.cuh"
#include "launch.h"

namespace pactk {
namespace p2psync {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// thread 0 waits until flags[kind][s] >= target for all s < n; block
// barrier. Returns false (in every thread) when the exchange has failed:
// already flagged, or a peer did not publish within the timeout (then the
// failure is raised, device and host side). Callers skip their peer reads
// and their exit signals on false.
__device__ __forceinline__ bool block_wait_flags(const uint64_t* flags, int kind, int n, uint64_t target,
                                                 P2PErr* err) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = *reinterpret_cast<volatile int*>(&err->flag) == 0;
    const uint64_t t0 = globaltimer();
    for (int s = 0; ok && s < n; ++s) {
      while (ld_acquire_sys(flags + kind * kP2PMaxRanks + s) < target) {
        if (globaltimer() - t0 > err->timeout_ns) {  // a peer died or stalled: fail, do not hang
          atomicExch(&err->flag, 1);
          if (err->host) *err->host = 1;
          __threadfence_system();
          ok = 0;
          break;
        }
        __nanosleep(64);
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// Fused signalling (saves a launch per signal): the ENTRY flag is published
// by block 0 before anyone waits -- the producer kernel ran earlier on this
// stream, so its stores are complete; the EXIT flag is published by the last
// CTA to finish (thread-fence reduction pattern), after every CTA's stores.
__device__ __forceinline__ void publish(const P2PView& v, int kind, uint64_t value) {
  __threadfence_system();
  for (int r = 0; r < v.n; ++r) st_release_sys(v.flags[r] + kind * kP2PMaxRanks + v.rank, value);
}
__device__ __forceinline__ void entry_signal(const P2PView& v, const P2PSig& sg) {
  if (sg.entry_kind >= 0 && blockIdx.x == 0 && threadIdx.x == 0) publish(v, sg.entry_kind, sg.entry_val);
}
__device__ __forceinline__ void exit_signal(const P2PView& v, const P2PSig& sg) {
  if (sg.exit_kind < 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(sg.counter, 1u) == gridDim.x - 1) {
      *sg.counter = 0;  // every other CTA has arrived: reset for the next launch
      publish(v, sg.exit_kind, sg.exit_val);
    }
  }
}

}  // namespace p2psync
}  // namespace pactk
