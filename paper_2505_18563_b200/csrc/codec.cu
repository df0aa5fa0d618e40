// codec.cu -- mask-indexed stream compaction (pack), scatter-expand (unpack,
// optionally fused with to_mean and the masked SGD step), GSE, and the
// mask bookkeeping kernels (fill, chunk popcounts, exclusive scan).
//
// Reference semantics: codec.cpp:14-38 (pack/unpack), sparsity.cpp:112-119
// (GSE), trainer.cpp:202-214 and 268-273 (to_mean + sgd_step), tensor.cpp
// 83-129 (mask layout, nnz).
//
// Layout: the gradient is cut into 1024-element chunks (16 mask words; the
// word array is padded to whole chunks). A mask carries chunk_off[c] = kept
// elements before chunk c, so one WARP owns one chunk end to end with no
// inter-warp communication. Pack and unpack are LANE-MAJOR: lane l owns mask
// half-word l (32 consecutive elements), so a lane's kept values are
// consecutive in the packed run from one warp scan of the half-word
// popcounts -- no per-slot ranks. The dense side moves through a per-warp,
// XOR-swizzled shared-memory stage (cp.async in, coalesced float4 out), so
// global accesses stay coalesced while the compaction / expansion works on
// the lane-major view. Persistent grids; warps stride over chunks; every
// kernel keeps a three-stage cp.async pipeline per warp (words of chunk
// i+2, data of chunk i+1, work on chunk i).
//
// The kernels are issue- and shared-memory-bound, not DRAM-bound, at the
// sizes of interest, so the formulation minimises instructions per element
// (ncu c2: the earlier register-resident pack issued ~570 warp-instructions
// per chunk at 65% issue utilisation and 33% of DRAM peak).
#include <cstdlib>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "launch.h"
#include "p2p_sync.cuh"

namespace pactk {

namespace {

constexpr int kCodecWarps = 8;  // 256-thread CTAs

// PACT_P2P_TRACE diagnostics of the n = 2 push exchange (%globaltimer ns):
// [0] pack entry (min) [1] pack exit (max) [2] unpack entry (min)
// [3] unpack past the PACKED wait (max) [4] unpack exit (max)
__device__ unsigned long long g_pair_trace[5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
std::atomic<unsigned long long> g_launches{0};

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename K>
int persistent_grid(K kernel, int warps = kCodecWarps) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, warps * 32, 0);
  if (per_sm <= 0) per_sm = 1;
  return sm_count() * per_sm;
}

// persistent grid of a kernel with `dyn` bytes of dynamic shared memory (opted in above 48 KiB)
template <typename K>
int persistent_grid_dyn(K kernel, int warps, int dyn) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, warps * 32, dyn);
  if (per_sm <= 0) per_sm = 1;
  return sm_count() * per_sm;
}

unsigned grid_for(int cap, uint64_t chunks, int warps = kCodecWarps) {
  const uint64_t need = (chunks + warps - 1) / warps;
  return (unsigned)(need < (uint64_t)cap ? need : (uint64_t)cap);
}

// per-warp stage of a chunk's 16 mask words + chunk_off[c], chunk_off[c+1]
constexpr int kWbuf = kChunkWords + 2;

// Slot j of the current chunk: nibble and in-chunk rank of lane's first
// element. `run` accumulates the kept count of the slots before (uniform).
struct Slot {
  uint32_t nib, pos;
};
__device__ __forceinline__ Slot chunk_slot(const uint64_t* wc, int j, uint32_t& run) {
  const int lane = threadIdx.x & 31;
  const ulonglong2 ab = reinterpret_cast<const ulonglong2*>(wc)[j];
  const uint64_t w = lane < 16 ? ab.x : ab.y;
  const int sh = 4 * (lane & 15);
  Slot s;
  s.nib = (uint32_t)(w >> sh) & 0xFu;
  const uint32_t pa = (uint32_t)__popcll(ab.x);
  s.pos = run + (uint32_t)__popcll(w & ((1ull << sh) - 1ull)) + (lane < 16 ? 0u : pa);
  run += pa + (uint32_t)__popcll(ab.y);
  return s;
}

// ------------------------------------------------------------------ pack
// kPush (NVLink one-shot, n = 2): the run is also written into the peer's
// incoming region (aligned float4 cells; scalar head / tail), and the last
// CTA publishes PACKED. (Tried: the LOCAL run as a TMA bulk copy smem ->
// global: c5 pack 264 -> 297 us; the remote run as a bulk copy is kept.)
constexpr int kPuWarps = 4;  // 128-thread CTAs

// dst and st are 16-byte aligned; values occupy [ph, ph + run)
__device__ __forceinline__ void write_run(float* __restrict__ dst, const float* st, uint32_t ph, uint32_t run) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t tot = ph + run;
  const uint32_t q0 = ph ? 1u : 0u, qe = tot >> 2;
  if (ph) {  // head: [ph, min(4, tot))
    const uint32_t i = ph + lane;
    if (i < 4 && i < tot) dst[i] = st[i];
  }
  for (uint32_t q = q0 + lane; q < qe; q += 32)
    reinterpret_cast<float4*>(dst)[q] = reinterpret_cast<const float4*>(st)[q];
  const uint32_t t0 = 4 * (qe > q0 ? qe : q0);
  if (t0 + lane < tot) dst[t0 + lane] = st[t0 + lane];
}

// ---------------------------------------------------------------- unpack
// kSgd: fused to_mean (scale) + masked SGD on weights; out (grad) optional.
// Three-stage cp.async pipeline per warp: mask words + offsets of chunk i+2,
// the packed run of chunk i+1 (exact length, from the offsets), expansion of
// chunk i with full-float4 streaming stores.
__device__ __forceinline__ void offs_words_issue(uint64_t* dst, const uint64_t* __restrict__ words,
                                                 const uint32_t* __restrict__ chunk_off, uint64_t c) {
  const int lane = threadIdx.x & 31;
  if (lane < 8) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + 2 * lane);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                 "l"(words + c * kChunkWords + 2 * lane)
                 : "memory");
  } else if (lane < 10) {  // chunk_off[c], chunk_off[c+1] -> low halves of dst[16], dst[17]
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + kChunkWords + (lane - 8));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(chunk_off + c + (lane - 8))
                 : "memory");
  }
}
// Copy a packed run of cnt floats into shared memory. When dst and src agree
// mod 16 bytes the interior moves as 16-byte cp.async.cg (a quarter of the
// copy instructions, and full-sector requests over NVLink), the ragged head
// and tail as 4-byte copies. Callers place dst at the source's 16-byte phase
// (run_phase) so the fast path always applies.
__device__ __forceinline__ uint32_t run_phase(const float* src) { return ((uintptr_t)src >> 2) & 3u; }
__device__ __forceinline__ void run_issue(float* dst, const float* __restrict__ src, uint32_t cnt) {
  const int lane = threadIdx.x & 31;
  auto cp4 = [&](uint32_t i) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + i);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src + i) : "memory");
  };
  if ((((uintptr_t)dst ^ (uintptr_t)src) & 15) != 0) {
    for (uint32_t i = lane; i < cnt; i += 32) cp4(i);
    return;
  }
  uint32_t head = (4u - run_phase(src)) & 3u;
  if (head > cnt) head = cnt;
  const uint32_t nvec = (cnt - head) >> 2, tail0 = head + 4 * nvec;
  if ((uint32_t)lane < head) cp4(lane);
  for (uint32_t q = lane; q < nvec; q += 32) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + head + 4 * q);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + head + 4 * q) : "memory");
  }
  if ((uint32_t)lane < cnt - tail0) cp4(tail0 + lane);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// Where a chunk's packed run comes from (the exchange fused into unpack):
//   kSrcLocal  this rank's packed (or already reduced) vector;
//   kSrcPair   NVLink one-shot, n = 2: the local run and the peer's run
//              (peer memory), summed at expansion -- the reference fold of
//              two terms, x_c + x_{c+1}, is the same in either order;
//   kSrcOwner  NVLink two-shot all-gather: the run read straight from the
//              owner's reduced chunk (owner = j / C, at most one owner
//              boundary per run since C >= 1024).
constexpr int kSrcLocal = 0, kSrcPair = 1, kSrcOwner = 2;

constexpr int kRunCap = kChunk + 4;  // a run plus its 16-byte phase

// source(s) of run [b, b + cnt); stage slot layout: run at phase offset
// run_phase(src), the pair variant's peer run kRunCap floats further
template <int kSrc>
__device__ __forceinline__ const float* run_src(const float* __restrict__ packed, const P2PView& v, uint32_t b,
                                                int which) {
  if constexpr (kSrc == kSrcLocal) return packed + b;
  else if constexpr (kSrc == kSrcPair) return (which ? v.packed[v.rank ^ 1] : packed) + b;
  else return v.reduced[b / v.C] + b;
}

template <int kSrc>
__device__ __forceinline__ void issue_run(float* dst, const float* __restrict__ packed, const P2PView& v,
                                          uint32_t b, uint32_t cnt) {
  if constexpr (kSrc == kSrcLocal) {
    const float* src = packed + b;
    run_issue(dst + run_phase(src), src, cnt);
  } else if constexpr (kSrc == kSrcPair) {
    const float* a = packed + b;
    const float* r = v.packed[v.rank ^ 1] + b;
    run_issue(dst + run_phase(a), a, cnt);
    run_issue(dst + kRunCap + run_phase(r), r, cnt);
  } else {  // owners' reduced chunks live at the absolute packed index
    const uint64_t o = b / v.C, nb = (o + 1) * v.C;
    const uint32_t n1 = nb - b < cnt ? (uint32_t)(nb - b) : cnt;
    const float* a = v.reduced[o] + b;
    const uint32_t ph = run_phase(a);
    run_issue(dst + ph, a, n1);
    if (n1 < cnt) run_issue(dst + ph + n1, v.reduced[o + 1] + b + n1, cnt - n1);
  }
}

// ------------------------------------------------------- pack, lane-major
// The register-resident pack above spends ~570 warp-instructions per chunk
// recomputing per-slot ranks (ncu c2: issue-bound, 65% issue slots busy at
// 33% of DRAM peak). This variant moves the chunk through shared memory so
// that the compaction is lane-major like the unpack: lane l owns mask
// half-word l (32 consecutive elements), its kept values land at one warp
// scan's offset, no per-slot ranks. Three-stage cp.async pipeline per warp
// (words + offsets of chunk i+2; the gradient slots of chunk i+1, issued only
// where the slot's 4-bit nibble is non-zero, so only sectors holding kept
// values are read; compaction of chunk i). The stage is XOR-swizzled (16-byte
// cell q of a 128-byte row at column (q ^ row) & 7) so both the slot-major
// cp.async writes and the lane-major LDS.128 reads are conflict-free; the
// compacted run is written back in place (after every lane has read its
// cells) at the destination's 16-byte phase and leaves as one coalesced run.
constexpr int kPushNone = 0, kPushStores = 1, kPushTma = 2;

// NVLink push of a staged run as one bulk async copy (TMA engine, smem ->
// peer global) for the whole 16-byte cells, scalar stores for the partial
// head / tail cells (they are shared with the neighbouring chunks' runs).
// The warp does not wait for the remote stores: the stage is recycled after
// cp.async.bulk.wait_group.read, the kernel exit waits for completion.
__device__ __forceinline__ void push_run_bulk(float* __restrict__ dst, const float* st, uint32_t ph, uint32_t run) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t tot = ph + run;
  const uint32_t q0 = ph ? 1u : 0u, qe = tot >> 2;
  if (ph) {
    const uint32_t i = ph + lane;
    if (i < 4 && i < tot) dst[i] = st[i];
  }
  const uint32_t t0 = 4 * (qe > q0 ? qe : q0);
  if (t0 + lane < tot) dst[t0 + lane] = st[t0 + lane];
  if (qe > q0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the compaction's STS -> async proxy
    __syncwarp();
    if (lane == 0) {
      asm volatile(
          "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
          " cp.async.bulk.commit_group;" ::"l"(dst + 4 * q0),
          "r"((uint32_t)__cvta_generic_to_shared(st + 4 * q0)), "r"((qe - q0) * 16u)
          : "memory");
    }
  }
}

constexpr int kPkStage = kChunk + 4;  // a chunk, or a run plus its 16-byte phase
__device__ __forceinline__ int swz_cell(int q) { return (q & ~7) | ((q ^ (q >> 3)) & 7); }

__device__ __forceinline__ void pack_data_issue(float* st, const float* __restrict__ g, uint64_t len, bool vec_ok,
                                                const uint64_t* wc, uint64_t c) {
  const int lane = threadIdx.x & 31;
  const uint64_t e0 = c * (uint64_t)kChunk;
#pragma unroll
  for (int j = 0; j < kVecPerLane; ++j) {
    const uint32_t nib = (uint32_t)(wc[2 * j + (lane >> 4)] >> (4 * (lane & 15))) & 0xFu;
    const int q = 32 * j + lane;
    const uint64_t ge = e0 + 4 * (uint64_t)q;
    float* d = st + 4 * swz_cell(q);
    if (nib) {
      if (vec_ok && ge + 4 <= len) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
                     "l"(g + ge)
                     : "memory");
      } else {  // unaligned base or ragged tail: kept (hence in-range) elements only
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if ((nib >> b) & 1)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(d + b)),
                         "l"(g + ge + b)
                         : "memory");
      }
    }
  }
}

template <int kPush>
__global__ void __launch_bounds__(kPuWarps * 32)
    pack_lm_kernel(const float* __restrict__ g, uint64_t len, const uint64_t* __restrict__ words,
                   const uint32_t* __restrict__ chunk_off, float* __restrict__ packed, uint64_t cb,
                   uint64_t ce, float* __restrict__ remote, P2PView v, P2PSig sg, int pdl_trigger) {
  __shared__ __align__(16) float dsm[kPuWarps][2][kPkStage];
  __shared__ __align__(16) uint64_t wsm[kPuWarps][3][kWbuf];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec_ok = (((uintptr_t)g) & 15) == 0;
  const uint64_t nwt = (uint64_t)gridDim.x * kPuWarps;
  uint64_t c = cb + (uint64_t)blockIdx.x * kPuWarps + warp;
  // a programmatic dependent (the single-GPU unpack) may be scheduled as soon
  // as SMs free up; it waits for this grid's completion before reading
  // `packed`. Only when the caller launches one: a PDL-capable successor of
  // another kind (e.g. a collective kernel) must not be let in early.
  if (pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if constexpr (kPush != kPushNone)
    if (sg.trace && threadIdx.x == 0) atomicMin(&g_pair_trace[0], gtimer());
  if (c < ce) {
    // prologue: words(c0), words(c1), data(c0)
    offs_words_issue(wsm[warp][0], words, chunk_off, c);
    cp_commit();
    if (c + nwt < ce) offs_words_issue(wsm[warp][1], words, chunk_off, c + nwt);
    cp_commit();
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    pack_data_issue(dsm[warp][0], g, len, vec_ok, wsm[warp][0], c);
    cp_commit();
    // lane-major rank of chunk i+1 computed during chunk i (as in unpack)
    uint32_t h = reinterpret_cast<const uint32_t*>(wsm[warp][0])[lane];
    uint32_t hc = __popc(h), incl = warp_incl_scan(hc);
    int wi = 0, pi = 0;
    for (; c < ce; c += nwt) {
      const int w1 = wi == 2 ? 0 : wi + 1, w2 = w1 == 2 ? 0 : w1 + 1;
      if (c + 2 * nwt < ce) offs_words_issue(wsm[warp][w2], words, chunk_off, c + 2 * nwt);
      cp_commit();
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // words(c+nwt), data(c) landed
      __syncwarp();
      if constexpr (kPush == kPushTma) {  // the bulk push of stage pi ^ 1 has read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
      if (c + nwt < ce) pack_data_issue(dsm[warp][pi ^ 1], g, len, vec_ok, wsm[warp][w1], c + nwt);
      cp_commit();
      const uint64_t* wc = wsm[warp][wi];
      const uint32_t base = reinterpret_cast<const uint32_t*>(wc + kChunkWords)[0];
      float* st = dsm[warp][pi];
      const uint32_t h_n = reinterpret_cast<const uint32_t*>(wsm[warp][w1])[lane];  // chunk c + nwt
      const uint32_t hc_n = __popc(h_n), incl_n = warp_incl_scan(hc_n);
      const uint32_t run = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t ph = (uint32_t)(((uintptr_t)(packed + base) >> 2) & 3u);
      // lane-major read of the lane's 32 elements (cells 8 l .. 8 l + 7)
      float x[32];
      const float4* S = reinterpret_cast<const float4*>(st);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 t = S[8 * lane + ((k ^ lane) & 7)];
        x[4 * k] = t.x, x[4 * k + 1] = t.y, x[4 * k + 2] = t.z, x[4 * k + 3] = t.w;
      }
      __syncwarp();
      // in-place compaction: per element a bit test, a predicated STS and a
      // predicated address increment
      // (four independent address chains of 8 elements, started from byte
      // popcounts: the chain of predicated increments is 8 deep, not 32)
      uint32_t sa[4];
      sa[0] = (uint32_t)__cvta_generic_to_shared(st + ph + incl - hc);
      sa[1] = sa[0] + 4u * (uint32_t)__popc(h & 0xffu);
      sa[2] = sa[0] + 4u * (uint32_t)__popc(h & 0xffffu);
      sa[3] = sa[0] + 4u * (uint32_t)__popc(h & 0xffffffu);
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.f32 [%0], %1;\n"
              " @p add.u32 %0, %0, 4;\n}"
              : "+r"(sa[q])
              : "f"(x[8 * q + e]), "r"(h & (1u << (8 * q + e)))
              : "memory");
      __syncwarp();
      float* dst = packed + base;
#pragma unroll 4
      for (uint32_t i = lane; i < run; i += 32) dst[i] = st[ph + i];
      if constexpr (kPush == kPushStores) write_run(remote + base - ph, st, ph, run);
      if constexpr (kPush == kPushTma) push_run_bulk(remote + base - ph, st, ph, run);
      __syncwarp();  // stage pi and word buffer wi are refilled next
      wi = w1;
      pi ^= 1;
      h = h_n;
      hc = hc_n;
      incl = incl_n;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if constexpr (kPush == kPushTma) {  // the bulk stores have landed in the peer's memory
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n fence.proxy.async.global;" ::: "memory");
      __syncwarp();
    }
  }
  if constexpr (kPush != kPushNone) {
    p2psync::exit_signal(v, sg);  // PACKED: every CTA's remote stores are done
    if (sg.trace && threadIdx.x == 0) atomicMax(&g_pair_trace[1], gtimer());
  }
}

// kA = packed runs in flight ahead of the expansion. 2 halves the exposed
// run latency but costs a third more shared memory (16 instead of 24 warps
// per SM): it wins once each warp has many chunks (c3 unpack 111 -> 104 us,
// c5 290 -> 262 us) and loses on short grids (c2 24.6 -> 26.6 us), so the
// launcher picks by chunks per warp. The pair variant keeps 1 (two runs
// per stage).
template <int kSrc, int kA>
__host__ __device__ constexpr int unpack_smem_bytes() {
  return kPuWarps * (kA + 1) * (kSrc == kSrcPair ? 2 : 1) * kRunCap * (int)sizeof(float);
}

template <bool kSgd, int kSrc, int kA>
__global__ void __launch_bounds__(kPuWarps * 32)
    unpack_kernel(const float* __restrict__ packed, uint64_t len, const uint64_t* __restrict__ words,
                  const uint32_t* __restrict__ chunk_off, float scale, int do_scale,
                  float* __restrict__ out, float lr, float* __restrict__ weights, uint64_t cb,
                  uint64_t ce, P2PView v, const uint64_t* __restrict__ flags, uint64_t target,
                  P2PErr* __restrict__ err, P2PSig sg, int bulk_out) {
  constexpr int kRS = kA + 1, kWS = kA + 2;  // run / word stages
  constexpr int kRun = kSrc == kSrcPair ? 2 * kRunCap : kRunCap;
  extern __shared__ __align__(16) float psm_base[];  // unpack_smem_bytes<kSrc, kA>()
  auto psm = [&](int w, int st) { return psm_base + (w * kRS + st) * kRun; };
  __shared__ __align__(16) uint64_t wsm[kPuWarps][kWS][kWbuf];
  if constexpr (kSrc != kSrcLocal) {  // peers' PACKED (one-shot) / REDUCED (two-shot) flags
    p2psync::entry_signal(v, sg);
    if (sg.trace && threadIdx.x == 0) atomicMin(&g_pair_trace[2], gtimer());
    if (!p2psync::block_wait_flags(flags, kSrc == kSrcPair ? kP2PPacked : kP2PReduced, v.n, target, err))
      return;  // the exchange failed: no peer reads, no READ signal (LinkError on the host)
    if (sg.trace && threadIdx.x == 0) atomicMax(&g_pair_trace[3], gtimer());
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec_ok = ((((uintptr_t)out) | (kSgd ? (uintptr_t)weights : 0)) & 15) == 0;
  const bool uni_scale = scale > 0.0f && scale <= 3.4028235e38f;  // positive, finite
  const uint64_t nwt = (uint64_t)gridDim.x * kPuWarps;
  uint64_t c = cb + (uint64_t)blockIdx.x * kPuWarps + warp;
  if (c < ce) {
  auto offs = [&](int slot, uint32_t& b, uint32_t& n) {
    const uint32_t* o = reinterpret_cast<const uint32_t*>(wsm[warp][slot] + kChunkWords);
    b = o[0];
    n = o[2] - o[0];
  };
  // cp.async groups, in commit order: words w0..w_kA, runs r0..r_{kA-1};
  // then per chunk i: w_{i+kA+1}, r_{i+kA}. At chunk i, waiting for all but
  // the newest kA groups leaves exactly r_i and w_{i+kA} landed.
  for (int j = 0; j <= kA; ++j) {
    if (c + j * nwt < ce) offs_words_issue(wsm[warp][j], words, chunk_off, c + j * nwt);
    cp_commit();
  }
  asm volatile("cp.async.wait_group 1;" ::: "memory");  // w0 .. w_{kA-1}
  __syncwarp();
  // launched as a programmatic dependent of the pack: the packed vector is
  // complete and visible only past this point (no-op otherwise). The NVLink
  // variants need no grid dependency: the PACKED / REDUCED flags they waited
  // for are published by the producers' last CTAs after all their stores.
  if constexpr (kSrc == kSrcLocal) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int j = 0; j < kA; ++j) {
    if (c + j * nwt < ce) {
      uint32_t b, n;
      offs(j, b, n);
      issue_run<kSrc>(psm(warp, j), packed, v, b, n);
    }
    cp_commit();
  }
  // (1') the chunk's lane-major rank, one chunk ahead: lane l owns the 32
  // elements of mask half-word l, whose kept values are consecutive in the
  // staged run from its warp rank. The scan of chunk i+1 is issued before
  // chunk i's expansion so its shuffle latency overlaps that work.
  uint32_t h = reinterpret_cast<const uint32_t*>(wsm[warp][0])[lane];
  uint32_t pos0 = warp_incl_scan((uint32_t)__popc(h)) - (uint32_t)__popc(h);
  int wi = 0, pi = 0;
  bool bulk_pending = false;  // the previous chunk left as a bulk store from stage pa
  for (; c < ce; c += nwt) {
    const int w1 = (wi + 1) % kWS, wa = (wi + kA) % kWS, wa1 = (wi + kA + 1) % kWS, pa = (pi + kA) % kRS;
    if (c + (kA + 1) * nwt < ce) offs_words_issue(wsm[warp][wa1], words, chunk_off, c + (kA + 1) * nwt);
    cp_commit();
    asm volatile("cp.async.wait_group %0;" ::"n"(kA) : "memory");  // run(c), words(c + kA nwt) landed
    if (bulk_pending) {  // stage pa (the previous chunk's) has been read by its bulk store
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      bulk_pending = false;
    }
    __syncwarp();
    if (c + kA * nwt < ce) {
      uint32_t b, n;
      offs(wa, b, n);
      issue_run<kSrc>(psm(warp, pa), packed, v, b, n);
    }
    cp_commit();
    const uint64_t* wc = wsm[warp][wi];
    const uint32_t rb = reinterpret_cast<const uint32_t*>(wsm[warp][wi] + kChunkWords)[0];
    const float* stage = psm(warp, pi) + run_phase(run_src<kSrc>(packed, v, rb, 0));
    const uint32_t h_n = reinterpret_cast<const uint32_t*>(wsm[warp][w1])[lane];  // chunk c + nwt
    const uint32_t pos0_n = warp_incl_scan((uint32_t)__popc(h_n)) - (uint32_t)__popc(h_n);
    // (1) lane-major expansion of chunk c: per element a bit test, a
    // predicated LDS at the lane's walking 32-bit shared address and a
    // predicated address increment. (Tried: unconditional loads at the
    // walking address + a bit mask, which frees the loads from the
    // predicate chain but puts all 32 lanes on the banks: c2 24.6 -> 28.6 us.)
    float x[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) x[e] = 0.0f;
    // (four independent walking addresses of 8 elements each, started from
    // byte popcounts: the predicated-increment chain is 8 deep, not 32)
    const uint32_t q1 = (uint32_t)__popc(h & 0xffu), q2 = (uint32_t)__popc(h & 0xffffu),
                   q3 = (uint32_t)__popc(h & 0xffffffu);
    if constexpr (kSrc != kSrcPair) {
      uint32_t sa[4];
      sa[0] = (uint32_t)__cvta_generic_to_shared(stage + pos0);
      sa[1] = sa[0] + 4u * q1;
      sa[2] = sa[0] + 4u * q2;
      sa[3] = sa[0] + 4u * q3;
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.f32 %0, [%1];\n"
              " @p add.u32 %1, %1, 4;\n}"
              : "+f"(x[8 * q + e]), "+r"(sa[q])
              : "r"(h & (1u << (8 * q + e))));
    } else {  // + the peer's value (one-shot fold, n = 2)
      const float* a0 = stage + pos0;
      const float* b0 = psm(warp, pi) + kRunCap + run_phase(run_src<kSrc>(packed, v, rb, 1)) + pos0;
      const float* sa[4] = {a0, a0 + q1, a0 + q2, a0 + q3};
      const float* sp[4] = {b0, b0 + q1, b0 + q2, b0 + q3};
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (h & (1u << (8 * q + e))) x[8 * q + e] = __fadd_rn(*sa[q]++, *sp[q]++);
    }
    // (2) transpose through the consumed run buffer (XOR-swizzled 16-byte
    // cells: conflict-free both ways) into the coalesced layout: store j of
    // lane l covers elements 128 j + 4 l .. + 3
    __syncwarp();
    float4* T = reinterpret_cast<float4*>(psm(warp, pi));
#pragma unroll
    for (int k = 0; k < 8; ++k)
      T[lane * 8 + (k ^ (lane & 7))] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
    __syncwarp();
    const uint64_t e0 = c * (uint64_t)kChunk + 4 * lane;
    // cell of store j: row 4j + l/8, column (l & 7) ^ (row & 7) -- the XOR
    // term depends on j's parity only, so two per-lane bases + immediates
    const int tb0 = (lane >> 3) * 8 + ((lane & 7) ^ (lane >> 3));
    const int tb1 = (lane >> 3) * 8 + ((lane & 7) ^ ((lane >> 3) + 4));
    if (!kSgd && bulk_out && vec_ok && (c + 1) * (uint64_t)kChunk <= len) {
      // whole chunk, bulk store: the swizzled cells are read back (and
      // scaled), rewritten linearly in place (each 128-byte row is permuted
      // among its own 8 lanes) and leave as ONE 4 KiB cp.async.bulk from
      // shared to global memory (the TMA engine) instead of 256 STG.128
      float4 y[kVecPerLane];
#pragma unroll
      for (int j = 0; j < kVecPerLane; ++j) y[j] = T[32 * j + ((j & 1) ? tb1 : tb0)];
      if (do_scale) {
#pragma unroll
        for (int j = 0; j < kVecPerLane; ++j) {
          const uint32_t nib = (uint32_t)(wc[2 * j + (lane >> 4)] >> (4 * (lane & 15))) & 0xFu;
          if (nib & 1) y[j].x = __fmul_rn(y[j].x, scale);
          if (nib & 2) y[j].y = __fmul_rn(y[j].y, scale);
          if (nib & 4) y[j].z = __fmul_rn(y[j].z, scale);
          if (nib & 8) y[j].w = __fmul_rn(y[j].w, scale);
        }
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kVecPerLane; ++j) T[32 * j + lane] = y[j];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
            " cp.async.bulk.commit_group;" ::"l"(out + c * (uint64_t)kChunk),
            "r"((uint32_t)__cvta_generic_to_shared(T)), "r"(kChunk * 4)
            : "memory");
      bulk_pending = true;
    } else if (!kSgd && (!do_scale || uni_scale) && vec_ok && (c + 1) * (uint64_t)kChunk <= len) {
      // whole chunk: 8 x (LDS.128, STG.128); a positive finite scale is
      // applied to every element (dropped ones are +0: +0 * scale == +0, the
      // masked rule's result)
#pragma unroll
      for (int j = 0; j < kVecPerLane; ++j) {
        float4 t = T[32 * j + ((j & 1) ? tb1 : tb0)];
        if (do_scale) {
          t.x = __fmul_rn(t.x, scale);
          t.y = __fmul_rn(t.y, scale);
          t.z = __fmul_rn(t.z, scale);
          t.w = __fmul_rn(t.w, scale);
        }
        st_stream_f4(reinterpret_cast<float4*>(out + e0 + 128 * j), t);
      }
    } else
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const uint64_t ge = e0 + 128 * j;
      if (ge >= len) continue;
      const float4 t = T[32 * j + ((j & 1) ? tb1 : tb0)];
      float o[4] = {t.x, t.y, t.z, t.w};
      const uint32_t nib = (uint32_t)(wc[2 * j + (lane >> 4)] >> (4 * (lane & 15))) & 0xFu;
      if (do_scale) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if ((nib >> b) & 1) o[b] = __fmul_rn(o[b], scale);
      }
      const bool full = vec_ok && ge + 4 <= len;
      if (!kSgd || out != nullptr) {
        if (full)
          st_stream_f4(reinterpret_cast<float4*>(out + ge), make_float4(o[0], o[1], o[2], o[3]));
        else
          for (int b = 0; b < 4 && ge + b < len; ++b) out[ge + b] = o[b];
      }
      if (kSgd) {
        float q[4];
        if (full) {
          const float4 w4 = *reinterpret_cast<const float4*>(weights + ge);
          q[0] = w4.x, q[1] = w4.y, q[2] = w4.z, q[3] = w4.w;
        } else {
          for (int b = 0; b < 4; ++b) q[b] = ge + b < len ? weights[ge + b] : 0.f;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b)  // trainer.cpp:208-212, no FMA contraction
          q[b] = ((nib >> b) & 1) ? __fsub_rn(q[b], __fmul_rn(lr, o[b])) : 0.0f;
        if (full)
          *reinterpret_cast<float4*>(weights + ge) = make_float4(q[0], q[1], q[2], q[3]);
        else
          for (int b = 0; b < 4 && ge + b < len; ++b) weights[ge + b] = q[b];
      }
    }
    __syncwarp();  // run buffer `pi` and word buffer `wi` are refilled next
    wi = w1;
    pi = pi + 1 == kRS ? 0 : pi + 1;
    h = h_n;
    pos0 = pos0_n;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (bulk_out) {  // the bulk stores are complete (and the stages free) before the CTA exits
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  }
  if constexpr (kSrc != kSrcLocal) {
    p2psync::exit_signal(v, sg);  // READ: peers may reuse their buffers
    if (sg.trace && threadIdx.x == 0) atomicMax(&g_pair_trace[4], gtimer());
  }
}

// ------------------------------------------------------------------- GSE
__global__ void __launch_bounds__(kCodecWarps * 32)
    gse_kernel(const float* g, uint64_t len, const uint64_t* __restrict__ words, float* out,
               uint64_t nchunks) {  // out may alias g (in-place GSE)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec_ok = ((((uintptr_t)g) | ((uintptr_t)out)) & 15) == 0;
  const uint64_t nwt = (uint64_t)gridDim.x * kCodecWarps;
  for (uint64_t c = (uint64_t)blockIdx.x * kCodecWarps + warp; c < nchunks; c += nwt) {
    const uint64_t* wc = words + c * kChunkWords;
    const uint64_t e0 = c * (uint64_t)kChunk + 4 * lane;
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const uint32_t nib = chunk_slot(wc, j, run).nib;
      const uint64_t ge = e0 + 128 * j;
      if (ge >= len) continue;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vec_ok && ge + 4 <= len) {
        if (nib) {
          v = ld_stream_f4(reinterpret_cast<const float4*>(g + ge));
          if (!(nib & 1)) v.x = 0.f;
          if (!(nib & 2)) v.y = 0.f;
          if (!(nib & 4)) v.z = 0.f;
          if (!(nib & 8)) v.w = 0.f;
        }
        st_stream_f4(reinterpret_cast<float4*>(out + ge), v);
      } else {
        for (int b = 0; b < 4 && ge + b < len; ++b) out[ge + b] = (nib >> b) & 1 ? g[ge + b] : 0.0f;
      }
    }
  }
}

// out[i] = in[i] * scale (dense-fallback epilogue of to_mean, trainer.cpp:268-273)
__global__ void __launch_bounds__(256) scale_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    uint64_t len, float scale) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += stride)
    out[i] = __fmul_rn(in[i], scale);
}

// ------------------------------------------------------- mask bookkeeping
__global__ void mask_fill_kernel(uint64_t* words, uint64_t nwords, uint64_t len, int keep,
                                 uint32_t* chunk_off, uint64_t nchunks) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nwords; i += stride) {
    uint64_t w = keep ? ~0ull : 0ull;
    if (keep && i == nwords - 1 && (len & 63)) w = (1ull << (len & 63)) - 1ull;
    words[i] = w;
  }
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= nchunks; t += stride) {
    const uint64_t e = t * (uint64_t)kChunk;
    chunk_off[t] = keep ? (uint32_t)(e < len ? e : len) : 0u;
  }
}

__global__ void clear_tail_kernel(uint64_t* words, uint64_t len) {
  const uint64_t last = (len - 1) >> 6;
  words[last] &= (1ull << (len & 63)) - 1ull;
}

// half a warp per chunk: popcount of its 16 words
__global__ void chunk_popc_kernel(const uint64_t* __restrict__ words, uint64_t nwords,
                                  uint32_t* __restrict__ popc, uint64_t nchunks) {
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t c = gt >> 4;
  const uint64_t wi = c * kChunkWords + (gt & 15);
  uint32_t v = (c < nchunks && wi < nwords) ? (uint32_t)__popcll(words[wi]) : 0u;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((gt & 15) == 0 && c < nchunks) popc[c] = v;
}

// Single-pass exclusive scan (decoupled look-back): 8192 values per CTA,
// tiles ordered by a ticket so every CTA's predecessors are running or done.
constexpr uint64_t kStAgg = 1ull << 62, kStIncl = 2ull << 62, kStMask = 3ull << 62;
constexpr int kScanPerThread = 8;  // 2 x uint4 per thread
constexpr int kScanItems = 1024 * kScanPerThread;

__global__ void __launch_bounds__(1024) scan_excl_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                         uint32_t* __restrict__ out,
                                                         uint64_t* __restrict__ state,
                                                         unsigned* __restrict__ ticket) {
  __shared__ uint32_t warp_tot[33];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t t = s_tile;
  const uint64_t base = t * kScanItems;
  uint32_t v[kScanPerThread];
  uint32_t s = 0;
  const uint64_t b0 = base + (uint64_t)tid * kScanPerThread;
  const bool vec = b0 + kScanPerThread <= n && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (vec) {
#pragma unroll
    for (int i = 0; i < kScanPerThread / 4; ++i) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + b0) + i);
      v[4 * i] = q.x;
      v[4 * i + 1] = q.y;
      v[4 * i + 2] = q.z;
      v[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanPerThread; ++i) v[i] = b0 + i < n ? in[b0 + i] : 0u;
  }
#pragma unroll
  for (int i = 0; i < kScanPerThread; ++i) s += v[i];
  const uint32_t inc = warp_incl_scan(s);
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = warp_tot[lane];
    const uint32_t xi = warp_incl_scan(x);
    warp_tot[lane] = xi - x;
    const uint64_t total = __shfl_sync(0xffffffffu, xi, 31);
    uint64_t before = 0;
    if (t == 0) {
      if (lane == 0) st_relaxed_u64(state, kStIncl | total);
    } else {
      if (lane == 0) st_relaxed_u64(state + t, kStAgg | total);
      int64_t look = (int64_t)t - 1;
      while (true) {
        const int64_t p = look - lane;
        uint64_t st = p >= 0 ? ld_relaxed_u64(state + p) : kStIncl;
        while (__any_sync(0xffffffffu, (st & kStMask) == 0))
          if ((st & kStMask) == 0) st = ld_relaxed_u64(state + p);
        const unsigned incl = __ballot_sync(0xffffffffu, (st & kStMask) == kStIncl);
        const int L = incl ? __ffs(incl) - 1 : 31;
        before += warp_sum(lane <= L ? (st & ~kStMask) : 0ull);
        if (incl) break;
        look -= 32;
      }
      if (lane == 0) st_relaxed_u64(state + t, kStIncl | (before + total));
    }
    if (lane == 0) {
      s_prefix = before;
      if (base + kScanItems >= n) out[n] = (uint32_t)(before + total);
    }
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_prefix + warp_tot[warp] + inc - s;
#pragma unroll
  for (int i = 0; i < kScanPerThread; ++i) {
    const uint32_t x = v[i];
    v[i] = run;
    run += x;
  }
  if (vec) {
#pragma unroll
    for (int i = 0; i < kScanPerThread / 4; ++i)
      reinterpret_cast<uint4*>(out + b0)[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < kScanPerThread; ++i)
      if (b0 + i < n) out[b0 + i] = v[i];
  }
}


// Bit-gather of mask segments: dst bits [dst_start[s], dst_start[s+1]) =
// src bits from src_begin[s]. Thread per destination word; the (few)
// segments overlapping it are found by binary search over dst_start. The
// words past the last destination bit are written 0 (whole chunk padding).
__device__ __forceinline__ uint64_t bits_at(const uint64_t* __restrict__ src, uint64_t nsrc_words,
                                            uint64_t b) {  // 64 bits of src from bit b
  const uint64_t w = b >> 6;
  const int sh = (int)(b & 63);
  const uint64_t lo = w < nsrc_words ? src[w] : 0ull;
  if (!sh) return lo;
  const uint64_t hi = w + 1 < nsrc_words ? src[w + 1] : 0ull;
  return (lo >> sh) | (hi << (64 - sh));
}

__global__ void mask_gather_kernel(const uint64_t* __restrict__ src, uint64_t nsrc_words,
                                   const uint64_t* __restrict__ src_begin,
                                   const uint64_t* __restrict__ dst_start, uint64_t nseg,
                                   uint64_t* __restrict__ dst, uint64_t dst_len, uint64_t ndst_words) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < ndst_words; w += stride) {
    const uint64_t d0 = w * 64, dend = d0 + 64 < dst_len ? d0 + 64 : dst_len;
    uint64_t out = 0;
    if (d0 < dst_len) {
      uint64_t lo = 0, hi = nseg;  // last segment with dst_start <= d0
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (dst_start[mid] <= d0) lo = mid; else hi = mid;
      }
      for (uint64_t sg = lo, d = d0; d < dend && sg < nseg; ++sg) {
        const uint64_t se = dst_start[sg + 1];
        if (se <= d) continue;  // empty segment
        const uint64_t e = se < dend ? se : dend;
        const int nb = (int)(e - d), at = (int)(d - d0);
        uint64_t v = bits_at(src, nsrc_words, src_begin[sg] + (d - dst_start[sg]));
        if (nb < 64) v &= (1ull << nb) - 1ull;
        out |= v << at;
        d = e;
      }
    }
    dst[w] = out;
  }
}

}  // namespace

uint64_t launches() { return g_launches; }

void pair_trace_reset(cudaStream_t s) {
  unsigned long long init[5] = {~0ull, 0, ~0ull, 0, 0};
  cudaMemcpyToSymbolAsync(g_pair_trace, init, sizeof init, 0, cudaMemcpyHostToDevice, s);
}
void pair_trace_read(unsigned long long out[5], cudaStream_t s) {
  cudaMemcpyFromSymbolAsync(out, g_pair_trace, 5 * sizeof(unsigned long long), 0, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
}
void note_launch(uint64_t n) { g_launches += n; }

void launch_pack(const float* g, uint64_t len, const uint64_t* words, const uint32_t* chunk_off,
                 float* packed, uint64_t cb, uint64_t ce, cudaStream_t s, bool pdl_trigger, float grid_frac) {
  if (ce <= cb) return;
  static int cap = 0;
  if (!cap) cap = persistent_grid(pack_lm_kernel<kPushNone>, kPuWarps);
  const int c = grid_frac > 0.f ? std::max(1, (int)(cap * grid_frac)) : cap;
  pack_lm_kernel<kPushNone><<<grid_for(c, ce - cb, kPuWarps), kPuWarps * 32, 0, s>>>(
      g, len, words, chunk_off, packed, cb, ce, nullptr, P2PView{}, P2PSig{}, pdl_trigger ? 1 : 0);
  note_launch();
}

void launch_pack_push(const float* g, uint64_t len, const uint64_t* words, const uint32_t* chunk_off,
                      float* packed, float* remote, const P2PView& v, const P2PSig& sg, cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  // PACT_PUSH_STORES=1: float4 stores instead of bulk async copies (measured
  // c2 n=2 pack 61 vs 55-61 us: the exchange is NVLink-bound either way)
  static const bool stores = getenv("PACT_PUSH_STORES") != nullptr;
  static int cap = 0;
  if (!cap)
    cap = stores ? persistent_grid(pack_lm_kernel<kPushStores>, kPuWarps)
                 : persistent_grid(pack_lm_kernel<kPushTma>, kPuWarps);
  const unsigned grid = grid_for(cap, nc, kPuWarps);
  if (stores)
    pack_lm_kernel<kPushStores><<<grid, kPuWarps * 32, 0, s>>>(g, len, words, chunk_off, packed, 0, nc, remote,
                                                               v, sg, 0);
  else
    pack_lm_kernel<kPushTma><<<grid, kPuWarps * 32, 0, s>>>(g, len, words, chunk_off, packed, 0, nc, remote, v,
                                                            sg, 0);
  note_launch();
}

namespace {
// PACT_UNPACK_BULK=1: whole chunks leave as one 4 KiB cp.async.bulk store per
// warp instead of 8 STG.128 per lane. Measured slower (B200, unpack us, STG
// vs bulk: c2 26.6 vs 28.7, c3 110 vs 142, c5 277 vs 357): the stage a bulk
// store reads from is the next run's landing buffer, so every chunk waits
// for the previous chunk's store to drain from shared memory before its
// prefetch can be issued, where streaming STG.128s retire into the LSU.
int unpack_bulk_out() {
  static const int v = getenv("PACT_UNPACK_BULK") != nullptr;
  return v;
}
// chunks per warp of the one-run-ahead grid above which two runs ahead win
constexpr uint64_t kDeepUnpackChunksPerWarp = 16;
template <bool kSgd>
void unpack_local(const float* packed, uint64_t len, const uint64_t* words, const uint32_t* chunk_off, float scale,
                  int do_scale, float* out, float lr, float* weights, uint64_t cb, uint64_t ce, cudaStream_t s,
                  bool pdl = false, float grid_frac = 0.f) {
  constexpr int kDyn1 = unpack_smem_bytes<kSrcLocal, 1>(), kDyn2 = unpack_smem_bytes<kSrcLocal, 2>();
  static DeviceCache<int> c1c, c2c;  // dyn-smem opt-ins are per device
  int& cap1 = c1c.get();
  int& cap2 = c2c.get();
  if (!cap1) {
    cap1 = persistent_grid_dyn(unpack_kernel<kSgd, kSrcLocal, 1>, kPuWarps, kDyn1);
    cap2 = persistent_grid_dyn(unpack_kernel<kSgd, kSrcLocal, 2>, kPuWarps, kDyn2);
  }
  const bool deep = (ce - cb) >= kDeepUnpackChunksPerWarp * (uint64_t)cap1 * kPuWarps;
  const int cb_ = deep ? cap2 : cap1;
  const int c = grid_frac > 0.f ? std::max(1, (int)(cb_ * grid_frac)) : cb_;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_for(c, ce - cb, kPuWarps));
  cfg.blockDim = dim3(kPuWarps * 32);
  cfg.dynamicSmemBytes = deep ? kDyn2 : kDyn1;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // PDL only on short grids: measured c1 25.7 -> 23.6 us and c2 46.1 ->
  // 44.1 us per step, but c3 174 -> 220 us and c5 0.78 -> 0.94 ms on long ones
  cfg.numAttrs = pdl && !deep ? 1 : 0;
  const P2PView v{};
  const P2PSig sg{};
  const uint64_t* nf = nullptr;
  P2PErr* ne = nullptr;
  if (deep)
    cudaLaunchKernelEx(&cfg, unpack_kernel<kSgd, kSrcLocal, 2>, packed, len, words, chunk_off, scale, do_scale, out,
                       lr, weights, cb, ce, v, nf, (uint64_t)0, ne, sg, unpack_bulk_out());
  else
    cudaLaunchKernelEx(&cfg, unpack_kernel<kSgd, kSrcLocal, 1>, packed, len, words, chunk_off, scale, do_scale, out,
                       lr, weights, cb, ce, v, nf, (uint64_t)0, ne, sg, unpack_bulk_out());
}
}  // namespace

void launch_unpack(const float* packed, uint64_t len, const uint64_t* words,
                   const uint32_t* chunk_off, float scale, int do_scale, float* out, uint64_t cb,
                   uint64_t ce, cudaStream_t s, bool pdl, float grid_frac) {
  if (ce <= cb) return;
  unpack_local<false>(packed, len, words, chunk_off, scale, do_scale, out, 0.f, nullptr, cb, ce, s, pdl, grid_frac);
  note_launch();
}

void launch_unpack_p2p(const float* packed_local, uint64_t len, const uint64_t* words,
                       const uint32_t* chunk_off, float scale, int do_scale, float* out, const P2PView& v,
                       int two_shot, const uint64_t* flags, uint64_t target, P2PErr* err, const P2PSig& sg,
                       cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  // every CTA runs the flag wait and the exit count, so each gets >= 1 chunk
  // per warp 0 (grid <= ceil(nc / kPuWarps))
  if (!two_shot) {
    constexpr int kDyn = unpack_smem_bytes<kSrcPair, 1>();
    static DeviceCache<int> cc;
    int& cap = cc.get();
    if (!cap) cap = persistent_grid_dyn(unpack_kernel<false, kSrcPair, 1>, kPuWarps, kDyn);
    // (Tried: a programmatic dependent launch after the push pack, waiting on
    // PACKED instead of the grid: the ~10 us gap after the push pack stays
    // and long grids slow down -- c3 0.26 -> 0.36 ms, c5 1.00 -> 1.21 ms.)
    unpack_kernel<false, kSrcPair, 1><<<grid_for(cap, nc, kPuWarps), kPuWarps * 32, kDyn, s>>>(
        packed_local, len, words, chunk_off, scale, do_scale, out, 0.f, nullptr, 0, nc, v, flags, target,
        err, sg, unpack_bulk_out());
  } else {
    static DeviceCache<int> cc;
    int& cap = cc.get();
    constexpr int kDyn = unpack_smem_bytes<kSrcOwner, 1>();
    if (!cap) cap = persistent_grid_dyn(unpack_kernel<false, kSrcOwner, 1>, kPuWarps, kDyn);
    unpack_kernel<false, kSrcOwner, 1><<<grid_for(cap, nc, kPuWarps), kPuWarps * 32, kDyn, s>>>(
        packed_local, len, words, chunk_off, scale, do_scale, out, 0.f, nullptr, 0, nc, v, flags, target,
        err, sg, unpack_bulk_out());
  }
  note_launch();
}

void launch_unpack_sgd(const float* packed, uint64_t len, const uint64_t* words,
                       const uint32_t* chunk_off, float scale, int do_scale, float lr,
                       float* grad_out, float* weights, cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  unpack_local<true>(packed, len, words, chunk_off, scale, do_scale, grad_out, lr, weights, 0, nc, s);
  note_launch();
}

void launch_gse(const float* g, uint64_t len, const uint64_t* words, float* out, cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  static int cap = 0;
  if (!cap) cap = persistent_grid(gse_kernel);
  gse_kernel<<<grid_for(cap, nc), kCodecWarps * 32, 0, s>>>(g, len, words, out, nc);
  note_launch();
}

void launch_scale(const float* in, float* out, uint64_t len, float scale, cudaStream_t s) {
  if (!len) return;
  uint64_t blocks = (len + 255) / 256;
  if (blocks > (uint64_t)sm_count() * 16) blocks = (uint64_t)sm_count() * 16;
  scale_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, len, scale);
  note_launch();
}

void launch_mask_fill(uint64_t* words, uint64_t len, int keep, uint32_t* chunk_off, cudaStream_t s) {
  const uint64_t nw = (len + 63) / 64, nc = (len + kChunk - 1) / kChunk;
  const uint64_t work = nw > nc + 1 ? nw : nc + 1;
  int grid = (int)((work + 255) / 256);
  if (grid > 4096) grid = 4096;
  mask_fill_kernel<<<grid, 256, 0, s>>>(words, nw, len, keep, chunk_off, nc);
  note_launch();
}

void launch_clear_tail(uint64_t* words, uint64_t len, cudaStream_t s) {
  if (!len || !(len & 63)) return;
  clear_tail_kernel<<<1, 1, 0, s>>>(words, len);
  note_launch();
}

namespace {
__global__ void words_differ_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b, uint64_t n16,
                                    int* __restrict__ flag) {
  bool d = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 x = __ldcs(a + i), y = __ldcs(b + i);
    d |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}
}  // namespace

void launch_words_differ(const uint64_t* a, const uint64_t* b, uint64_t nwords, int* flag, cudaStream_t s) {
  const uint64_t n16 = (nwords + 1) / 2;  // both padded to whole 16-word chunks
  if (!n16) return;
  uint64_t blocks = (n16 + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  words_differ_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(a),
                                                       reinterpret_cast<const uint4*>(b), n16, flag);
  note_launch();
}

void launch_tile_popc(const uint64_t* words, uint64_t len, uint32_t* popc, cudaStream_t s) {
  const uint64_t nc = (len + kChunk - 1) / kChunk;
  if (!nc) return;
  chunk_popc_kernel<<<(unsigned)((nc * 16 + 255) / 256), 256, 0, s>>>(words, (len + 63) / 64, popc, nc);
  note_launch();
}

void launch_mask_gather(const uint64_t* src, uint64_t src_len, const uint64_t* src_begin,
                        const uint64_t* dst_start, uint64_t nseg, uint64_t* dst, uint64_t dst_len,
                        uint64_t dst_words_padded, cudaStream_t s) {
  if (!dst_words_padded) return;
  uint64_t grid = (dst_words_padded + 255) / 256;
  if (grid > 8192) grid = 8192;
  mask_gather_kernel<<<(unsigned)grid, 256, 0, s>>>(src, (src_len + 63) / 64, src_begin, dst_start,
                                                    nseg, dst, dst_len, dst_words_padded);
  note_launch();
}

size_t scan_scratch_bytes(uint64_t n) { return ((n + kScanItems - 1) / kScanItems + 1) * 8 + 8; }

namespace {
__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, GatherIdx idx, uint32_t* __restrict__ out) {
  if ((int)threadIdx.x < idx.n) out[threadIdx.x] = src[idx.i[threadIdx.x]];
}
}  // namespace
void launch_gather_u32(const uint32_t* src, const GatherIdx& idx, uint32_t* out, cudaStream_t s) {
  gather_u32_kernel<<<1, 96, 0, s>>>(src, idx, out);
  note_launch();
}

void launch_scan_excl(const uint32_t* in, uint64_t n, uint32_t* out, void* scratch, cudaStream_t s) {
  const uint64_t tiles = n ? (n + kScanItems - 1) / kScanItems : 1;
  cudaMemsetAsync(scratch, 0, tiles * 8 + 8, s);
  uint64_t* state = static_cast<uint64_t*>(scratch);
  scan_excl_kernel<<<(unsigned)tiles, 1024, 0, s>>>(in, n, out, state,
                                                    reinterpret_cast<unsigned*>(state + tiles));
  note_launch();
}

}  // namespace pactk
