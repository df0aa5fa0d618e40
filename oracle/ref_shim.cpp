// ref_shim.cpp -- C entry points over the UNMODIFIED reference hot path.
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile together with the
// reference's own sources (/root/reference/proj/src/{tensor,sparsity,codec,
// collective}.cpp, compiled in place, namespace renamed with -Dpact=pactref)
// into oracle/_ref/libpactref.so. Used to pin the C restatement
// (oracle/pact_oracle.c), to generate tests/golden/ fixtures, and as the CPU
// baseline arm of bench.py. Nothing under paper_2505_18563_b200/ links it.
//
// Every function catches pactref::Error and returns its Errc as 1 + enum
// index (the oracle's status convention); 0 = ok.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <thread>
#include <vector>

#include "pact/codec.hpp"
#include "pact/collective.hpp"
#include "pact/sparsity.hpp"
#include "pact/tensor.hpp"

using namespace pact;  // == pactref under -Dpact=pactref

namespace {

int code_of(const Error& e) { return 1 + static_cast<int>(e.code()); }

std::vector<bool> bits_of(const uint64_t* words, size_t len) {
  std::vector<bool> b(len);
  for (size_t i = 0; i < len; ++i) b[i] = (words[i >> 6] >> (i & 63)) & 1u;
  return b;
}

void copy_words(const SparsityMask& m, uint64_t* out) {
  std::memcpy(out, m.words().data(), m.words().size() * sizeof(uint64_t));
}

template <typename Fn>
int guarded(Fn fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    return code_of(e);
  } catch (...) {
    return 1 + static_cast<int>(Errc::RunFailure);
  }
}

// tests/test_collective.cpp:24-35 pattern: n worker threads on one SimCluster
template <typename Fn>
void run_workers(int n, Fn fn) {
  SimCluster cluster(n);
  WorkerTopology topo = WorkerTopology::uniform(n, {1e9, 0.0});
  std::vector<std::thread> threads;
  std::vector<std::exception_ptr> errs(n);
  for (int r = 0; r < n; ++r)
    threads.emplace_back([&, r] {
      try {
        Comm comm(topo, r, cluster.transport_at(r));
        fn(r, comm);
      } catch (...) {
        errs[r] = std::current_exception();
        cluster.poison();
      }
    });
  for (auto& t : threads) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

int ref_magnitude_prune(const float* w, size_t len, float ratio, uint64_t* words, uint64_t* nnz,
                        uint64_t* digest) {
  return guarded([&] {
    SparsityMask m = magnitude_prune(FlatTensor(std::vector<float>(w, w + len)), ratio);
    copy_words(m, words);
    *nnz = m.nnz();
    *digest = m.digest();
  });
}

int ref_mask_from_words(const uint64_t* words, size_t len, uint64_t* nnz, uint64_t* digest) {
  return guarded([&] {
    SparsityMask m = SparsityMask::from_bits(bits_of(words, len));
    *nnz = m.nnz();
    *digest = m.digest();
  });
}

int ref_gse(const float* g, const uint64_t* words, size_t glen, size_t mlen, float* out) {
  return guarded([&] {
    FlatTensor r = enforce_gradient_sparsity(FlatTensor(std::vector<float>(g, g + glen)),
                                             SparsityMask::from_bits(bits_of(words, mlen)));
    std::memcpy(out, r.data(), r.size() * sizeof(float));
  });
}

int ref_pack(const float* g, const uint64_t* words, size_t glen, size_t mlen, uint32_t epoch,
             float* packed, uint64_t* count, uint64_t* digest) {
  return guarded([&] {
    PackedGradient p = pack(FlatTensor(std::vector<float>(g, g + glen)),
                            SparsityMask::from_bits(bits_of(words, mlen)), epoch);
    std::memcpy(packed, p.values.data(), p.values.size() * sizeof(float));
    *count = p.values.size();
    *digest = p.mask_digest;
  });
}

int ref_unpack(const float* packed, uint64_t count, uint64_t packed_digest, const uint64_t* words,
               size_t len, float* out) {
  return guarded([&] {
    PackedGradient p{packed_digest, 0, std::vector<float>(packed, packed + count)};
    FlatTensor r = unpack(p, SparsityMask::from_bits(bits_of(words, len)));
    std::memcpy(out, r.data(), r.size() * sizeof(float));
  });
}

int ref_encode_header(uint8_t kind, uint32_t epoch, uint64_t digest, uint64_t count,
                      uint8_t out[26]) {
  return guarded([&] {
    wire::Bytes b = wire::encode_header(
        {static_cast<wire::PayloadKind>(kind), epoch, digest, count});
    std::memcpy(out, b.data(), b.size());
  });
}

int ref_decode_header(const uint8_t* in, size_t len, uint8_t* kind, uint32_t* epoch,
                      uint64_t* digest, uint64_t* count) {
  return guarded([&] {
    wire::Bytes b(len);
    std::memcpy(b.data(), in, len);
    wire::FrameHeader h = wire::decode_header(b);
    *kind = static_cast<uint8_t>(h.kind);
    *epoch = h.epoch;
    *digest = h.mask_digest;
    *count = h.value_count;
  });
}

// MaskTracker over a digest sequence (words supplied as all_ones/with_bit
// would be too indirect: the tracker only consumes digests, so masks are
// synthesised per distinct digest index).
int ref_tracker_sequence(uint32_t threshold, const uint64_t* const* masks, const size_t* lens,
                         const int* seq, size_t nseq, int* status_out) {
  return guarded([&] {
    MaskTracker t(threshold);
    for (size_t i = 0; i < nseq; ++i) {
      SparsityMask m = SparsityMask::from_bits(bits_of(masks[seq[i]], lens[seq[i]]));
      status_out[i] = t.observe(m) == TrackerStatus::Stable ? 1 : 0;
    }
  });
}

int ref_decide_sync_mode(int requested, int stable) {
  return static_cast<int>(decide_sync_mode(static_cast<SyncMode>(requested),
                                           stable ? TrackerStatus::Stable : TrackerStatus::Unstable));
}

int ref_ring_allreduce(int n, const float* const* in, size_t len, float* const* out,
                       uint64_t* bytes_out) {
  return guarded([&] {
    run_workers(n, [&](int r, Comm& c) {
      FlatTensor s = ring_allreduce(FlatTensor(std::vector<float>(in[r], in[r] + len)), c);
      std::memcpy(out[r], s.data(), len * sizeof(float));
      bytes_out[r] = c.bytes_sent();
    });
  });
}

int ref_full_allreduce(int n, const float* const* in, size_t len, float* const* out,
                       uint64_t* bytes_out) {
  return guarded([&] {
    run_workers(n, [&](int r, Comm& c) {
      AggregateResult a = full_allreduce(FlatTensor(std::vector<float>(in[r], in[r] + len)), c);
      std::memcpy(out[r], a.tensor.data(), len * sizeof(float));
      bytes_out[r] = a.stats.bytes_on_wire;
    });
  });
}

int ref_masked_allreduce(int n, const float* const* grads, const uint64_t* const* masks,
                         const int* stable, const uint64_t* advertised_or_null, uint32_t epoch,
                         size_t len, float* const* out, int* mode_out, uint64_t* bytes_out) {
  return guarded([&] {
    run_workers(n, [&](int r, Comm& c) {
      std::optional<uint64_t> adv;
      if (advertised_or_null) adv = advertised_or_null[r];
      AggregateResult a = masked_allreduce(
          FlatTensor(std::vector<float>(grads[r], grads[r] + len)),
          SparsityMask::from_bits(bits_of(masks[r], len)),
          stable[r] ? TrackerStatus::Stable : TrackerStatus::Unstable, epoch, c, adv);
      std::memcpy(out[r], a.tensor.data(), len * sizeof(float));
      mode_out[r] = a.stats.mode_used == SyncMode::PackedAllReduce ? 1 : 0;
      bytes_out[r] = a.stats.bytes_on_wire;
    });
  });
}

// ------------------------------------------------------ TopK

int ref_topk_select(const float* g, size_t len, float rate, uint32_t* idx, float* val, uint64_t* k_out) {
  return guarded([&] {
    TopKPayload p = topk_select(FlatTensor(std::vector<float>(g, g + len)), rate);
    std::memcpy(idx, p.indices.data(), p.indices.size() * 4);
    std::memcpy(val, p.values.data(), p.values.size() * 4);
    *k_out = p.indices.size();
  });
}

int ref_topk_densify(const uint32_t* idx, const float* val, size_t k, size_t len, float* out) {
  return guarded([&] {
    TopKPayload p;
    p.indices.assign(idx, idx + k);
    p.values.assign(val, val + k);
    p.original_len = len;
    FlatTensor d = topk_densify(p);
    std::memcpy(out, d.data(), len * sizeof(float));
  });
}

int ref_topk_decode_check(const uint8_t* frame, size_t bytes, size_t original_len, uint64_t* k_out) {
  return guarded([&] {
    wire::Bytes b(bytes);
    std::memcpy(b.data(), frame, bytes);
    TopKPayload p = wire::decode_topk(b, original_len);
    *k_out = p.indices.size();
  });
}

int ref_topk_aggregate(int n, const float* const* grads, size_t len, float rate, uint32_t epoch,
                       float* const* out, uint64_t* bytes_out) {
  return guarded([&] {
    run_workers(n, [&](int r, Comm& c) {
      AggregateResult a =
          topk_allgather_aggregate(FlatTensor(std::vector<float>(grads[r], grads[r] + len)), rate, epoch, c);
      std::memcpy(out[r], a.tensor.data(), len * sizeof(float));
      bytes_out[r] = a.stats.bytes_on_wire;
    });
  });
}

// -------------------------------------------------- binary16

void ref_float_to_half(const float* in, size_t n, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = float_to_half(in[i]);
}
void ref_half_to_float(const uint16_t* in, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = half_to_float(in[i]);
}

int ref_fp16_allreduce(int n, const float* const* in, size_t len, float* const* out,
                       uint64_t* bytes_out) {
  return guarded([&] {
    run_workers(n, [&](int r, Comm& c) {
      AggregateResult a = fp16_allreduce(FlatTensor(std::vector<float>(in[r], in[r] + len)), c);
      std::memcpy(out[r], a.tensor.data(), len * sizeof(float));
      bytes_out[r] = a.stats.bytes_on_wire;
    });
  });
}

// ------------------------------------------------- ternary

int ref_ternarize(const float* v, size_t n, uint64_t seed, float* scale_out, uint8_t* sign_bytes) {
  return guarded([&] {
    TernaryGradient t = ternarize(FlatTensor(std::vector<float>(v, v + n)), seed);
    *scale_out = t.scale;
    std::memcpy(sign_bytes, t.sign_words.data(), t.sign_words.size());
  });
}

int ref_deternarize(float scale, const uint8_t* sign_bytes, size_t n, float* out) {
  return guarded([&] {
    TernaryGradient t;
    t.scale = scale;
    t.len = n;
    t.sign_words.assign(sign_bytes, sign_bytes + (n + 3) / 4);
    FlatTensor d = deternarize(t);
    std::memcpy(out, d.data(), n * sizeof(float));
  });
}

// wire::decode_ternary on a raw frame; scale/len/digest out, sign bytes copied
int ref_decode_ternary(const uint8_t* frame, size_t bytes, float* scale, uint64_t* len,
                       uint64_t* digest, uint8_t* sign_bytes) {
  return guarded([&] {
    wire::Bytes b(bytes);
    std::memcpy(b.data(), frame, bytes);
    uint64_t d = 0;
    TernaryGradient t = wire::decode_ternary(b, &d);
    *scale = t.scale;
    *len = t.len;
    *digest = d;
    if (sign_bytes) std::memcpy(sign_bytes, t.sign_words.data(), t.sign_words.size());
  });
}

int ref_encode_ternary(float scale, const uint8_t* sign_bytes, size_t n, uint32_t epoch,
                       uint64_t digest, uint8_t* out, size_t* out_bytes) {
  return guarded([&] {
    TernaryGradient t;
    t.scale = scale;
    t.len = n;
    t.sign_words.assign(sign_bytes, sign_bytes + (n + 3) / 4);
    wire::Bytes b = wire::encode_ternary(t, epoch, digest);
    std::memcpy(out, b.data(), b.size());
    *out_bytes = b.size();
  });
}

// ternary_allgather_aggregate over SimCluster (collective.cpp:311-368)
int ref_ternary_aggregate(int n, const float* const* grads, const uint64_t* const* masks,
                          const int* stable, const uint64_t* seeds, uint32_t epoch, size_t len,
                          float* const* out, int* mode_out, uint64_t* bytes_out) {
  return guarded([&] {
    run_workers(n, [&](int r, Comm& c) {
      AggregateResult a = ternary_allgather_aggregate(
          FlatTensor(std::vector<float>(grads[r], grads[r] + len)),
          SparsityMask::from_bits(bits_of(masks[r], len)),
          stable[r] ? TrackerStatus::Stable : TrackerStatus::Unstable, seeds[r], epoch, c);
      std::memcpy(out[r], a.tensor.data(), len * sizeof(float));
      mode_out[r] = static_cast<int>(a.stats.mode_used);
      bytes_out[r] = a.stats.bytes_on_wire;
    });
  });
}

// ---------------------------------------------------------------------------
// CPU baseline arm: prepared inputs so only the reference call is timed.
// ---------------------------------------------------------------------------

struct RefBench {
  int n = 0;
  size_t len = 0;
  std::vector<FlatTensor> grads;         // one per simulated worker
  std::unique_ptr<SparsityMask> mask;    // shared global mask
  // per-thread slices for the n=1 (pack -> unpack) arm
  std::vector<FlatTensor> slice_grads;
  std::vector<SparsityMask> slice_masks;
};

void* ref_bench_create(int n, const float* const* grads, const uint64_t* words, size_t len,
                       int slices) {
  auto* b = new RefBench;
  b->n = n;
  b->len = len;
  for (int r = 0; r < n; ++r) b->grads.emplace_back(std::vector<float>(grads[r], grads[r] + len));
  b->mask = std::make_unique<SparsityMask>(SparsityMask::from_bits(bits_of(words, len)));
  if (slices > 0) {
    const size_t per = (len + slices - 1) / slices;
    for (int s = 0; s < slices; ++s) {
      size_t lo = std::min(len, per * s), hi = std::min(len, per * (s + 1));
      std::vector<bool> bits(hi - lo);
      for (size_t i = lo; i < hi; ++i) bits[i - lo] = (words[i >> 6] >> (i & 63)) & 1u;
      b->slice_grads.emplace_back(std::vector<float>(grads[0] + lo, grads[0] + hi));
      b->slice_masks.push_back(SparsityMask::from_bits(bits));
    }
  }
  return b;
}

void ref_bench_destroy(void* h) { delete static_cast<RefBench*>(h); }

// reference masked_allreduce (tracker Stable) over SimCluster, n threads;
// returns wall seconds of the whole collective (thread spawn to join).
double ref_bench_masked(void* h, uint32_t epoch) {
  auto* b = static_cast<RefBench*>(h);
  auto t0 = std::chrono::steady_clock::now();
  run_workers(b->n, [&](int r, Comm& c) {
    AggregateResult a = masked_allreduce(b->grads[r], *b->mask, TrackerStatus::Stable, epoch, c);
    (void)a;
  });
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// n=1 arm: reference pack -> unpack on every slice, one thread per slice.
double ref_bench_pack_unpack(void* h, uint32_t epoch) {
  auto* b = static_cast<RefBench*>(h);
  const size_t ns = b->slice_grads.size();
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (size_t s = 0; s < ns; ++s)
    th.emplace_back([&, s] {
      PackedGradient p = pack(b->slice_grads[s], b->slice_masks[s], epoch);
      FlatTensor u = unpack(p, b->slice_masks[s]);
      (void)u;
    });
  for (auto& t : th) t.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// single-thread reference magnitude_prune on the given weights (seconds)
double ref_bench_prune(const float* w, size_t len, float ratio) {
  FlatTensor t(std::vector<float>(w, w + len));
  auto t0 = std::chrono::steady_clock::now();
  SparsityMask m = magnitude_prune(t, ratio);
  (void)m;
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
