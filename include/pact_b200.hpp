// pact_b200.hpp -- C++ drop-in for the reference hot-path API, on the B200
// C-ABI (include/pact_c.h). Header-only; link libpact_b200.so and cudart.
//
// Same names and signatures as the reference headers for the path
// (/root/reference/proj/include/pact/{tensor,sparsity,codec,collective}.hpp),
// same error contract (pact::Error carrying pact::Errc). Host `FlatTensor`
// overloads stage through the device (H2D -> sm_100a kernels -> D2H) so a
// reference caller can switch by changing its include path; device overloads
// (raw device pointers + cudaStream_t) are the zero-copy hot path.
//
// Differences: SparsityMask lives on the GPU (words()/test() copy back);
// Comm is an NCCL communicator (one process per GPU) created from a unique id
// instead of a ring Transport; SyncStats::seconds is measured device time.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pact_c.h"

namespace pact {

// ---------------------------------------------------------------- errors
enum class Errc {  // include/pact/error.hpp:10-26, same order
  DuplicateParam, InvalidView, InvalidRatio, InvalidRate, NumericalFailure, ShapeMismatch,
  MaskMismatch, CorruptPayload, LinkError, UndefinedMetric, MissingFile, ParseError, UnknownKey,
  BadTopology, RunFailure,
};

class Error : public std::runtime_error {  // error.hpp:51-62
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

namespace detail {
inline void check(pact_status st) {
  if (st == PACT_OK) return;
  const std::string msg = pact_last_error();
  if (st >= 1 && st <= 15) throw Error(static_cast<Errc>(st - 1), msg);
  throw Error(Errc::RunFailure, msg);  // CUDA / NCCL / argument failures
}
inline void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw Error(Errc::RunFailure, cudaGetErrorString(e));
}
inline pact_ctx* ctx() {  // one context per process-current device
  static thread_local int dev = -1;
  static thread_local pact_ctx* c = nullptr;
  int d = 0;
  cuda(cudaGetDevice(&d));
  if (!c || d != dev) {
    check(pact_ctx_create(d, &c));
    dev = d;
  }
  return c;
}
struct DevFree {
  void operator()(void* p) const { cudaFree(p); }
};
template <typename T>
std::unique_ptr<T, DevFree> dev_alloc(size_t n) {
  void* p = nullptr;
  cuda(cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
  return std::unique_ptr<T, DevFree>(static_cast<T*>(p));
}
}  // namespace detail

// ---------------------------------------------------------------- tensor
class FlatTensor {  // tensor.hpp:22-51 (host buffer)
 public:
  FlatTensor() = default;
  explicit FlatTensor(std::vector<float> v) : v_(std::move(v)) {}
  static FlatTensor zeros(size_t n) { return FlatTensor(std::vector<float>(n, 0.0f)); }
  size_t size() const { return v_.size(); }
  float operator[](size_t i) const { return v_[i]; }
  float& at(size_t i) { return v_[i]; }
  const float* data() const { return v_.data(); }
  float* data() { return v_.data(); }
  const std::vector<float>& values() const { return v_; }
  bool operator==(const FlatTensor& o) const { return v_ == o.v_; }

 private:
  std::vector<float> v_;
};

class SparsityMask {  // tensor.hpp:78-106, device resident
 public:
  SparsityMask() = default;
  explicit SparsityMask(size_t len) : m_(make(len)) {}

  static SparsityMask all_ones(size_t len) { return filled(len, 1); }
  static SparsityMask all_zeros(size_t len) { return filled(len, 0); }
  static SparsityMask from_bits(const std::vector<bool>& bits) {  // tensor.cpp:97-105
    std::vector<uint64_t> w((bits.size() + 63) / 64, 0);
    for (size_t i = 0; i < bits.size(); ++i)
      if (bits[i]) w[i >> 6] |= uint64_t{1} << (i & 63);
    return from_words(w, bits.size());
  }
  static SparsityMask from_words(const std::vector<uint64_t>& w, size_t len) {
    SparsityMask m(len);
    auto d = detail::dev_alloc<uint64_t>(w.size());
    detail::cuda(cudaMemcpy(d.get(), w.data(), w.size() * 8, cudaMemcpyHostToDevice));
    detail::check(pact_mask_set_words(m.m_.get(), d.get(), nullptr));
    return m;
  }
  SparsityMask with_bit(size_t i, bool keep) const {  // tensor.cpp:107-115
    std::vector<uint64_t> w = words();
    if (keep)
      w[i >> 6] |= uint64_t{1} << (i & 63);
    else
      w[i >> 6] &= ~(uint64_t{1} << (i & 63));
    return from_words(w, size());
  }

  size_t size() const { return info().len; }
  size_t nnz() const { return info().nnz; }
  uint64_t digest() const {
    uint64_t d = 0;
    detail::check(pact_mask_digest(m_.get(), nullptr, &d));
    return d;
  }
  std::vector<uint64_t> words() const {
    const pact_mask_info i = info();
    std::vector<uint64_t> w((i.len + 63) / 64);
    detail::cuda(cudaMemcpy(w.data(), i.words, w.size() * 8, cudaMemcpyDeviceToHost));
    return w;
  }
  bool test(size_t i) const { return (words()[i >> 6] >> (i & 63)) & 1u; }
  bool operator==(const SparsityMask& o) const { return size() == o.size() && words() == o.words(); }

  pact_mask* handle() const { return m_.get(); }

 private:
  struct Del {
    void operator()(pact_mask* m) const { pact_mask_destroy(m); }
  };
  static std::shared_ptr<pact_mask> make(size_t len) {
    pact_mask* m = nullptr;
    detail::check(pact_mask_create(detail::ctx(), len, &m));
    return std::shared_ptr<pact_mask>(m, Del{});
  }
  static SparsityMask filled(size_t len, int keep) {
    SparsityMask m(len);
    detail::check(pact_mask_fill(m.m_.get(), keep, nullptr));
    return m;
  }
  pact_mask_info info() const {
    pact_mask_info i{};
    detail::check(pact_mask_info_get(m_.get(), &i));
    return i;
  }
  std::shared_ptr<pact_mask> m_;
};

inline uint64_t mask_digest(const SparsityMask& m) { return m.digest(); }

// -------------------------------------------------------------- sparsity
enum class TrackerStatus { Stable, Unstable };

class MaskTracker {  // sparsity.hpp:37-54
 public:
  explicit MaskTracker(uint32_t stability_threshold = 3) { pact_tracker_init(&t_, stability_threshold); }
  TrackerStatus observe(const SparsityMask& mask) { return observe_digest(mask.digest()); }
  TrackerStatus observe_digest(uint64_t d) {
    return pact_tracker_observe(&t_, d) ? TrackerStatus::Stable : TrackerStatus::Unstable;
  }
  TrackerStatus status() const {
    return pact_tracker_status(&t_) ? TrackerStatus::Stable : TrackerStatus::Unstable;
  }
  uint32_t stable_count() const { return t_.stable_count; }
  std::optional<uint64_t> last_digest() const {
    return t_.has_last ? std::optional<uint64_t>(t_.last_digest) : std::nullopt;
  }

 private:
  pact_tracker t_{};
};

inline TrackerStatus tracker_observe(MaskTracker& t, const SparsityMask& m) { return t.observe(m); }

// device overload: weights already on the GPU
inline SparsityMask magnitude_prune(const float* d_weights, size_t len, float ratio,
                                    cudaStream_t s = nullptr) {
  uint64_t k;
  detail::check(pact_drop_count(ratio, len, &k));  // InvalidRatio before any allocation
  SparsityMask m(len);
  detail::check(pact_prune_magnitude(detail::ctx(), d_weights, len, ratio, m.handle(), s, nullptr));
  return m;
}

// sparsity.cpp:44-59
inline SparsityMask magnitude_prune(const FlatTensor& weights, float ratio) {
  uint64_t k;
  detail::check(pact_drop_count(ratio, weights.size(), &k));
  auto d = detail::dev_alloc<float>(weights.size());
  detail::cuda(cudaMemcpy(d.get(), weights.data(), weights.size() * 4, cudaMemcpyHostToDevice));
  return magnitude_prune(d.get(), weights.size(), ratio);
}

// sparsity.hpp:15-31, sparsity.cpp:11-15. GraSP (PruneMethod::Grasp) is off
// the gradient-sync path (out of scope): build_prune_mask rejects it.
enum class PruneMethod { Magnitude, Grasp };
enum class GraspKeep { MostNegative, MostPositive };
struct PruneConfig {
  float ratio = 0.0f;  // fraction of elements to drop, in [0, 1)
  PruneMethod method = PruneMethod::Magnitude;
  float grasp_epsilon = 1e-2f;
  GraspKeep grasp_keep = GraspKeep::MostNegative;
  void validate() const {
    if (!(ratio >= 0.0f && ratio < 1.0f))
      throw Error(Errc::InvalidRatio, "prune ratio " + std::to_string(ratio) + " outside [0, 1)");
    if (!(grasp_epsilon > 0.0f)) throw Error(Errc::InvalidRatio, "grasp_epsilon must be positive");
  }
};
using GradientFn = std::function<FlatTensor(const FlatTensor&)>;  // sparsity.hpp:69

// sparsity.cpp:121-128
inline SparsityMask build_prune_mask(const FlatTensor& weights, const PruneConfig& cfg,
                                     const GradientFn& grad_of = nullptr) {
  cfg.validate();
  if (cfg.method == PruneMethod::Magnitude) return magnitude_prune(weights, cfg.ratio);
  if (!grad_of) throw Error(Errc::NumericalFailure, "gradient-flow pruning needs a gradient function");
  throw Error(Errc::RunFailure, "GraSP pruning is not part of the B200 gradient-sync path");
}

// sparsity.cpp:112-119
inline FlatTensor enforce_gradient_sparsity(const FlatTensor& grad, const SparsityMask& mask) {
  if (grad.size() != mask.size()) throw Error(Errc::ShapeMismatch, "gradient/mask length mismatch");
  auto d = detail::dev_alloc<float>(grad.size());
  detail::cuda(cudaMemcpy(d.get(), grad.data(), grad.size() * 4, cudaMemcpyHostToDevice));
  detail::check(pact_gse(detail::ctx(), d.get(), grad.size(), mask.handle(), d.get(), nullptr));
  std::vector<float> out(grad.size());
  detail::cuda(cudaMemcpy(out.data(), d.get(), out.size() * 4, cudaMemcpyDeviceToHost));
  return FlatTensor(std::move(out));
}

// ----------------------------------------------------------------- codec
struct PackedGradient {  // codec.hpp:19-23
  uint64_t mask_digest = 0;
  uint32_t epoch = 0;
  std::vector<float> values;
};

inline PackedGradient pack(const FlatTensor& grad, const SparsityMask& mask, uint32_t epoch) {
  if (grad.size() != mask.size()) throw Error(Errc::ShapeMismatch, "gradient/mask length mismatch");
  const size_t n = grad.size(), k = mask.nnz();
  auto dg = detail::dev_alloc<float>(n);
  auto dp = detail::dev_alloc<float>(k);
  detail::cuda(cudaMemcpy(dg.get(), grad.data(), n * 4, cudaMemcpyHostToDevice));
  detail::check(pact_pack(detail::ctx(), dg.get(), n, mask.handle(), dp.get(), 0, UINT64_MAX, nullptr));
  PackedGradient p{mask.digest(), epoch, std::vector<float>(k)};
  detail::cuda(cudaMemcpy(p.values.data(), dp.get(), k * 4, cudaMemcpyDeviceToHost));
  return p;
}

inline FlatTensor unpack(const PackedGradient& p, const SparsityMask& mask) {  // codec.cpp:27-38
  const size_t n = mask.size();
  auto dp = detail::dev_alloc<float>(p.values.size());
  auto dout = detail::dev_alloc<float>(n);
  detail::cuda(cudaMemcpy(dp.get(), p.values.data(), p.values.size() * 4, cudaMemcpyHostToDevice));
  detail::check(pact_unpack(detail::ctx(), dp.get(), p.values.size(), p.mask_digest, 1, mask.handle(),
                            1.0f, dout.get(), 0, UINT64_MAX, nullptr));
  std::vector<float> out(n);
  detail::cuda(cudaMemcpy(out.data(), dout.get(), n * 4, cudaMemcpyDeviceToHost));
  return FlatTensor(std::move(out));
}

// codec.cpp:40-75: ternary payload (host copy of the device result)
struct TernaryGradient {  // codec.hpp:32-40
  float scale = 0.0f;
  size_t len = 0;
  std::vector<uint8_t> sign_words;  // 4 elements per byte, little-endian pairs
  int sign_at(size_t i) const {
    const uint8_t pair = (sign_words[i >> 2] >> (2 * (i & 3))) & 0x3;
    if (pair == 3) throw Error(Errc::CorruptPayload, "reserved ternary sign pattern 11");
    return pair == 1 ? 1 : (pair == 2 ? -1 : 0);
  }
};

// codec.cpp:50-68; draws from a counter-based SplitMix64 stream of `seed`
// (pact_c.h: the reference's sequential mt19937_64 stream is replaced)
inline TernaryGradient ternarize(const FlatTensor& grad, uint64_t seed) {
  const size_t n = grad.size();
  auto dg = detail::dev_alloc<float>(n);
  auto ds = detail::dev_alloc<uint8_t>(pact_ternary_sign_bytes(n));
  auto dsc = detail::dev_alloc<float>(1);
  detail::cuda(cudaMemcpy(dg.get(), grad.data(), n * 4, cudaMemcpyHostToDevice));
  detail::check(pact_ternarize(detail::ctx(), dg.get(), n, seed, dsc.get(), ds.get(), nullptr));
  TernaryGradient t;
  t.len = n;
  t.sign_words.resize((n + 3) / 4);
  detail::cuda(cudaMemcpy(&t.scale, dsc.get(), 4, cudaMemcpyDeviceToHost));
  detail::cuda(cudaMemcpy(t.sign_words.data(), ds.get(), t.sign_words.size(), cudaMemcpyDeviceToHost));
  return t;
}

inline FlatTensor deternarize(const TernaryGradient& t) {  // codec.cpp:70-75
  const size_t sb = pact_ternary_sign_bytes(t.len);
  std::vector<uint8_t> padded(sb ? sb : 1, 0);
  std::memcpy(padded.data(), t.sign_words.data(), std::min(t.sign_words.size(), padded.size()));
  auto ds = detail::dev_alloc<uint8_t>(padded.size());
  auto dsc = detail::dev_alloc<float>(1);
  auto dout = detail::dev_alloc<float>(t.len);
  detail::cuda(cudaMemcpy(ds.get(), padded.data(), padded.size(), cudaMemcpyHostToDevice));
  detail::cuda(cudaMemcpy(dsc.get(), &t.scale, 4, cudaMemcpyHostToDevice));
  detail::check(pact_deternarize(detail::ctx(), dsc.get(), ds.get(), t.len, dout.get(), nullptr));
  std::vector<float> out(t.len);
  detail::cuda(cudaMemcpy(out.data(), dout.get(), t.len * 4, cudaMemcpyDeviceToHost));
  return FlatTensor(std::move(out));
}

inline FlatTensor fp16_roundtrip(const FlatTensor& grad) {  // codec.cpp:142-146
  auto d = detail::dev_alloc<float>(grad.size());
  detail::cuda(cudaMemcpy(d.get(), grad.data(), grad.size() * 4, cudaMemcpyHostToDevice));
  detail::check(pact_fp16_roundtrip(detail::ctx(), d.get(), d.get(), grad.size(), nullptr));
  std::vector<float> out(grad.size());
  detail::cuda(cudaMemcpy(out.data(), d.get(), out.size() * 4, cudaMemcpyDeviceToHost));
  return FlatTensor(std::move(out));
}

struct TopKPayload {  // codec.hpp:60-66
  std::vector<uint32_t> indices;
  std::vector<float> values;
  size_t original_len = 0;
};

inline TopKPayload topk_select(const FlatTensor& grad, float rate) {  // codec.cpp:147-172
  uint64_t k = 0;
  detail::check(pact_topk_count(grad.size(), rate, &k));
  auto dg = detail::dev_alloc<float>(grad.size());
  auto di = detail::dev_alloc<uint32_t>(k);
  auto dv = detail::dev_alloc<float>(k);
  detail::cuda(cudaMemcpy(dg.get(), grad.data(), grad.size() * 4, cudaMemcpyHostToDevice));
  detail::check(pact_topk_select(detail::ctx(), dg.get(), grad.size(), rate, di.get(), dv.get(), &k, nullptr));
  TopKPayload p{std::vector<uint32_t>(k), std::vector<float>(k), grad.size()};
  detail::cuda(cudaMemcpy(p.indices.data(), di.get(), k * 4, cudaMemcpyDeviceToHost));
  detail::cuda(cudaMemcpy(p.values.data(), dv.get(), k * 4, cudaMemcpyDeviceToHost));
  return p;
}

inline FlatTensor topk_densify(const TopKPayload& p) {  // codec.cpp:174-182
  const size_t k = p.indices.size();
  auto di = detail::dev_alloc<uint32_t>(k);
  auto dv = detail::dev_alloc<float>(k);
  auto dout = detail::dev_alloc<float>(p.original_len);
  detail::cuda(cudaMemcpy(di.get(), p.indices.data(), k * 4, cudaMemcpyHostToDevice));
  detail::cuda(cudaMemcpy(dv.get(), p.values.data(), k * 4, cudaMemcpyHostToDevice));
  detail::check(pact_topk_densify(detail::ctx(), di.get(), dv.get(), k, p.original_len, dout.get(), nullptr));
  std::vector<float> out(p.original_len);
  detail::cuda(cudaMemcpy(out.data(), dout.get(), out.size() * 4, cudaMemcpyDeviceToHost));
  return FlatTensor(std::move(out));
}

namespace wire {  // codec.hpp:80-103
enum class PayloadKind : uint8_t { Full = 0, Packed = 1, Ternary = 2, Fp16 = 3, TopK = 4 };
inline constexpr size_t kHeaderSize = PACT_HEADER_BYTES;
struct FrameHeader {
  PayloadKind kind = PayloadKind::Full;
  uint32_t epoch = 0;
  uint64_t mask_digest = 0;
  uint64_t value_count = 0;
};
using Bytes = std::vector<std::byte>;
inline Bytes encode_header(const FrameHeader& h) {
  pact_frame_header c{static_cast<uint8_t>(h.kind), h.epoch, h.mask_digest, h.value_count};
  Bytes b(kHeaderSize);
  detail::check(pact_header_encode(&c, reinterpret_cast<uint8_t*>(b.data())));
  return b;
}
inline FrameHeader decode_header(const Bytes& f) {
  pact_frame_header c{};
  detail::check(pact_header_decode(reinterpret_cast<const uint8_t*>(f.data()), f.size(), &c));
  return {static_cast<PayloadKind>(c.kind), c.epoch, c.mask_digest, c.value_count};
}
namespace detail {
inline void put_f32s(Bytes& b, const float* v, size_t n) {  // little-endian binary32 (codec.cpp:214-218)
  const size_t o = b.size();
  b.resize(o + 4 * n);
  for (size_t i = 0; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, v + i, 4);
    for (int k = 0; k < 4; ++k) b[o + 4 * i + k] = static_cast<std::byte>((u >> (8 * k)) & 0xffu);
  }
}
inline void get_f32s(const Bytes& b, size_t off, float* v, size_t n) {  // codec.cpp:220-237
  for (size_t i = 0; i < n; ++i) {
    uint32_t u = 0;
    for (int k = 0; k < 4; ++k) u |= static_cast<uint32_t>(std::to_integer<uint8_t>(b[off + 4 * i + k])) << (8 * k);
    std::memcpy(v + i, &u, 4);
  }
}
inline void need(const Bytes& b, size_t n) {  // codec.cpp:239-241
  if (b.size() < n) throw Error(Errc::CorruptPayload, "frame truncated");
}
}  // namespace detail
// codec.cpp:277-291
inline Bytes encode_full(const FlatTensor& grad, uint32_t epoch) {
  Bytes b = encode_header({PayloadKind::Full, epoch, 0, grad.size()});
  detail::put_f32s(b, grad.data(), grad.size());
  return b;
}
inline FlatTensor decode_full(const Bytes& frame) {
  const FrameHeader h = decode_header(frame);
  if (h.kind != PayloadKind::Full) throw Error(Errc::CorruptPayload, "not a full frame");
  detail::need(frame, kHeaderSize + h.value_count * 4);
  std::vector<float> v(h.value_count);
  detail::get_f32s(frame, kHeaderSize, v.data(), v.size());
  return FlatTensor(std::move(v));
}
// codec.cpp:293-311
inline Bytes encode_packed(const PackedGradient& packed) {
  Bytes b = encode_header({PayloadKind::Packed, packed.epoch, packed.mask_digest, packed.values.size()});
  detail::put_f32s(b, packed.values.data(), packed.values.size());
  return b;
}
inline PackedGradient decode_packed(const Bytes& frame) {
  const FrameHeader h = decode_header(frame);
  if (h.kind != PayloadKind::Packed) throw Error(Errc::CorruptPayload, "not a packed frame");
  detail::need(frame, kHeaderSize + h.value_count * 4);
  PackedGradient p;
  p.mask_digest = h.mask_digest;
  p.epoch = h.epoch;
  p.values.resize(h.value_count);
  detail::get_f32s(frame, kHeaderSize, p.values.data(), p.values.size());
  return p;
}
}  // namespace wire

// ------------------------------------------------------------ collective
enum class SyncMode : uint8_t { FullAllReduce, PackedAllReduce, TernaryAllGather, TopKAllGather, Fp16AllReduce };

inline SyncMode decide_sync_mode(SyncMode requested, TrackerStatus t) {  // collective.cpp:62-67
  return static_cast<SyncMode>(
      pact_decide_sync_mode(static_cast<int>(requested), t == TrackerStatus::Stable));
}

struct SyncStats {  // collective.hpp:73-77
  uint64_t bytes_on_wire = 0;
  double seconds = 0.0;
  SyncMode mode_used = SyncMode::FullAllReduce;
};

struct AggregateResult {  // collective.hpp:130-133
  FlatTensor tensor;
  SyncStats stats;
};

class Comm {  // collective.hpp:89-116, NCCL-backed
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(PACT_UNIQUE_ID_BYTES);
    detail::check(pact_comm_unique_id(id.data()));
    return id;
  }
  Comm(int rank, int n, const std::vector<uint8_t>& id) {
    pact_comm* c = nullptr;
    detail::check(pact_comm_create(detail::ctx(), id.data(), n, rank, &c));
    c_.reset(c);
  }
  int rank() const { return pact_comm_rank(c_.get()); }
  int world_size() const { return pact_comm_size(c_.get()); }
  pact_comm* handle() const { return c_.get(); }

 private:
  struct Del {
    void operator()(pact_comm* c) const { pact_comm_destroy(c); }
  };
  std::unique_ptr<pact_comm, Del> c_;
};

// collective.cpp:269-309; returns the SUM. `policy` (extension):
// the adaptive knobs, e.g. density_threshold from calibrate_density.
inline AggregateResult masked_allreduce(const FlatTensor& grad, const SparsityMask& mask,
                                        TrackerStatus tracker, uint32_t epoch, Comm& comm,
                                        std::optional<uint64_t> advertised_digest = {},
                                        const pact_policy& policy = pact_policy{}) {
  if (grad.size() != mask.size()) throw Error(Errc::ShapeMismatch, "gradient/mask length mismatch");
  std::vector<float> out(grad.size());
  pact_sync_stats st{};
  pact_policy pol = policy;
  uint64_t adv = advertised_digest.value_or(0);
  detail::check(pact_masked_allreduce_host(comm.handle(), detail::ctx(), grad.data(), grad.size(),
                                           mask.handle(), tracker == TrackerStatus::Stable, epoch,
                                           advertised_digest ? &adv : nullptr, &pol, out.data(), &st,
                                           nullptr));
  return {FlatTensor(std::move(out)),
          {st.bytes_on_wire, st.seconds, static_cast<SyncMode>(st.mode_used)}};
}

// Extension (north_star (4)): the measured crossover density above which
// the dense allreduce is faster than pack -> packed allreduce -> unpack on
// this communicator for gradients of `len` elements. Collective.
inline double calibrate_density(Comm& comm, size_t len) {
  double thr = 1.0;
  detail::check(pact_calibrate_density(comm.handle(), detail::ctx(), len, nullptr, nullptr, 0, nullptr, nullptr,
                                       &thr, nullptr));
  return thr;
}

// collective.cpp:165-216: the SUM with the reference ring's own fold order,
// bit-identical on every rank (NVLink peer memory; ShapeMismatch when the
// ranks' lengths differ)
inline FlatTensor ring_allreduce(const FlatTensor& local, Comm& comm) {
  auto d = detail::dev_alloc<float>(local.size());
  detail::cuda(cudaMemcpy(d.get(), local.data(), local.size() * 4, cudaMemcpyHostToDevice));
  detail::check(pact_ring_allreduce(comm.handle(), d.get(), d.get(), local.size(), nullptr));
  std::vector<float> out(local.size());
  detail::cuda(cudaMemcpy(out.data(), d.get(), out.size() * 4, cudaMemcpyDeviceToHost));
  return FlatTensor(std::move(out));
}

// collective.cpp:222-247: every rank ends with all n payloads, indexed by
// rank (payload sizes may differ: the sizes go first, then padded frames)
inline std::vector<std::vector<std::byte>> allgather(const std::vector<std::byte>& payload, Comm& comm) {
  const int n = comm.world_size();
  const uint64_t mine = payload.size();
  std::vector<uint64_t> sizes(n);
  detail::check(pact_allgather_frames(comm.handle(), reinterpret_cast<const uint8_t*>(&mine), 8,
                                      reinterpret_cast<uint8_t*>(sizes.data()), nullptr));
  const uint64_t mx = std::max<uint64_t>(1, *std::max_element(sizes.begin(), sizes.end()));
  std::vector<uint8_t> frame(mx, 0), all((size_t)n * mx);
  std::memcpy(frame.data(), payload.data(), payload.size());
  detail::check(pact_allgather_frames(comm.handle(), frame.data(), mx, all.data(), nullptr));
  std::vector<std::vector<std::byte>> out(n);
  for (int r = 0; r < n; ++r) {
    out[r].resize(sizes[r]);
    std::memcpy(out[r].data(), all.data() + (size_t)r * mx, sizes[r]);
  }
  return out;
}

// collective.cpp:253-259; returns the SUM
inline AggregateResult full_allreduce(const FlatTensor& grad, Comm& comm) {
  auto d = detail::dev_alloc<float>(grad.size());
  detail::cuda(cudaMemcpy(d.get(), grad.data(), grad.size() * 4, cudaMemcpyHostToDevice));
  pact_sync_stats st{};
  detail::check(pact_full_allreduce(comm.handle(), d.get(), d.get(), grad.size(), 1.0f, &st, nullptr));
  std::vector<float> out(grad.size());
  detail::cuda(cudaMemcpy(out.data(), d.get(), out.size() * 4, cudaMemcpyDeviceToHost));
  return {FlatTensor(std::move(out)), {st.bytes_on_wire, st.seconds, SyncMode::FullAllReduce}};
}

namespace detail {
// host-buffer aggregate call: H2D grad, device path, D2H result
template <typename F>
AggregateResult host_aggregate(const FlatTensor& grad, F&& call) {
  auto d = dev_alloc<float>(grad.size());
  auto o = dev_alloc<float>(grad.size());
  cuda(cudaMemcpy(d.get(), grad.data(), grad.size() * 4, cudaMemcpyHostToDevice));
  pact_sync_stats st{};
  call(d.get(), o.get(), &st);
  std::vector<float> out(grad.size());
  cuda(cudaMemcpy(out.data(), o.get(), out.size() * 4, cudaMemcpyDeviceToHost));
  return {FlatTensor(std::move(out)), {st.bytes_on_wire, st.seconds, static_cast<SyncMode>(st.mode_used)}};
}
}  // namespace detail

// collective.cpp:311-368; returns the MEAN
inline AggregateResult ternary_allgather_aggregate(const FlatTensor& grad, const SparsityMask& mask,
                                                   TrackerStatus tracker, uint64_t seed, uint32_t epoch,
                                                   Comm& comm) {
  if (grad.size() != mask.size()) throw Error(Errc::ShapeMismatch, "gradient/mask length mismatch");
  return detail::host_aggregate(grad, [&](float* d, float* o, pact_sync_stats* st) {
    detail::check(pact_ternary_allgather_aggregate(comm.handle(), detail::ctx(), d, grad.size(), mask.handle(),
                                                   tracker == TrackerStatus::Stable, seed, epoch, o, st,
                                                   nullptr));
  });
}

// collective.cpp:370-390; returns the MEAN
inline AggregateResult topk_allgather_aggregate(const FlatTensor& grad, float rate, uint32_t epoch,
                                                Comm& comm) {
  return detail::host_aggregate(grad, [&](float* d, float* o, pact_sync_stats* st) {
    detail::check(pact_topk_allgather_aggregate(comm.handle(), detail::ctx(), d, grad.size(), rate, epoch, o,
                                                st, nullptr));
  });
}

// collective.cpp:261-267 (binary16 ring, F16Wire); returns the SUM
inline AggregateResult fp16_allreduce(const FlatTensor& grad, Comm& comm) {
  return detail::host_aggregate(grad, [&](float* d, float* o, pact_sync_stats* st) {
    detail::check(pact_fp16_allreduce(comm.handle(), detail::ctx(), d, o, grad.size(), st, nullptr));
  });
}

}  // namespace pact
