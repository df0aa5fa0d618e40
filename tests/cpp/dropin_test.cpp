// dropin_test.cpp -- the reference's own hot-path unit assertions
// (/root/reference/proj/tests/test_{tensor,sparsity,codec}.cpp), rerun
// against the C++ drop-in header include/pact_b200.hpp on the GPU.
// Built and run by tests/test_cpp_dropin.py. Exit code = failed checks.
#include <cmath>
#include <cstdio>
#include <random>

#include "pact_b200.hpp"

using namespace pact;

static int g_fail = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

template <typename F>
static Errc code_of(F f) {
  try {
    f();
  } catch (const Error& e) {
    return e.code();
  }
  return Errc::RunFailure;
}

int main() {
  // test_tensor.cpp:89-92, 130-135
  CHECK(SparsityMask::all_zeros(64).digest() == 0xa8c7f832281a39c5ULL);
  {
    SparsityMask m = SparsityMask::all_zeros(130).with_bit(0, true).with_bit(64, true).with_bit(129, true);
    CHECK(m.nnz() == 3);
    CHECK(m.test(0) && m.test(64) && m.test(129));
    CHECK(m.with_bit(64, false).nnz() == 2);
    CHECK(SparsityMask::all_ones(77).nnz() == 77);
  }
  // test_sparsity.cpp:13-47
  {
    SparsityMask m = magnitude_prune(FlatTensor({0.1f, -0.5f, 0.3f, 0.0f}), 0.5f);
    CHECK(m.nnz() == 2);
    CHECK(!m.test(0) && m.test(1) && m.test(2) && !m.test(3));
    CHECK(magnitude_prune(FlatTensor({0.1f, 0.2f, 0.3f}), 0.0f).nnz() == 3);
    CHECK(code_of([] { magnitude_prune(FlatTensor({1.0f}), 1.0f); }) == Errc::InvalidRatio);
    CHECK(code_of([] { magnitude_prune(FlatTensor({1.0f}), -0.1f); }) == Errc::InvalidRatio);
    SparsityMask t = magnitude_prune(FlatTensor({0.5f, -0.5f, 0.5f, 0.5f}), 0.5f);
    CHECK(!t.test(0) && !t.test(1) && t.test(2) && t.test(3));
  }
  // test_sparsity.cpp:49-69: sort oracle on gaussians
  {
    std::mt19937_64 rng(17);
    std::normal_distribution<float> nd;
    for (int trial = 0; trial < 20; ++trial) {
      std::vector<float> w(1000);
      for (auto& x : w) x = nd(rng);
      SparsityMask m = magnitude_prune(FlatTensor(w), 0.8f);
      CHECK(m.nnz() == 200);
      float min_kept = 1e30f, max_dropped = 0.0f;
      for (size_t i = 0; i < w.size(); ++i) {
        if (m.test(i))
          min_kept = std::fmin(min_kept, std::fabs(w[i]));
        else
          max_dropped = std::fmax(max_dropped, std::fabs(w[i]));
      }
      CHECK(min_kept >= max_dropped);
    }
  }
  // test_sparsity.cpp:162-202: GSE
  {
    FlatTensor out = enforce_gradient_sparsity(FlatTensor({0.2f, -0.3f, 0.7f}),
                                               SparsityMask::from_bits({false, true, false}));
    CHECK(out[0] == 0.0f && out[1] == -0.3f && out[2] == 0.0f);
    FlatTensor g({0.5f, -1.5f, 2.5f});
    CHECK(enforce_gradient_sparsity(g, SparsityMask::all_ones(3)) == g);
    CHECK(code_of([] { enforce_gradient_sparsity(FlatTensor({1.0f}), SparsityMask::all_ones(2)); }) ==
          Errc::ShapeMismatch);
  }
  // test_sparsity.cpp:204-222: tracker
  {
    MaskTracker t(3);
    SparsityMask a = SparsityMask::all_ones(8);
    CHECK(t.observe(a) == TrackerStatus::Unstable);
    CHECK(t.observe(a) == TrackerStatus::Unstable);
    CHECK(t.observe(a) == TrackerStatus::Unstable);
    CHECK(t.observe(a) == TrackerStatus::Stable);
    MaskTracker t2(2);
    SparsityMask b = a.with_bit(3, false);
    for (int i = 0; i < 10; ++i) {
      CHECK(t2.observe(a) == TrackerStatus::Unstable);
      CHECK(t2.observe(b) == TrackerStatus::Unstable);
    }
  }
  // test_codec.cpp:31-94: pack / unpack
  {
    SparsityMask m = SparsityMask::from_bits({false, true, false});
    PackedGradient p = pack(FlatTensor({0.0f, -0.3f, 0.0f}), m, 9);
    CHECK(p.values == std::vector<float>{-0.3f});
    CHECK(p.epoch == 9 && p.mask_digest == m.digest());
    FlatTensor g({1.0f, 2.0f, 3.0f});
    CHECK(pack(g, SparsityMask::all_ones(3), 0).values == g.values());
    FlatTensor g2({5.0f, -0.3f, 7.0f});
    CHECK(unpack(pack(g2, m, 0), m) == enforce_gradient_sparsity(g2, m));
    SparsityMask ones2 = SparsityMask::all_ones(2);
    PackedGradient bad = pack(FlatTensor({1.0f, 2.0f}), ones2, 0);
    bad.mask_digest ^= 1;
    CHECK(code_of([&] { unpack(bad, ones2); }) == Errc::MaskMismatch);
    SparsityMask ones3 = SparsityMask::all_ones(3);
    PackedGradient shortp{ones3.digest(), 0, {1.0f, 2.0f}};
    CHECK(code_of([&] { unpack(shortp, ones3); }) == Errc::CorruptPayload);
    std::mt19937_64 rng(11);
    std::uniform_real_distribution<double> u(0, 1);
    std::normal_distribution<float> nd;
    for (int trial = 0; trial < 200; ++trial) {
      const size_t len = 1 + rng() % 256;
      std::vector<float> v(len);
      std::vector<bool> bits(len);
      const double p_keep = u(rng);
      for (size_t i = 0; i < len; ++i) {
        v[i] = nd(rng);
        bits[i] = u(rng) < p_keep;
      }
      SparsityMask mm = SparsityMask::from_bits(bits);
      FlatTensor gg(v);
      CHECK(unpack(pack(gg, mm, trial), mm) == enforce_gradient_sparsity(gg, mm));
    }
  }
  // test_codec.cpp:247-274: header bytes
  {
    wire::Bytes b = wire::encode_header({wire::PayloadKind::Packed, 0x01020304u, 0x1122334455667788ULL, 5});
    CHECK(b.size() == 26);
    CHECK(std::to_integer<char>(b[0]) == 'P' && std::to_integer<uint8_t>(b[4]) == 1);
    CHECK(std::to_integer<uint8_t>(b[6]) == 0x04 && std::to_integer<uint8_t>(b[10]) == 0x88);
    wire::FrameHeader h = wire::decode_header(b);
    CHECK(h.kind == wire::PayloadKind::Packed && h.epoch == 0x01020304u && h.value_count == 5);
  }
  // test_collective.cpp:350-361: decide_sync_mode
  CHECK(decide_sync_mode(SyncMode::PackedAllReduce, TrackerStatus::Unstable) == SyncMode::FullAllReduce);
  CHECK(decide_sync_mode(SyncMode::PackedAllReduce, TrackerStatus::Stable) == SyncMode::PackedAllReduce);
  CHECK(decide_sync_mode(SyncMode::Fp16AllReduce, TrackerStatus::Unstable) == SyncMode::Fp16AllReduce);
  CHECK(code_of([] { Comm c(0, 1, Comm::unique_id()); }) == Errc::BadTopology);  // n >= 2

  // test_codec.cpp:96-136: ternarize / deternarize
  {
    TernaryGradient t = ternarize(FlatTensor({1.0f, -1.0f}), 123);
    CHECK(t.scale == 1.0f && t.sign_at(0) == 1 && t.sign_at(1) == -1);
    TernaryGradient z = ternarize(FlatTensor::zeros(9), 5);
    CHECK(z.scale == 0.0f);
    for (size_t i = 0; i < 9; ++i) CHECK(z.sign_at(i) == 0);
    std::mt19937_64 rng(13);
    std::normal_distribution<float> nd;
    std::vector<float> g(97);
    for (auto& x : g) x = nd(rng);
    TernaryGradient r = ternarize(FlatTensor(g), 31337);
    FlatTensor dec = deternarize(r);
    for (size_t i = 0; i < dec.size(); ++i) CHECK(dec[i] == r.scale || dec[i] == -r.scale || dec[i] == 0.0f);
    TernaryGradient bad;
    bad.scale = 1.0f;
    bad.len = 1;
    bad.sign_words = {0x3};
    CHECK(code_of([&] { bad.sign_at(0); }) == Errc::CorruptPayload);
    CHECK(code_of([&] { deternarize(bad); }) == Errc::CorruptPayload);
  }
  // codec.cpp:77-146: binary16 clamping and round trip
  {
    FlatTensor h = fp16_roundtrip(FlatTensor({1.0f, 65520.0f, -1e30f, 0.1f, 5.96e-8f}));
    CHECK(h[0] == 1.0f && h[1] == 65504.0f && h[2] == -65504.0f);
    CHECK(h[3] == 0.0999755859375f && h[4] == 5.9604644775390625e-8f);
  }
  // test_codec.cpp: topk: ties -> lower index, ascending
  {
    TopKPayload p = topk_select(FlatTensor({0.5f, -2.0f, 0.5f, 2.0f, 0.5f}), 0.6f);
    CHECK((p.indices == std::vector<uint32_t>{0, 1, 3}));
    CHECK((p.values == std::vector<float>{0.5f, -2.0f, 2.0f}));
    FlatTensor d = topk_densify(p);
    CHECK(d == FlatTensor({0.5f, -2.0f, 0.0f, 2.0f, 0.0f}));
    CHECK(code_of([] { topk_select(FlatTensor({1.0f}), 0.0f); }) == Errc::InvalidRate);
    TopKPayload oob{{7}, {1.0f}, 3};
    CHECK(code_of([&] { topk_densify(oob); }) == Errc::CorruptPayload);
  }

  // test_codec.cpp:276-287: packed frame payload size is 4*nnz + header
  {
    std::mt19937_64 rng(71);
    std::normal_distribution<float> nd;
    std::uniform_real_distribution<double> u(0, 1);
    std::vector<float> v(200);
    std::vector<bool> bits(200);
    for (size_t i = 0; i < 200; ++i) {
      v[i] = nd(rng);
      bits[i] = u(rng) < 0.4;
    }
    SparsityMask m = SparsityMask::from_bits(bits);
    PackedGradient p = pack(FlatTensor(v), m, 2);
    wire::Bytes b = wire::encode_packed(p);
    CHECK(b.size() == wire::kHeaderSize + 4 * m.nnz());
    PackedGradient back = wire::decode_packed(b);
    CHECK(back.values == p.values);
    CHECK(back.mask_digest == p.mask_digest);
    CHECK(back.epoch == p.epoch);
    b.pop_back();
    CHECK(code_of([&] { wire::decode_packed(b); }) == Errc::CorruptPayload);  // truncated
    CHECK(code_of([&] { wire::decode_packed(wire::encode_full(FlatTensor(v), 0)); }) == Errc::CorruptPayload);
    CHECK(wire::decode_full(wire::encode_full(FlatTensor(v), 3)) == FlatTensor(v));
  }
  // sparsity.cpp:11-15, 121-128: build_prune_mask(Magnitude) == magnitude_prune
  {
    std::mt19937_64 rng(5);
    std::normal_distribution<float> nd;
    std::vector<float> w(5000);
    for (auto& x : w) x = nd(rng);
    PruneConfig cfg;
    cfg.ratio = 0.7f;
    SparsityMask a = build_prune_mask(FlatTensor(w), cfg), b = magnitude_prune(FlatTensor(w), 0.7f);
    CHECK(a.words() == b.words() && a.nnz() == 1500);
    PruneConfig bad;
    bad.ratio = 1.0f;
    CHECK(code_of([&] { build_prune_mask(FlatTensor(w), bad); }) == Errc::InvalidRatio);
    PruneConfig eps;
    eps.grasp_epsilon = 0.0f;
    CHECK(code_of([&] { eps.validate(); }) == Errc::InvalidRatio);
    PruneConfig grasp;
    grasp.method = PruneMethod::Grasp;
    grasp.ratio = 0.5f;
    CHECK(code_of([&] { build_prune_mask(FlatTensor(w), grasp); }) == Errc::NumericalFailure);
  }

  std::printf("dropin_test: %d failure(s)\n", g_fail);
  return g_fail;
}
