// cluster_test.cpp -- the reference's collective unit assertions
// (/root/reference/proj/tests/test_collective.cpp:46-285), rerun on real GPUs
// through the C++ drop-in header include/pact_b200.hpp. The reference runs
// its workers as threads of one process (SimCluster, test_collective.cpp:
// 23-35); here every worker is a PROCESS on its own GPU (the B200 topology:
// one process per GPU, NCCL + CUDA IPC), started by tests/test_cpp_dropin.py
// as `cluster_test <rank> <world> <id-file>`; rank 0 publishes the NCCL
// unique id through the file. Every rank rebuilds all ranks' inputs from the
// seeds, so each checks its own result against the whole-cluster oracle.
// Exit code = failed checks.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "pact_b200.hpp"

using namespace pact;

static std::atomic<int> g_fail{0};
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

static FlatTensor random_tensor(std::mt19937_64& g, size_t len) {  // test_collective.cpp:17-21
  std::normal_distribution<float> d(0.0f, 1.0f);
  std::vector<float> v(len);
  for (float& x : v) x = d(g);
  return FlatTensor(std::move(v));
}

static std::vector<double> sequential_sum(const std::vector<FlatTensor>& in) {  // :37-42
  std::vector<double> out(in[0].size(), 0.0);
  for (const auto& t : in)
    for (size_t i = 0; i < t.size(); ++i) out[i] += t[i];
  return out;
}

// per worker: a process (one rank each) or a thread of one process (all
// ranks, `cluster_test threads <world> <id-file>`: the reference's own
// SimCluster topology, every thread driving its own GPU)
static thread_local int g_rank = 0;
static int g_world = 0;
static const char* g_idfile = nullptr;
static thread_local int g_round = 0;

// fn(rank, comm) on the first n ranks (the others idle this round); one
// communicator per round, its unique id passed through <id-file>.<round>
template <typename Fn>
static void run_workers(int n, Fn fn) {
  const int round = g_round++;
  char path[512];
  std::snprintf(path, sizeof path, "%s.%d", g_idfile, round);
  if (g_rank >= n) return;
  std::vector<uint8_t> id(PACT_UNIQUE_ID_BYTES);
  if (g_rank == 0) {
    id = Comm::unique_id();
    char tmp[520];
    std::snprintf(tmp, sizeof tmp, "%s.tmp", path);
    FILE* f = std::fopen(tmp, "wb");
    std::fwrite(id.data(), 1, id.size(), f);
    std::fclose(f);
    std::rename(tmp, path);
  } else {
    for (int t = 0; t < 60000; ++t) {  // <= 60 s
      FILE* f = std::fopen(path, "rb");
      if (f) {
        const size_t got = std::fread(id.data(), 1, id.size(), f);
        std::fclose(f);
        if (got == id.size()) break;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  try {
    Comm comm(g_rank, n, id);
    fn(g_rank, comm);
  } catch (const std::exception& e) {
    std::printf("FAIL rank %d round %d: %s\n", g_rank, round, e.what());
    ++g_fail;
  }
}

static std::vector<bool> bits_of(size_t len, size_t off_bit, bool drop_extra, size_t extra) {
  std::vector<bool> b(len, true);
  b[off_bit] = false;
  if (drop_extra) b[extra] = false;
  return b;
}

static void body();

int main(int argc, char** argv) {
  if (argc < 4) {
    std::printf("usage: cluster_test <rank>|threads <world> <id-file>\n");
    return 2;
  }
  g_world = std::atoi(argv[2]);
  g_idfile = argv[3];
  if (std::string(argv[1]) == "threads") {
    std::vector<std::thread> th;
    for (int r = 0; r < g_world; ++r)
      th.emplace_back([r] {
        g_rank = r;
        detail::cuda(cudaSetDevice(r));
        body();
      });
    for (auto& t : th) t.join();
    std::printf("cluster_test threads x%d: %d failed check(s)\n", g_world, g_fail.load());
    return g_fail.load();
  }
  g_rank = std::atoi(argv[1]);
  detail::cuda(cudaSetDevice(g_rank));
  body();
  std::printf("cluster_test rank %d/%d: %d failed check(s)\n", g_rank, g_world, g_fail.load());
  return g_fail.load();
}

static void body() {
  const int ngpu = g_world;
  const int nmax = std::min(g_world, 4);
  const int r0 = g_rank;  // checks below look at this rank's own result

  // test_collective.cpp:46-54: two workers sum [1,2] and [3,4]
  {
    std::vector<FlatTensor> in{FlatTensor({1.0f, 2.0f}), FlatTensor({3.0f, 4.0f})};
    std::vector<FlatTensor> out(2);
    run_workers(2, [&](int r, Comm& c) { out[r] = full_allreduce(in[r], c).tensor; });
    if (r0 < 2) CHECK(out[r0].size() == 2 && out[r0][0] == 4.0f && out[r0][1] == 6.0f);
  }
  // :56-62 zeros stay zeros
  {
    std::vector<FlatTensor> out(nmax);
    run_workers(nmax, [&](int r, Comm& c) { out[r] = full_allreduce(FlatTensor::zeros(37), c).tensor; });
    if (r0 < nmax)
      for (size_t i = 0; i < out[r0].size(); ++i) CHECK(out[r0][i] == 0.0f);
  }
  // :210-244 masked allreduce on a stable mask halves the bytes
  {
    const int n = nmax;
    const size_t len = 100000;
    std::vector<bool> bits(len);
    for (size_t i = 0; i < len; ++i) bits[i] = (i % 2) == 0;
    std::mt19937_64 g(123);
    std::vector<FlatTensor> raw;
    for (int r = 0; r < n; ++r) raw.push_back(random_tensor(g, len));
    std::vector<SyncStats> ps(n), fs(n);
    std::vector<FlatTensor> po(n), fo(n);
    run_workers(n, [&](int r, Comm& c) {
      const SparsityMask mask = SparsityMask::from_bits(bits);  // device resident: one per GPU
      const FlatTensor grad = enforce_gradient_sparsity(raw[r], mask);
      auto a = masked_allreduce(grad, mask, TrackerStatus::Stable, 1, c);
      po[r] = std::move(a.tensor);
      ps[r] = a.stats;
      auto b = masked_allreduce(grad, mask, TrackerStatus::Unstable, 1, c);
      fo[r] = std::move(b.tensor);
      fs[r] = b.stats;
    });
    if (r0 < n) {
      CHECK(ps[r0].mode_used == SyncMode::PackedAllReduce);
      CHECK(fs[r0].mode_used == SyncMode::FullAllReduce);
      const double ratio = (double)ps[r0].bytes_on_wire / (double)fs[r0].bytes_on_wire;
      CHECK(ratio <= 0.51 && ratio >= 0.49);
      for (size_t i = 0; i < len; i += 97)
        CHECK(std::fabs(po[r0][i] - fo[r0][i]) <= 1e-5 * std::max(1.0f, std::fabs(fo[r0][i])));
    }
  }
  // :246-260 the unstable masked path equals the full path bit-for-bit
  {
    const int n = std::min(nmax, 3);
    std::mt19937_64 g(9);
    std::vector<FlatTensor> raw;
    for (int r = 0; r < n; ++r) raw.push_back(random_tensor(g, 257));
    std::vector<FlatTensor> a(n), b(n);
    run_workers(n, [&](int r, Comm& c) {
      const SparsityMask mask = SparsityMask::all_ones(257).with_bit(13, false);
      const FlatTensor grad = enforce_gradient_sparsity(raw[r], mask);
      a[r] = masked_allreduce(grad, mask, TrackerStatus::Unstable, 0, c).tensor;
      b[r] = full_allreduce(grad, c).tensor;
    });
    if (r0 < n) CHECK(a[r0] == b[r0]);
  }
  // :262-285 divergent masks trigger the fallback and still match the oracle
  {
    const int n = nmax;
    const size_t len = 300;
    std::mt19937_64 g(44);
    std::vector<FlatTensor> grads;
    for (int r = 0; r < n; ++r) grads.push_back(random_tensor(g, len));
    const auto expect = sequential_sum(grads);
    std::vector<SyncStats> st(n);
    std::vector<FlatTensor> out(n);
    run_workers(n, [&](int r, Comm& c) {
      const SparsityMask mine = SparsityMask::from_bits(bits_of(len, 5, r == n / 2, 6));  // one worker disagrees
      auto res = masked_allreduce(grads[r], mine, TrackerStatus::Stable, 7, c);
      out[r] = std::move(res.tensor);
      st[r] = res.stats;
    });
    if (r0 < n) {
      CHECK(st[r0].mode_used == SyncMode::FullAllReduce);
      for (size_t i = 0; i < len; ++i)
        CHECK(std::fabs(out[r0][i] - expect[i]) <= 1e-5 * std::max(1.0, std::fabs(expect[i])));
    }
  }
  // collective.cpp:165-216 ring_allreduce in the reference's own fold order:
  // bit-identical to ((x_c + x_{c+1}) + ...) + x_{c-1} per ChunkMap chunk c
  {
    const int n = nmax;
    {
      std::vector<FlatTensor> in;
      for (int r = 0; r < n; ++r) in.push_back(FlatTensor(std::vector<float>(n, r == 0 ? 1e8f : r == 1 ? -1e8f : 1.0f)));
      std::vector<FlatTensor> out(n);
      run_workers(n, [&](int r, Comm& c) { out[r] = ring_allreduce(in[r], c); });
      if (r0 < n) {
        const size_t len = in[0].size(), C = (len + n - 1) / n;
        for (size_t i = 0; i < len; ++i) {
          const int c = (int)(i / C);
          float acc = in[c][i];
          for (int s = 1; s < n; ++s) acc += in[(c + s) % n][i];
          CHECK(out[r0][i] == acc);  // n = 3: [1, 0, 0] (SURVEY A.6 probe)
        }
      }
    }
    std::mt19937_64 g(77);
    std::vector<FlatTensor> raw;
    for (int r = 0; r < n; ++r) raw.push_back(random_tensor(g, 100003));
    std::vector<FlatTensor> out(n);
    run_workers(n, [&](int r, Comm& c) { out[r] = ring_allreduce(raw[r], c); });
    if (r0 < n) {
      const size_t len = raw[0].size(), C = (len + n - 1) / n;
      for (size_t i = 0; i < len; ++i) {
        const int c = (int)(i / C);
        float acc = raw[c][i];
        for (int s = 1; s < n; ++s) acc += raw[(c + s) % n][i];
        CHECK(out[r0][i] == acc);
      }
    }
    // lengths that disagree: ShapeMismatch on every rank
    std::vector<int> code(n, -1);
    run_workers(n, [&](int r, Comm& c) {
      try {
        ring_allreduce(FlatTensor::zeros(r == 0 ? 11 : 10), c);
        code[r] = 0;
      } catch (const Error& e) {
        code[r] = (int)e.code();
      }
    });
    if (r0 < n) CHECK(code[r0] == (int)Errc::ShapeMismatch);
  }
  // collective.cpp:222-247 allgather: payloads of different sizes, by rank
  {
    const int n = nmax;
    std::vector<std::vector<std::vector<std::byte>>> got(n);
    run_workers(n, [&](int r, Comm& c) {
      got[r] = allgather(std::vector<std::byte>((size_t)r + 1, static_cast<std::byte>(r + 1)), c);
    });
    if (r0 < n) {
      CHECK((int)got[r0].size() == n);
      for (int q = 0; q < n && q < (int)got[r0].size(); ++q) {
        CHECK(got[r0][q].size() == (size_t)q + 1);
        for (auto b : got[r0][q]) CHECK(std::to_integer<int>(b) == q + 1);
      }
    }
  }
  // extension: the measured dense/sparse crossover is unanimous
  {
    const int n = 2;
    std::vector<double> thr(n, -1.0);
    run_workers(n, [&](int r, Comm& c) { thr[r] = calibrate_density(c, size_t{1} << 20); });
    if (r0 < n) {
      CHECK(thr[r0] > 0.0 && thr[r0] <= 1.0);
      // unanimous: the threshold summed over the ranks is n times this one
      std::vector<FlatTensor> tot(n);
      run_workers(n, [&](int r, Comm& c) { tot[r] = full_allreduce(FlatTensor({(float)thr[r]}), c).tensor; });
      CHECK(tot[r0][0] == (float)(n * (float)thr[r0]));
    } else {
      run_workers(n, [](int, Comm&) {});
    }
  }
  (void)ngpu;
}
