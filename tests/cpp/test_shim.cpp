// test_shim.cpp — the reference's own test assertions, restated against the
// drop-in header include/chw_b200/chw.hpp (proj/tests/transforms_test.cpp,
// tally_test.cpp, parallel_test.cpp, orderings_test.cpp; cited per check).
//   ./test_shim cpu   validation/geometry/tally checks that never touch a GPU
//   ./test_shim gpu   transforms on the GPU vs the C oracle (test infrastructure)
#include "chw_b200/chw.hpp"

#include <cstdio>
#include <cstring>
#include <random>
#include <string>

extern "C" {
int chw_oracle_chw_forward_f64(double* x, size_t n, int mode, uint64_t* adds, uint64_t* mults);
int chw_oracle_chw_forward_i64(int64_t* x, size_t n, int mode, uint64_t* adds, uint64_t* mults);
}

static int g_fail = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

template <class E, class F>
static bool throws_as(F&& f, const char* needle = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

using I = std::int64_t;
using namespace chw;
static constexpr auto kU = ScalingMode::Unnormalized;
static constexpr auto kO = ScalingMode::Orthonormal;

static void cpu_checks() {
  // transforms_test.cpp:77-86 — length / mode validation (thrown before any device work)
  std::vector<I> bad(3, 0);
  CHECK(throws_as<std::invalid_argument>([&] { chw_forward_inplace(std::span<I>(bad), kU); },
                                         "chw_forward: length 3 is not a power of two"));
  std::vector<I> empty;
  CHECK(throws_as<std::invalid_argument>([&] { chw_forward_inplace(std::span<I>(empty), kU); },
                                         "length 0 is not a power of two"));
  std::vector<I> two{1, 2};
  CHECK(throws_as<std::invalid_argument>([&] { chw_forward_inplace(std::span<I>(two), kO); },
                                         "orthonormal mode requires a floating-point signal"));
  CHECK(throws_as<std::invalid_argument>([&] { haar_forward_inplace(std::span<I>(bad), kU); },
                                         "haar_forward: length 3 is not a power of two"));
  CHECK(throws_as<std::invalid_argument>([&] { haar_forward_inplace(std::span<I>(empty), kU); }));
  CHECK(throws_as<std::invalid_argument>([&] { haar_forward_inplace(std::span<I>(two), kO); }));
  // transforms_test.cpp:88-110 — stage slices
  CHECK((stage_blocks(2, 1) == std::vector<BlockSlice>{{2, 2}}));
  CHECK((stage_blocks(4, 2) == std::vector<BlockSlice>{{4, 4}, {12, 4}}));
  CHECK((stage_blocks(4, 3) == std::vector<BlockSlice>{{2, 2}, {6, 2}, {10, 2}, {14, 2}}));
  CHECK(throws_as<std::invalid_argument>([] { stage_blocks(4, 0); }));
  CHECK(throws_as<std::invalid_argument>([] { stage_blocks(4, 4); }));
  for (int m = 2; m <= 12; ++m)
    for (int r = 1; r <= m - 1; ++r) {
      const auto blocks = stage_blocks(m, r);
      CHECK(blocks.size() == std::size_t{1} << (r - 1));
      std::size_t prev_end = 0;
      for (const auto& b : blocks) {
        CHECK(b.size == std::size_t{1} << (m - r));
        CHECK(b.offset % b.size == 0);
        CHECK(b.offset >= prev_end);
        prev_end = b.offset + b.size;
      }
    }
  // transforms_test.cpp:117-120 / tally_test.cpp:50-56 — length 1: identity, tally untouched
  OpTally t{3, 4};
  CHECK(chw_forward<I>({5}, kU, &t) == std::vector<I>{5});
  CHECK((t == OpTally{3, 4}));
  // tally_test.cpp:21-28
  OpTally r;
  r.additions = 5;
  r.multiplications = 7;
  r.reset();
  CHECK(r == OpTally{});
  // transforms_test.cpp:194-208 — normalize
  CHECK(normalized(std::vector<double>{5.0}, 0) == std::vector<double>{5.0});
  CHECK((normalized(std::vector<I>{1, 1, 1, 1}, 2) == std::vector<double>{0.5, 0.5, 0.5, 0.5}));
  std::vector<double> wrong(4, 0.0);
  CHECK(throws_as<std::invalid_argument>([&] { normalize_inplace(std::span<double>(wrong), 3); }));
  // parallel_test.cpp:83-88 — argument validation
  std::vector<I> x4{1, 2, 3, 4};
  CHECK(throws_as<std::invalid_argument>([&] { parallel_execute(x4, 0, kU); }, "workers must be >= 1, got 0"));
  std::vector<I> x3{1, 2, 3};
  CHECK(throws_as<std::invalid_argument>([&] { parallel_execute(x3, 2, kU); }));
  CHECK(throws_as<std::invalid_argument>([&] { parallel_execute(x4, 2, kO); }));
  // orderings_test.cpp:21-25
  CHECK(natural_to_dyadic(0).map == std::vector<std::uint32_t>{0});
  CHECK((natural_to_dyadic(2).map == std::vector<std::uint32_t>{0, 2, 1, 3}));
}

static void gpu_checks() {
  // transforms_test.cpp:112-121 — impulse KATs and the tally
  OpTally t;
  CHECK((chw_forward<I>({1, 0, 0, 0}, kU, &t) == std::vector<I>{1, 1, 1, 1}));
  CHECK(t.additions == 8);
  CHECK((chw_forward<I>({0, 1, 0, 0}, kU) == std::vector<I>{1, 1, -1, -1}));
  // transforms_test.cpp:134-143 — additions m*2^m (closed form, GPU result checked too)
  std::mt19937_64 rng(55);
  std::uniform_int_distribution<I> d(-1000, 1000);
  for (int m = 1; m <= 14; ++m) {
    std::vector<I> x(std::size_t{1} << m);
    for (auto& v : x) v = d(rng);
    std::vector<I> ref = x;
    chw_oracle_chw_forward_i64(ref.data(), ref.size(), 1, nullptr, nullptr);
    OpTally tt;
    chw_forward_inplace(std::span<I>(x), kU, &tt);
    CHECK(tt.additions == std::uint64_t(m) << m);
    CHECK(tt.multiplications == 0);
    CHECK(x == ref);
  }
  // Orthonormal double: bitwise equal to the reference algorithm (tally m*2^m mults)
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int m = 0; m <= 16; ++m) {
    std::vector<double> x(std::size_t{1} << m);
    for (auto& v : x) v = u(rng);
    std::vector<double> ref = x;
    chw_oracle_chw_forward_f64(ref.data(), ref.size(), 0, nullptr, nullptr);
    OpTally tt;
    const auto y = chw_forward(x, kO, &tt);
    CHECK(std::memcmp(y.data(), ref.data(), ref.size() * sizeof(double)) == 0);
    if (m > 0) CHECK(tt.multiplications == std::uint64_t(m) << m);
  }
  // tally_test.cpp:30-36 — cascade + normalize on length 16 tallies (64, 16)
  {
    std::vector<I> x(16);
    for (auto& v : x) v = d(rng);
    OpTally tt;
    const auto y = chw_forward(x, kU, &tt);
    normalized(y, 4, &tt);
    CHECK(tt.additions == 64 && tt.multiplications == 16);
  }
  // transforms_test.cpp:27-45 — Haar KATs and counts on the GPU
  {
    OpTally th;
    CHECK((haar_forward<I>({1, 0, 0, 0}, kU, &th) == std::vector<I>{1, 1, 1, 0}));
    CHECK(th.additions == 6);
    for (int m = 0; m <= 12; ++m) {
      std::vector<I> x(std::size_t{1} << m);
      for (auto& v : x) v = d(rng);
      OpTally t2;
      haar_forward_inplace(std::span<I>(x), kU, &t2);
      CHECK(t2.additions == 2 * ((std::uint64_t{1} << m) - 1));
    }
    std::vector<double> x(16);
    for (auto& v : x) v = u(rng);
    OpTally t3;
    haar_forward_inplace(std::span<double>(x), kO, &t3);
    CHECK(t3.additions == 30 && t3.multiplications == 30);
  }
  // transforms_test.cpp:145-170, orderings_test.cpp:79-84 — natural and dyadic FWHT
  {
    OpTally tf;
    CHECK((fwht_natural<I>({1, 0}, kU, &tf) == std::vector<I>{1, 1}));
    CHECK(tf.additions == 2);
    const std::vector<I> x{0, 1, 0, 0};
    const auto nat = fwht_natural(x, kU);
    CHECK((std::vector<I>{nat[0], nat[2], nat[1], nat[3]} == chw_forward(x, kU)));
    for (int m = 0; m <= 8; ++m) {
      std::vector<I> y(std::size_t{1} << m);
      for (auto& v : y) v = d(rng);
      CHECK(fwht_dyadic(y, kU) == chw_forward(y, kU));
    }
  }
  // parallel_test.cpp:21-58 — equal to serial for every worker count, bitwise for doubles
  for (int m : {2, 5, 9, 13}) {
    std::vector<I> x(std::size_t{1} << m);
    for (auto& v : x) v = d(rng);
    const auto serial = chw_forward(x, kU);
    for (int w : {1, 2, 4, 8}) CHECK(parallel_execute(x, w, kU) == serial);
  }
  for (int m : {3, 8, 11}) {
    std::vector<double> x(std::size_t{1} << m);
    for (auto& v : x) v = u(rng);
    const auto serial = chw_forward(x, kO);
    for (int w : {2, 4, 8}) {
      const auto p = parallel_execute(x, w, kO);
      CHECK(std::memcmp(p.data(), serial.data(), serial.size() * sizeof(double)) == 0);
    }
  }
  CHECK((parallel_execute<I>({42}, 8, kU) == std::vector<I>{42}));
  CHECK((parallel_execute<I>({1, 2}, 8, kU) == std::vector<I>{3, -1}));
  // batched overload, host buffer, 33 rows of 2^10 doubles
  {
    const std::size_t n = 1024, rows = 33;
    std::vector<double> x(n * rows);
    for (auto& v : x) v = u(rng);
    std::vector<double> ref = x;
    for (std::size_t r = 0; r < rows; ++r)
      chw_oracle_chw_forward_f64(ref.data() + r * n, n, 0, nullptr, nullptr);
    OpTally tt;
    chw_forward_batched_inplace(std::span<double>(x), n, kO, &tt);
    CHECK(std::memcmp(x.data(), ref.data(), x.size() * sizeof(double)) == 0);
    CHECK(tt.additions == rows * 10 * n);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_checks();
  if (mode == "gpu") gpu_checks();
  std::printf("%s: %s (%d failures)\n", mode.c_str(), g_fail ? "FAILED" : "ok", g_fail);
  return g_fail ? 1 : 0;
}
