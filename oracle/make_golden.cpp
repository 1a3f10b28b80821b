// make_golden.cpp — golden-vector generator (TEST INFRASTRUCTURE ONLY).
//
// Runs the UNMODIFIED reference (headers from /root/reference/proj/include via
// -I) on inputs drawn exactly as the reference's own tests draw them
// (proj/tests/test_support.hpp:13-26: std::mt19937_64(seed), ints uniform in
// [-bound, bound], reals uniform [-1, 1)), with the seeds of the test cases it
// mirrors.  Writes <outdir>/index.txt ("name dtype count" per line) plus one
// raw little-endian .bin per array.  tests/golden/make_golden.py packs them into
// tests/golden/golden.npz, which the tests read (the GPU box has no reference).

#include <chw/oracle.hpp>
#include <chw/orderings.hpp>
#include <chw/transforms.hpp>

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <random>
#include <string>
#include <vector>

using I = std::int64_t;
using chw::ScalingMode;

namespace {

std::string g_dir;
std::ofstream g_index;

template <class T>
void emit(const std::string& name, const std::vector<T>& v) {
  const char* dt = std::is_same_v<T, double> ? "f64" : (std::is_same_v<T, I> ? "i64" : "u64");
  g_index << name << ' ' << dt << ' ' << v.size() << '\n';
  std::ofstream f(g_dir + "/" + name + ".bin", std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

std::vector<I> rand_int(std::mt19937_64& rng, size_t n, I bound = 1000) {
  std::uniform_int_distribution<I> d(-bound, bound);
  std::vector<I> x(n);
  for (auto& v : x) v = d(rng);
  return x;
}
std::vector<double> rand_real(std::mt19937_64& rng, size_t n) {
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  std::vector<double> x(n);
  for (auto& v : x) v = d(rng);
  return x;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: make_golden <outdir>\n");
    return 2;
  }
  g_dir = argv[1];
  g_index.open(g_dir + "/index.txt");
  const auto U = ScalingMode::Unnormalized;
  const auto O = ScalingMode::Orthonormal;

  // transforms_test.cpp:112-121 — impulse KATs and the length-1 identity.
  {
    chw::OpTally t;
    emit("kat_impulse0_out", chw::chw_forward<I>({1, 0, 0, 0}, U, &t));
    emit("kat_impulse0_tally", std::vector<std::uint64_t>{t.additions, t.multiplications});
    emit("kat_impulse1_out", chw::chw_forward<I>({0, 1, 0, 0}, U));
    chw::OpTally t1;
    emit("kat_len1_out", chw::chw_forward<I>({9}, U, &t1));
    emit("kat_len1_tally", std::vector<std::uint64_t>{t1.additions, t1.multiplications});
    chw::OpTally th;
    emit("kat_haar_out", chw::haar_forward<I>({1, 0, 0, 0}, U, &th));
    emit("kat_haar_tally", std::vector<std::uint64_t>{th.additions, th.multiplications});
  }
  // transforms_test.cpp:123-132 — CHW == dense dyadic, exact int, seed 44.
  {
    std::mt19937_64 rng(44);
    for (int m = 0; m <= 8; ++m) {
      const auto h = chw::hadamard_dyadic_dense<I>(m, U);
      std::vector<I> xs, ys, ds;
      for (int trial = 0; trial < 20; ++trial) {
        const auto x = rand_int(rng, size_t{1} << m);
        const auto y = chw::chw_forward(x, U);
        const auto d = chw::mat_vec(h, x);
        xs.insert(xs.end(), x.begin(), x.end());
        ys.insert(ys.end(), y.begin(), y.end());
        ds.insert(ds.end(), d.begin(), d.end());
      }
      emit("dense_int_m" + std::to_string(m) + "_in", xs);
      emit("dense_int_m" + std::to_string(m) + "_out", ys);
      emit("dense_int_m" + std::to_string(m) + "_dense", ds);
    }
  }
  // transforms_test.cpp:134-143 — additions == m*2^m, seed 55.
  {
    std::mt19937_64 rng(55);
    std::vector<std::uint64_t> adds, mults;
    for (int m = 1; m <= 14; ++m) {
      auto x = rand_int(rng, size_t{1} << m);
      chw::OpTally t;
      chw::chw_forward_inplace(std::span<I>(x), U, &t);
      adds.push_back(t.additions);
      mults.push_back(t.multiplications);
    }
    emit("count_adds_m1_14", adds);
    emit("count_mults_m1_14", mults);
  }
  // transforms_test.cpp:36-45 — Haar additions, seed 11.
  {
    std::mt19937_64 rng(11);
    std::vector<std::uint64_t> adds;
    for (int m = 0; m <= 12; ++m) {
      auto x = rand_int(rng, size_t{1} << m);
      chw::OpTally t;
      chw::haar_forward_inplace(std::span<I>(x), U, &t);
      adds.push_back(t.additions);
    }
    emit("haar_adds_m0_12", adds);
  }
  // transforms_test.cpp:241-248 — orthonormal vs dense (<= 1e-12), seed 333.
  {
    std::mt19937_64 rng(333);
    for (int m = 0; m <= 8; ++m) {
      const auto x = rand_real(rng, size_t{1} << m);
      chw::OpTally t;
      emit("ortho_m" + std::to_string(m) + "_in", x);
      emit("ortho_m" + std::to_string(m) + "_out", chw::chw_forward(x, O, &t));
      emit("ortho_m" + std::to_string(m) + "_dense",
           chw::mat_vec(chw::hadamard_dyadic_dense<double>(m, O), x));
      emit("ortho_m" + std::to_string(m) + "_tally",
           std::vector<std::uint64_t>{t.additions, t.multiplications});
    }
  }
  // transforms_test.cpp:228-239 — Parseval cases, seed 222.
  {
    std::mt19937_64 rng(222);
    for (int m : {1, 4, 8, 12}) {
      const auto x = rand_real(rng, size_t{1} << m);
      emit("parseval_m" + std::to_string(m) + "_in", x);
      emit("parseval_m" + std::to_string(m) + "_out", chw::chw_forward(x, O));
    }
  }
  // transforms_test.cpp:160-170 and 172-192 — fwht_dyadic, Haar-Walsh (seeds 77, 88).
  {
    std::mt19937_64 rng(77);
    for (int m = 0; m <= 8; ++m) {
      const auto x = rand_int(rng, size_t{1} << m);
      emit("fwhtdy_m" + std::to_string(m) + "_in", x);
      emit("fwhtdy_m" + std::to_string(m) + "_out", chw::fwht_dyadic(x, U));
      emit("fwhtnat_m" + std::to_string(m) + "_out", chw::fwht_natural(x, U));
    }
    std::mt19937_64 rng2(88);
    const auto h7 = rand_int(rng2, 128);
    emit("haarwalsh_m7_in", h7);
    emit("haarwalsh_m7_out", chw::haar_walsh_forward(h7, U));
    emit("haarwalsh_m7_dense", chw::mat_vec(chw::haar_walsh_dense<I>(7), h7));
  }
  // Multi-row f64 fixtures at the cfg1 row length and a sweep of m, drawn the
  // way `chw generate --kind random-float` draws (chw_main.cpp:290-294).
  {
    std::mt19937_64 rng(1609066410ULL);
    std::vector<double> xs, ys;
    for (int r = 0; r < 16; ++r) {
      const auto x = rand_real(rng, 1024);
      const auto y = chw::chw_forward(x, O);
      xs.insert(xs.end(), x.begin(), x.end());
      ys.insert(ys.end(), y.begin(), y.end());
    }
    emit("cfg1_rows16_in", xs);
    emit("cfg1_rows16_out", ys);
    std::mt19937_64 rng3(7);
    for (int m = 0; m <= 14; ++m) {
      const auto x = rand_real(rng3, size_t{1} << m);
      emit("sweep_f64_m" + std::to_string(m) + "_in", x);
      emit("sweep_f64_m" + std::to_string(m) + "_ortho", chw::chw_forward(x, O));
      emit("sweep_f64_m" + std::to_string(m) + "_unnorm", chw::chw_forward(x, U));
    }
    std::mt19937_64 rng4(8);
    for (int m = 0; m <= 14; ++m) {
      const auto x = rand_int(rng4, size_t{1} << m);
      emit("sweep_i64_m" + std::to_string(m) + "_in", x);
      emit("sweep_i64_m" + std::to_string(m) + "_out", chw::chw_forward(x, U));
    }
  }
  // orderings_test.cpp:37-41 — closed-form permutations.
  {
    std::vector<std::uint64_t> p;
    for (auto v : chw::natural_to_dyadic(4).map) p.push_back(v);
    emit("perm_nat2dy_m4", p);
    std::vector<std::uint64_t> g;
    for (auto v : chw::dyadic_to_sequency(4).map) g.push_back(v);
    emit("perm_dy2seq_m4", g);
  }
  return 0;
}
