// chw_b200_cli — the reference's command-line front end on the B200 backend
// (SURVEY §8 f4).  Mirrors proj/tools/chw_main.cpp's `transform`, `generate`
// and `bench` subcommands: same options, defaults, file formats, diagnostics
// on stderr / data on stdout, and exit codes (2 invalid argument or capacity,
// 3 format or I/O, 4 anything else).  `verify` (dense-matrix oracle) and
// `simulate` (task-graph simulator) are out of scope.
//
// Additions: `transform --rows R` treats the file as R concatenated signals of
// equal length and transforms them in one batched GPU call; `bench` times the
// GPU batched path and prints the reference's CSV columns.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "chw_b200/chw.hpp"
#include "chw_b200/signal_io.hpp"

namespace {

using namespace chw;

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --key value / --flag parser with allowed-value checks (CLI11's IsMember).
struct Args {
  std::map<std::string, std::string> kv;
  std::map<std::string, bool> flags;
  std::string get(const std::string& k, const std::string& def) const {
    auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  bool has(const std::string& k) const { return kv.count(k) != 0; }
};

Args parse(int argc, char** argv, int first, const std::map<std::string, std::string>& alias,
           const std::vector<std::string>& flag_names) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (alias.count(k)) k = alias.at(k);
    bool is_flag = false;
    for (const auto& f : flag_names)
      if (k == f) is_flag = true;
    if (is_flag) {
      a.flags[k] = true;
      continue;
    }
    if (k.rfind("--", 0) != 0) throw ParseError("unexpected argument '" + k + "'");
    if (i + 1 >= argc) throw ParseError(k + " requires a value");
    a.kv[k] = argv[++i];
  }
  return a;
}

void require(const Args& a, const std::string& k) {
  if (!a.has(k)) throw ParseError(k + " is required");
}
void member(const Args& a, const std::string& k, std::initializer_list<const char*> allowed) {
  if (!a.has(k)) return;
  for (const char* v : allowed)
    if (a.kv.at(k) == v) return;
  throw ParseError(k + ": '" + a.kv.at(k) + "' not in the allowed set");
}

SignalFormat fmt_of(const std::string& s) { return s == "binary" ? SignalFormat::Binary : SignalFormat::Text; }
ScalingMode mode_of(const std::string& s) {
  return s == "orthonormal" ? ScalingMode::Orthonormal : ScalingMode::Unnormalized;
}

template <SampleValue T>
std::vector<T> permute(const std::vector<T>& x, std::size_t rows, std::size_t n, const std::vector<uint32_t>& p) {
  std::vector<T> out(x.size());
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t i = 0; i < n; ++i) out[r * n + i] = x[r * n + p[i]];
  return out;
}

// chw_main.cpp:53-97, batched.
template <SampleValue T>
int run_transform(const Args& a) {
  const SignalFormat fmt = fmt_of(a.get("--format", "text"));
  const ScalingMode mode = mode_of(a.get("--mode", "unnormalized"));
  const std::string algo = a.get("--algo", "chw");
  const std::string order = a.get("--order", "");
  const std::size_t rows = a.has("--rows") ? std::stoull(a.kv.at("--rows")) : 0;
  // One signal: the reference's power-of-two count check; --rows R: any count
  // that splits into R power-of-two rows.
  std::vector<T> x = read_signal<T>(a.kv.at("--input"), fmt, rows ? 1 : 0);
  const std::size_t R = rows ? rows : 1;
  if (x.size() % R != 0) throw std::invalid_argument("--rows does not divide the sample count");
  const std::size_t n = x.size() / R;
  detail::require_pow2(n, "transform");
  const int m = level_of(n);
  OpTally tally;
  OpTally* tp = a.flags.count("--count-ops") ? &tally : nullptr;
  std::string native = "dyadic";
  if (algo == "chw") {
    if (R == 1)
      chw_forward_inplace(std::span<T>(x), mode, tp);
    else
      chw_forward_batched_inplace(std::span<T>(x), n, mode, tp);
  } else {
    for (std::size_t r = 0; r < R; ++r) {
      std::span<T> row(x.data() + r * n, n);
      if (algo == "fwht") {
        fwht_natural_inplace(row, mode, tp);
        native = "natural";
      } else if (algo == "haar") {
        haar_forward_inplace(row, mode, tp);
        native = "";
      } else {
        haar_walsh_forward_inplace(row, mode, tp);
      }
    }
  }
  if (!order.empty() && order != native) {
    if (native.empty()) throw std::invalid_argument("--order does not apply to the haar algorithm");
    std::vector<uint32_t> p(n);
    if (native == "natural") {  // to dyadic first
      for (std::size_t i = 0; i < n; ++i) p[i] = static_cast<uint32_t>(bit_reverse(i, m));
      x = permute(x, R, n, p);
    }
    if (order == "natural") {
      for (std::size_t i = 0; i < n; ++i) p[bit_reverse(i, m)] = static_cast<uint32_t>(i);
      x = permute(x, R, n, p);
    } else if (order == "sequency") {
      for (std::size_t i = 0; i < n; ++i) p[i] = static_cast<uint32_t>(gray_encode(i));
      x = permute(x, R, n, p);
    }
  }
  write_signal<T>(x, a.kv.at("--output"), fmt);
  if (tp) std::cerr << "additions=" << tally.additions << " multiplications=" << tally.multiplications << "\n";
  return 0;
}

// chw_main.cpp:279-304 — same generators, seeds and ranges.
int run_generate(const Args& a) {
  const int m = std::stoi(a.kv.at("--m"));
  if (m < 0 || m > 24) throw std::invalid_argument("generate: need 0 <= m <= 24");
  const std::size_t n = std::size_t{1} << m;
  const SignalFormat fmt = fmt_of(a.get("--format", "text"));
  const std::string kind = a.get("--kind", "random-int");
  std::mt19937_64 rng(std::stoull(a.get("--seed", "0")));
  if (kind == "random-float") {
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::vector<double> x(n);
    for (auto& v : x) v = dist(rng);
    write_signal<double>(x, a.kv.at("--output"), fmt);
  } else {
    std::vector<std::int64_t> x(n, 0);
    if (kind == "impulse") {
      x[0] = 1;
    } else {
      std::uniform_int_distribution<std::int64_t> dist(-1000, 1000);
      for (auto& v : x) v = dist(rng);
    }
    write_signal<std::int64_t>(x, a.kv.at("--output"), fmt);
  }
  return 0;
}

// chw_main.cpp:224-275 analogue for the GPU: CSV algo,n,reps,ns_per_element,additions.
int run_bench(const Args& a) {
  const int min_m = std::stoi(a.get("--min-m", "4"));
  const int max_m = std::stoi(a.get("--max-m", "20"));
  const int reps = std::stoi(a.get("--reps", "5"));
  const std::size_t rows = std::stoull(a.get("--rows", "1"));
  if (min_m < 1 || min_m > max_m || max_m > 24) throw std::invalid_argument("bench: need 1 <= min-m <= max-m <= 24");
  if (reps < 1) throw std::invalid_argument("bench: reps must be >= 1");
  std::mt19937_64 rng(std::stoull(a.get("--seed", "0")));
  std::uniform_int_distribution<std::int64_t> dist(-1000, 1000);
  std::cout << "algo,n,reps,ns_per_element,additions\n";
  using Clock = std::chrono::steady_clock;
  for (int m = min_m; m <= max_m; ++m) {
    const std::size_t n = std::size_t{1} << m;
    std::vector<std::int64_t> input(n * rows);
    for (auto& v : input) v = dist(rng);
    OpTally tally;
    std::vector<std::int64_t> buf = input;
    chw_forward_batched_inplace(std::span<std::int64_t>(buf), n, ScalingMode::Unnormalized, &tally);
    std::chrono::nanoseconds el{0};
    for (int r = 0; r < reps; ++r) {
      buf = input;
      const auto t0 = Clock::now();
      chw_forward_batched_inplace(std::span<std::int64_t>(buf), n, ScalingMode::Unnormalized);
      el += Clock::now() - t0;
    }
    const double ns = static_cast<double>(el.count()) / (static_cast<double>(reps) * n * rows);
    std::cout << (rows > 1 ? "chw-b200-x" + std::to_string(rows) : std::string("chw-b200")) << ',' << n << ','
              << reps << ',' << ns << ',' << tally.additions / rows << "\n";
  }
  return 0;
}

void usage() {
  std::cerr << "usage: chw_b200_cli <transform|generate|bench> [options]\n"
               "  transform -i FILE -o FILE [--algo chw|fwht|haar|haar-walsh] [--mode unnormalized|orthonormal]\n"
               "            [--order natural|dyadic|sequency] [--format text|binary] [--count-ops] [--rows R]\n"
               "  generate  -m M -o FILE [--format text|binary] [--kind random-int|random-float|impulse] [--seed S]\n"
               "  bench     [--min-m A] [--max-m B] [--reps K] [--rows R] [--seed S]\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 2;
  }
  const std::string cmd = argv[1];
  Args a;
  try {
    if (cmd == "transform") {
      a = parse(argc, argv, 2, {{"-i", "--input"}, {"-o", "--output"}}, {"--count-ops"});
      require(a, "--input");
      require(a, "--output");
      member(a, "--algo", {"chw", "fwht", "haar", "haar-walsh"});
      member(a, "--mode", {"unnormalized", "orthonormal"});
      member(a, "--order", {"natural", "dyadic", "sequency"});
      member(a, "--format", {"text", "binary"});
    } else if (cmd == "generate") {
      a = parse(argc, argv, 2, {{"-m", "--m"}, {"-o", "--output"}}, {});
      require(a, "--m");
      require(a, "--output");
      member(a, "--format", {"text", "binary"});
      member(a, "--kind", {"random-int", "random-float", "impulse"});
    } else if (cmd == "bench") {
      a = parse(argc, argv, 2, {}, {});
    } else if (cmd == "-h" || cmd == "--help") {
      usage();
      return 0;
    } else {
      throw ParseError("unknown subcommand '" + cmd + "'");
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    usage();
    return 2;
  }
  try {
    if (cmd == "transform")
      return mode_of(a.get("--mode", "unnormalized")) == ScalingMode::Unnormalized ? run_transform<std::int64_t>(a)
                                                                                   : run_transform<double>(a);
    if (cmd == "generate") return run_generate(a);
    return run_bench(a);
  } catch (const CapacityError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const FormatError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  }
}
