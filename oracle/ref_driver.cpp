// ref_driver.cpp — C-ABI wrapper around the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no transform arithmetic of its
// own: it includes the reference headers straight from
// /root/reference/proj/include (via -I in oracle/Makefile, never copied) and
// links the reference's own src/parallel.cpp + src/schedule.cpp, so that
// oracle/_ref/libchw_ref.so is the reference's CPU implementation behind a C
// ABI.  Used to (1) generate tests/golden/ fixtures, (2) validate the C
// restatement in oracle/chw_oracle.c, and (3) time the reference CPU path in
// bench.py (cpu_baseline.kind = "reference", --impl reference).
//
// Return codes: 0 ok, -1 std::invalid_argument, -3 chw::StructureError,
// -4 chw::ResourceError, -9 anything else.  The exception text is kept in a
// thread-local buffer readable via ref_last_error().

#include <chw/common.hpp>
#include <chw/errors.hpp>
#include <chw/op_tally.hpp>
#include <chw/orderings.hpp>
#include <chw/parallel.hpp>
#include <chw/transforms.hpp>

#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

chw::ScalingMode to_mode(int mode) {
  return mode == 0 ? chw::ScalingMode::Orthonormal : chw::ScalingMode::Unnormalized;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const chw::StructureError& e) {
    g_err = e.what();
    return -3;
  } catch (const chw::ResourceError& e) {
    g_err = e.what();
    return -4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

void fill_tally(const chw::OpTally& t, uint64_t* adds, uint64_t* mults) {
  if (adds) *adds = t.additions;
  if (mults) *mults = t.multiplications;
}

// Rows statically split across threads, one n/2 scratch per thread
// (transforms.hpp:126-137 accepts caller scratch; SPEC.md:233 allows
// concurrent calls on disjoint buffers).
template <class T>
int batch(T* x, size_t rows, size_t n, int mode, int threads) {
  return guarded([&] {
    if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
    if (threads < 1) threads = 1;
    if (static_cast<size_t>(threads) > rows) threads = rows ? static_cast<int>(rows) : 1;
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(threads));
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          std::vector<T> scratch(n / 2 + 1);
          const size_t r0 = rows * static_cast<size_t>(t) / static_cast<size_t>(threads);
          const size_t r1 = rows * static_cast<size_t>(t + 1) / static_cast<size_t>(threads);
          for (size_t r = r0; r < r1; ++r) {
            chw::chw_forward_inplace(std::span<T>(x + r * n, n), to_mode(mode), nullptr,
                                     std::span<T>(scratch));
          }
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(t)] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_chw_forward_f64(double* x, size_t n, int mode, uint64_t* adds, uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::chw_forward_inplace(std::span<double>(x, n), to_mode(mode), &t);
    fill_tally(t, adds, mults);
  });
}
int ref_chw_forward_i64(int64_t* x, size_t n, int mode, uint64_t* adds, uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::chw_forward_inplace(std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n),
                             to_mode(mode), &t);
    fill_tally(t, adds, mults);
  });
}
int ref_haar_forward_f64(double* x, size_t n, int mode, uint64_t* adds, uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::haar_forward_inplace(std::span<double>(x, n), to_mode(mode), &t);
    fill_tally(t, adds, mults);
  });
}
int ref_haar_forward_i64(int64_t* x, size_t n, int mode, uint64_t* adds, uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::haar_forward_inplace(std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n),
                              to_mode(mode), &t);
    fill_tally(t, adds, mults);
  });
}
int ref_haar_inverse_f64(double* x, size_t n, int mode) {
  return guarded([&] { chw::haar_inverse_inplace(std::span<double>(x, n), to_mode(mode)); });
}
int ref_haar_inverse_i64(int64_t* x, size_t n, int mode) {
  return guarded([&] {
    chw::haar_inverse_inplace(std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n),
                              to_mode(mode));
  });
}
int ref_fwht_natural_f64(double* x, size_t n, int mode) {
  return guarded([&] { chw::fwht_natural_inplace(std::span<double>(x, n), to_mode(mode)); });
}
int ref_fwht_natural_i64(int64_t* x, size_t n, int mode) {
  return guarded([&] {
    chw::fwht_natural_inplace(std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n),
                              to_mode(mode));
  });
}
int ref_fwht_dyadic_f64(double* x, size_t n, int mode) {
  return guarded([&] { chw::fwht_dyadic_inplace(std::span<double>(x, n), to_mode(mode)); });
}
int ref_fwht_dyadic_i64(int64_t* x, size_t n, int mode) {
  return guarded([&] {
    chw::fwht_dyadic_inplace(std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n),
                             to_mode(mode));
  });
}
int ref_haar_walsh_forward_f64(double* x, size_t n, int mode) {
  return guarded(
      [&] { chw::haar_walsh_forward_inplace(std::span<double>(x, n), to_mode(mode)); });
}
int ref_haar_walsh_forward_i64(int64_t* x, size_t n, int mode) {
  return guarded([&] {
    chw::haar_walsh_forward_inplace(
        std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n), to_mode(mode));
  });
}
int ref_normalize_f64(double* x, size_t n, int m, uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::normalize_inplace(std::span<double>(x, n), m, &t);
    fill_tally(t, nullptr, mults);
  });
}
int ref_parallel_execute_f64(double* x, size_t n, int workers, int mode, uint64_t* adds,
                             uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::parallel_execute_inplace(std::span<double>(x, n), workers, to_mode(mode), &t);
    fill_tally(t, adds, mults);
  });
}
int ref_parallel_execute_i64(int64_t* x, size_t n, int workers, int mode, uint64_t* adds,
                             uint64_t* mults) {
  return guarded([&] {
    chw::OpTally t;
    chw::parallel_execute_inplace(std::span<std::int64_t>(reinterpret_cast<std::int64_t*>(x), n),
                                  workers, to_mode(mode), &t);
    fill_tally(t, adds, mults);
  });
}
uint64_t ref_bit_reverse(uint64_t v, int bits) { return chw::bit_reverse(v, bits); }
int ref_chw_batch_f64(double* x, size_t rows, size_t n, int mode, int threads) {
  return batch<double>(x, rows, n, mode, threads);
}
int ref_chw_batch_i64(int64_t* x, size_t rows, size_t n, int mode, int threads) {
  return batch<std::int64_t>(reinterpret_cast<std::int64_t*>(x), rows, n, mode, threads);
}
int ref_stage_blocks(int m, int r, uint64_t* offsets, uint64_t* sizes, size_t cap, size_t* count) {
  return guarded([&] {
    const auto b = chw::stage_blocks(m, r);
    *count = b.size();
    for (size_t i = 0; i < b.size() && i < cap; ++i) {
      offsets[i] = b[i].offset;
      sizes[i] = b[i].size;
    }
  });
}
int ref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
