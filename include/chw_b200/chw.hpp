// chw_b200/chw.hpp — drop-in replacement for the reference's transform API.
//
// Reproduces the declarations of the reference's proj/include headers that sit
// on the CHW hot path, in namespace chw, with the same
// signatures, defaults, validation order, exception types and messages — but
// every transform runs on the B200 through the C ABI (chw_b200.h).  A caller of
// the reference switches by replacing
//     #include "chw/transforms.hpp"  (and parallel.hpp, common.hpp, ...)
// with
//     #include "chw_b200/chw.hpp"
// and linking libchw_b200.so.  Spans may point to host memory (staged through
// the pipelined host path) or device memory (transformed in place on the
// current device); every call is synchronous, as in the reference.
//
// Replaced reference declarations (file:line under /root/reference/proj/include/chw):
//   ScalingMode                      common.hpp:15
//   SampleValue                      common.hpp:19-20
//   is_pow2 / level_of               common.hpp:22-25
//   detail::kInvSqrt2, require_pow2, require_mode   common.hpp:27-48
//   CapacityError ... ResourceError  errors.hpp:8-36
//   OpTally                          op_tally.hpp:12-22
//   bit_reverse, natural_to_dyadic, dyadic_to_sequency, Permutation  orderings.hpp:16-90
//   BlockSlice, stage_blocks         transforms.hpp:20-42
//   haar_forward(_inplace)           transforms.hpp:49-80, 214-218
//   haar_inverse(_inplace)           transforms.hpp:85-120, 220-224
//   haar_walsh_forward(_inplace)     transforms.hpp:190-198, 244-248
//   chw_forward_inplace              transforms.hpp:126-143
//   fwht_natural(_inplace), fwht_dyadic(_inplace)  transforms.hpp:147-185, 232-242
//   normalize_inplace                transforms.hpp:202-210
//   chw_forward                      transforms.hpp:226-230
//   normalized                       transforms.hpp:250-260
//   parallel_execute(_inplace)       parallel.hpp:16-22 (parallel.cpp:84-103)
// Added (the reference has no batched entry point): chw_forward_batched_inplace.
#pragma once

#include <bit>
#include <cmath>
#include <concepts>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../chw_b200.h"

namespace chw {

enum class ScalingMode { Orthonormal, Unnormalized };

template <class T>
concept SampleValue = std::same_as<T, std::int64_t> || std::same_as<T, double>;

constexpr bool is_pow2(std::size_t n) { return std::has_single_bit(n); }
constexpr int level_of(std::size_t n) { return std::bit_width(n) - 1; }

class CapacityError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class StructureError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class FormatError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ResourceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
// CUDA runtime failure (no reference counterpart: the reference has no device).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct OpTally {
  std::uint64_t additions = 0;
  std::uint64_t multiplications = 0;
  void reset() {
    additions = 0;
    multiplications = 0;
  }
  friend bool operator==(const OpTally&, const OpTally&) = default;
};

namespace detail {

inline constexpr double kInvSqrt2 = 0.70710678118654752440;

inline void require_pow2(std::size_t n, const char* what) {
  if (n == 0 || !is_pow2(n)) {
    throw std::invalid_argument(std::string(what) + ": length " + std::to_string(n) +
                                " is not a power of two");
  }
}

template <SampleValue T>
void require_mode(ScalingMode mode, const char* what) {
  if constexpr (std::is_integral_v<T>) {
    if (mode == ScalingMode::Orthonormal) {
      throw std::invalid_argument(std::string(what) +
                                  ": orthonormal mode requires a floating-point signal");
    }
  }
}

template <class T>
constexpr chw_dtype dtype_of() {
  if constexpr (std::is_same_v<T, double>)
    return CHW_F64;
  else if constexpr (std::is_same_v<T, float>)
    return CHW_F32;
  else
    return CHW_I64;
}

inline chw_mode mode_of(ScalingMode m) {
  return m == ScalingMode::Orthonormal ? CHW_ORTHONORMAL : CHW_UNNORMALIZED;
}

// Map a C-ABI status back onto the reference's exception types.
inline void raise(chw_status s) {
  if (s == CHW_OK) return;
  const std::string msg = chw_b200_last_error();
  switch (s) {
    case CHW_ERR_LENGTH:
    case CHW_ERR_MODE:
    case CHW_ERR_ARGUMENT:
    case CHW_ERR_WORKSPACE:
      throw std::invalid_argument(msg);
    case CHW_ERR_RESOURCE:
      throw ResourceError(msg);
    case CHW_ERR_UNSUPPORTED:
      throw CapacityError(msg);
    default:
      throw DeviceError(std::string(chw_b200_status_string(s)) + ": " + msg);
  }
}

inline void tally_chw(OpTally* tally, std::size_t n, ScalingMode mode, std::uint64_t rows) {
  if (!tally || n < 2) return;
  std::uint64_t a = 0, m = 0;
  raise(chw_b200_op_tally(0, n, mode_of(mode), &a, &m));
  tally->additions += a * rows;
  tally->multiplications += m * rows;
}

// rows x n contiguous values at `data` (host or device), in place, synchronous.
template <class T>
void run_rows(T* data, std::size_t rows, std::size_t n, ScalingMode mode, chw_order order = CHW_ORDER_DYADIC) {
  if (rows == 0) return;
  if (chw_b200_is_device_pointer(data)) {
    raise(chw_b200_forward_ordered(data, data, dtype_of<T>(), static_cast<std::int64_t>(rows), n,
                                   mode_of(mode), order, nullptr, 0, nullptr));
    raise(chw_b200_stream_synchronize(nullptr));
  } else {
    raise(chw_b200_forward_host_ordered(data, data, dtype_of<T>(), static_cast<std::int64_t>(rows), n,
                                        mode_of(mode), order));
  }
}

}  // namespace detail

// ---------------------------------------------------------------------------
// orderings.hpp
// ---------------------------------------------------------------------------
struct Permutation {
  std::vector<std::uint32_t> map;
  std::size_t size() const { return map.size(); }
  friend bool operator==(const Permutation&, const Permutation&) = default;
};

constexpr std::size_t bit_reverse(std::size_t v, int bits) {
  std::size_t r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (v & 1u);
    v >>= 1;
  }
  return r;
}

constexpr std::uint64_t gray_encode(std::uint64_t v) { return v ^ (v >> 1); }

inline Permutation natural_to_dyadic(int m) {
  if (m < 0 || m > 31)
    throw std::invalid_argument("natural_to_dyadic: level " + std::to_string(m) + " out of range");
  Permutation p;
  p.map.resize(std::size_t{1} << m);
  for (std::size_t i = 0; i < p.map.size(); ++i) p.map[i] = static_cast<std::uint32_t>(bit_reverse(i, m));
  return p;
}

inline Permutation dyadic_to_sequency(int m) {
  if (m < 0 || m > 31)
    throw std::invalid_argument("dyadic_to_sequency: level " + std::to_string(m) + " out of range");
  Permutation p;
  p.map.resize(std::size_t{1} << m);
  for (std::size_t i = 0; i < p.map.size(); ++i) p.map[i] = static_cast<std::uint32_t>(gray_encode(i));
  return p;
}

// ---------------------------------------------------------------------------
// transforms.hpp
// ---------------------------------------------------------------------------
struct BlockSlice {
  std::size_t offset = 0;
  std::size_t size = 0;
  friend bool operator==(const BlockSlice&, const BlockSlice&) = default;
};

inline std::vector<BlockSlice> stage_blocks(int m, int r) {
  if (r < 1 || r > m - 1) {
    throw std::invalid_argument("stage_blocks: stage " + std::to_string(r) + " out of range for m=" +
                                std::to_string(m));
  }
  const std::size_t size = std::size_t{1} << (m - r);
  std::vector<BlockSlice> out;
  out.reserve(std::size_t{1} << (r - 1));
  for (std::size_t q = 0; q < (std::size_t{1} << (r - 1)); ++q) out.push_back({q * 2 * size + size, size});
  return out;
}

// The dyadic-order WHT of one signal, on the GPU.  `scratch` is accepted for
// signature compatibility; the device manages its own workspace.
template <SampleValue T>
void chw_forward_inplace(std::span<T> x, ScalingMode mode, OpTally* tally = nullptr,
                         std::span<T> scratch = {}) {
  (void)scratch;
  detail::require_pow2(x.size(), "chw_forward");
  detail::require_mode<T>(mode, "chw_forward");
  if (x.size() > 1) detail::run_rows(x.data(), 1, x.size(), mode);
  detail::tally_chw(tally, x.size(), mode, 1);
}

// Batched overload (no reference counterpart): `rows` contiguous rows of `n`.
template <class T>
  requires SampleValue<T> || std::same_as<T, float>
void chw_forward_batched_inplace(std::span<T> rows, std::size_t n, ScalingMode mode,
                                 OpTally* tally = nullptr) {
  detail::require_pow2(n, "chw_forward");
  if constexpr (std::is_integral_v<T>) detail::require_mode<T>(mode, "chw_forward");
  if (rows.size() % n != 0)
    throw std::invalid_argument("chw_forward: buffer of " + std::to_string(rows.size()) +
                                " values is not a whole number of rows of " + std::to_string(n));
  if (n > 1) detail::run_rows(rows.data(), rows.size() / n, n, mode);
  detail::tally_chw(tally, n, mode, rows.size() / n);
}

// transforms.hpp:147-172 — natural (Sylvester) order WHT, on the GPU: the CHW
// network without the final bit reversal; bitwise equal to the reference.
template <SampleValue T>
void fwht_natural_inplace(std::span<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  detail::require_pow2(x.size(), "fwht_natural");
  detail::require_mode<T>(mode, "fwht_natural");
  if (x.size() > 1) detail::run_rows(x.data(), 1, x.size(), mode, CHW_ORDER_NATURAL);
  detail::tally_chw(tally, x.size(), mode, 1);
}

// transforms.hpp:177-185 — natural WHT + bit reversal: the dyadic transform.
template <SampleValue T>
void fwht_dyadic_inplace(std::span<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  detail::require_pow2(x.size(), "fwht_natural");
  detail::require_mode<T>(mode, "fwht_natural");
  if (x.size() > 1) detail::run_rows(x.data(), 1, x.size(), mode, CHW_ORDER_DYADIC);
  detail::tally_chw(tally, x.size(), mode, 1);
}

template <SampleValue T>
std::vector<T> fwht_natural(std::vector<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  fwht_natural_inplace(std::span<T>(x), mode, tally);
  return x;
}

template <SampleValue T>
std::vector<T> fwht_dyadic(std::vector<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  fwht_dyadic_inplace(std::span<T>(x), mode, tally);
  return x;
}

inline void normalize_inplace(std::span<double> x, int m, OpTally* tally = nullptr) {
  if (m < 0 || x.size() != (std::size_t{1} << m)) {
    throw std::invalid_argument("normalize: signal length " + std::to_string(x.size()) +
                                " does not match level " + std::to_string(m));
  }
  if (!x.empty() && chw_b200_is_device_pointer(x.data())) {
    // Device span: one multiply per element on the GPU (bit-identical), synchronous.
    detail::raise(chw_b200_normalize(x.data(), CHW_F64, 1, x.size(), m, nullptr));
    detail::raise(chw_b200_stream_synchronize(nullptr));
  } else {
    const double c = 1.0 / std::sqrt(std::ldexp(1.0, m));
    for (double& v : x) v *= c;
  }
  if (tally) tally->multiplications += x.size();
}

// transforms.hpp:49-80 — the Haar transform Psi_m, on the GPU (bit-exact in f64).
template <SampleValue T>
void haar_forward_inplace(std::span<T> x, ScalingMode mode, OpTally* tally = nullptr, std::span<T> scratch = {}) {
  (void)scratch;
  detail::require_pow2(x.size(), "haar_forward");
  detail::require_mode<T>(mode, "haar_forward");
  if (x.size() > 1) {
    if (chw_b200_is_device_pointer(x.data())) {
      detail::raise(chw_b200_haar_forward(x.data(), x.data(), detail::dtype_of<T>(), 1, x.size(),
                                          detail::mode_of(mode), nullptr, 0, nullptr));
      detail::raise(chw_b200_stream_synchronize(nullptr));
    } else {
      detail::raise(chw_b200_haar_forward_host(x.data(), x.data(), detail::dtype_of<T>(), 1, x.size(),
                                               detail::mode_of(mode)));
    }
  }
  if (tally && x.size() > 1) {
    std::uint64_t a = 0, m = 0;
    detail::raise(chw_b200_op_tally(1, x.size(), detail::mode_of(mode), &a, &m));
    tally->additions += a;
    tally->multiplications += m;
  }
}

// transforms.hpp:85-120 — inverse Haar (int64: StructureError on a signal that
// is not an integer forward-transform output).
template <SampleValue T>
void haar_inverse_inplace(std::span<T> x, ScalingMode mode, std::span<T> scratch = {}) {
  (void)scratch;
  detail::require_pow2(x.size(), "haar_inverse");
  detail::require_mode<T>(mode, "haar_inverse");
  if (x.size() < 2) return;
  chw_status s;
  if (chw_b200_is_device_pointer(x.data())) {
    s = chw_b200_haar_inverse(x.data(), x.data(), detail::dtype_of<T>(), 1, x.size(), detail::mode_of(mode),
                              nullptr, 0, nullptr);
    if (s == CHW_OK) s = chw_b200_stream_synchronize(nullptr);
  } else {
    s = chw_b200_haar_inverse_host(x.data(), x.data(), detail::dtype_of<T>(), 1, x.size(), detail::mode_of(mode));
  }
  if (s == CHW_ERR_STRUCTURE) throw StructureError(chw_b200_last_error());
  detail::raise(s);
}

template <SampleValue T>
std::vector<T> haar_inverse(std::vector<T> y, ScalingMode mode) {
  haar_inverse_inplace(std::span<T>(y), mode);
  return y;
}

// transforms.hpp:190-198 — dyadic WHT of each scale block [2^j, 2^(j+1)).
template <SampleValue T>
void haar_walsh_forward_inplace(std::span<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  detail::require_pow2(x.size(), "haar_walsh_forward");
  detail::require_mode<T>(mode, "haar_walsh_forward");
  if (x.size() >= 4) {
    if (chw_b200_is_device_pointer(x.data())) {
      detail::raise(chw_b200_haar_walsh_forward(x.data(), x.data(), detail::dtype_of<T>(), 1, x.size(),
                                                detail::mode_of(mode), nullptr));
      detail::raise(chw_b200_stream_synchronize(nullptr));
    } else {
      detail::raise(chw_b200_haar_walsh_forward_host(x.data(), x.data(), detail::dtype_of<T>(), 1, x.size(),
                                                     detail::mode_of(mode)));
    }
  }
  for (int j = 1; j <= level_of(x.size()) - 1; ++j) detail::tally_chw(tally, std::size_t{1} << j, mode, 1);
}

template <SampleValue T>
std::vector<T> haar_walsh_forward(std::vector<T> h, ScalingMode mode, OpTally* tally = nullptr) {
  haar_walsh_forward_inplace(std::span<T>(h), mode, tally);
  return h;
}

template <SampleValue T>
std::vector<T> haar_forward(std::vector<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  haar_forward_inplace(std::span<T>(x), mode, tally);
  return x;
}

template <SampleValue T>
std::vector<T> chw_forward(std::vector<T> x, ScalingMode mode, OpTally* tally = nullptr) {
  chw_forward_inplace(std::span<T>(x), mode, tally);
  return x;
}

inline std::vector<double> normalized(std::vector<double> x, int m, OpTally* tally = nullptr) {
  normalize_inplace(std::span<double>(x), m, tally);
  return x;
}

inline std::vector<double> normalized(const std::vector<std::int64_t>& x, int m,
                                      OpTally* tally = nullptr) {
  std::vector<double> out(x.begin(), x.end());
  normalize_inplace(std::span<double>(out), m, tally);
  return out;
}

// ---------------------------------------------------------------------------
// parallel.hpp — the paper's node-per-scale executor.  Same contract: bitwise
// equal to the serial transform for every worker count; workers < 1 throws.
// ---------------------------------------------------------------------------
template <SampleValue T>
void parallel_execute_inplace(std::span<T> x, int workers, ScalingMode mode, OpTally* tally = nullptr) {
  detail::require_pow2(x.size(), "parallel_execute");
  detail::require_mode<T>(mode, "parallel_execute");
  if (workers < 1) {
    throw std::invalid_argument("parallel_execute: workers must be >= 1, got " + std::to_string(workers));
  }
  chw_forward_inplace(x, mode, tally);
}

template <SampleValue T>
std::vector<T> parallel_execute(std::vector<T> x, int workers, ScalingMode mode, OpTally* tally = nullptr) {
  parallel_execute_inplace(std::span<T>(x), workers, mode, tally);
  return x;
}

}  // namespace chw
