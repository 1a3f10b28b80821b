// chw_b200/signal_io.hpp — the reference's signal file formats.
//
// Same formats, validation and error types as proj/include/chw/signal_io.hpp
// and proj/src/signal_io.cpp:
//   Text   — one decimal value per line; blank lines and '#' lines skipped;
//            unparsable token -> FormatError "<path>:<line>: cannot parse '<tok>'".
//   Binary — little-endian IEEE-754 doubles, no header; byte size must be a
//            multiple of 8; integers must be exact 64-bit values.
//   The sample count must be a power of two (FormatError otherwise) — or, for
//   the batched readers added here, a multiple of the row length.
// Unreadable/unwritable files -> IoError.
#pragma once

#include <bit>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "chw.hpp"

namespace chw {

enum class SignalFormat { Text, Binary };

namespace io_detail {

inline std::string_view trim(std::string_view s) {
  const auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
  while (!s.empty() && ws(s.front())) s.remove_prefix(1);
  while (!s.empty() && ws(s.back())) s.remove_suffix(1);
  return s;
}

template <class T>
T parse_token(std::string_view tok, const std::filesystem::path& path, std::size_t line) {
  T v{};
  const auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc{} || p != tok.data() + tok.size())
    throw FormatError(path.string() + ":" + std::to_string(line) + ": cannot parse '" + std::string(tok) + "'");
  return v;
}

inline void check_count(std::size_t count, std::size_t row, const std::filesystem::path& path) {
  if (row == 0) {
    if (count == 0 || !is_pow2(count))
      throw FormatError(path.string() + ": sample count " + std::to_string(count) + " is not a power of two");
  } else if (count == 0 || count % row != 0) {
    throw FormatError(path.string() + ": sample count " + std::to_string(count) +
                      " is not a whole number of rows of " + std::to_string(row));
  }
}

template <class T>
T from_double(double v, const std::filesystem::path& path, std::size_t idx) {
  if constexpr (std::is_integral_v<T>) {
    if (!std::isfinite(v) || v != std::floor(v) || v < -9.223372036854775808e18 || v >= 9.223372036854775808e18)
      throw FormatError(path.string() + ": value #" + std::to_string(idx) + " is not an exact 64-bit integer");
    return static_cast<T>(v);
  } else {
    return v;
  }
}

}  // namespace io_detail

// `row` = 0: one signal (power-of-two count); row > 0: a batch of rows of that length.
template <SampleValue T>
std::vector<T> read_signal(const std::filesystem::path& path, SignalFormat format, std::size_t row = 0) {
  std::vector<T> v;
  if (format == SignalFormat::Text) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open '" + path.string() + "' for reading");
    std::string line;
    std::size_t ln = 0;
    while (std::getline(in, line)) {
      ++ln;
      const std::string_view tok = io_detail::trim(line);
      if (tok.empty() || tok.front() == '#') continue;
      v.push_back(io_detail::parse_token<T>(tok, path, ln));
    }
    if (in.bad()) throw IoError("read error on '" + path.string() + "'");
  } else {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path.string() + "' for reading");
    std::vector<unsigned char> b((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) throw IoError("read error on '" + path.string() + "'");
    if (b.size() % 8 != 0)
      throw FormatError(path.string() + ": byte size " + std::to_string(b.size()) + " is not a multiple of 8");
    v.resize(b.size() / 8);
    for (std::size_t i = 0; i < v.size(); ++i) {
      std::uint64_t u = 0;
      for (int k = 7; k >= 0; --k) u = (u << 8) | b[8 * i + k];
      v[i] = io_detail::from_double<T>(std::bit_cast<double>(u), path, i);
    }
  }
  io_detail::check_count(v.size(), row, path);
  return v;
}

template <SampleValue T>
void write_signal(std::span<const T> x, const std::filesystem::path& path, SignalFormat format) {
  if (format == SignalFormat::Text) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot open '" + path.string() + "' for writing");
    char buf[64];
    for (const T& val : x) {
      const auto [p, ec] = std::to_chars(buf, buf + sizeof(buf), val);
      if (ec != std::errc{}) throw IoError("cannot format value for '" + path.string() + "'");
      out.write(buf, p - buf);
      out.put('\n');
    }
    out.flush();
    if (!out) throw IoError("write error on '" + path.string() + "'");
  } else {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path.string() + "' for writing");
    std::vector<unsigned char> b(8 * x.size());
    for (std::size_t i = 0; i < x.size(); ++i) {
      std::uint64_t u = std::bit_cast<std::uint64_t>(static_cast<double>(x[i]));
      for (int k = 0; k < 8; ++k, u >>= 8) b[8 * i + k] = static_cast<unsigned char>(u & 0xffu);
    }
    out.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
    out.flush();
    if (!out) throw IoError("write error on '" + path.string() + "'");
  }
}

}  // namespace chw
