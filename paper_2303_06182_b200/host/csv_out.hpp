// Deterministic CSV output for the drop-in reporting functions (placements,
// comm plans, cache sweeps, load matrices): comma-separated fields, '\n' line
// ends, doubles printed with %.12g -- the reference's format
// (proj/include/moesim/csv.hpp), so files are byte-identical to its output.
#pragma once

#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace moesim::detail {

class CsvOut {
 public:
  explicit CsvOut(const std::filesystem::path& path) : f_(path, std::ios::binary) {
    if (!f_) throw std::runtime_error("cannot write file: " + path.string());
  }

  template <class... Fields>
  void line(const Fields&... fields) {
    bool first = true;
    ((put(fields, first), first = false), ...);
    f_ << '\n';
  }

  static std::string number(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.12g", v);
    return buf;
  }

 private:
  template <class T>
  void put(const T& v, bool first) {
    if (!first) f_ << ',';
    if constexpr (std::is_floating_point_v<T>)
      f_ << number(v);
    else if constexpr (std::is_integral_v<T>)
      f_ << std::to_string(static_cast<long long>(v));
    else
      f_ << v;
  }

  std::ofstream f_;
};

}  // namespace moesim::detail
