// TEST-ONLY SHIM (oracle infrastructure, not product code).
// The reference's decimal.cpp includes <boost/multiprecision/cpp_int.hpp> for
// max_digits_per_limb only (reference proj/src/decimal.cpp:6,14,38-52); boost
// is not installed here. This is a minimal unsigned big integer with exactly
// the operators that function uses, written for this repo.
#pragma once
#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  cpp_int(unsigned long long v) { set(v); }
  cpp_int(int v) { set((unsigned long long)v); }
  cpp_int(unsigned v) { set(v); }
  cpp_int(unsigned long v) { set(v); }

  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    std::uint64_t c = 0;
    for (std::size_t i = 0; i < a.w_.size() || i < b.w_.size() || c; ++i) {
      std::uint64_t s = c + a.at(i) + b.at(i);
      r.w_.push_back(std::uint32_t(s));
      c = s >> 32;
    }
    r.trim();
    return r;
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {  // requires a >= b
    cpp_int r;
    std::int64_t br = 0;
    for (std::size_t i = 0; i < a.w_.size(); ++i) {
      std::int64_t s = std::int64_t(a.at(i)) - std::int64_t(b.at(i)) - br;
      br = s < 0;
      r.w_.push_back(std::uint32_t(s + (br ? (std::int64_t(1) << 32) : 0)));
    }
    r.trim();
    return r;
  }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    r.w_.assign(a.w_.size() + b.w_.size() + 1, 0);
    for (std::size_t i = 0; i < a.w_.size(); ++i) {
      std::uint64_t c = 0;
      for (std::size_t j = 0; j < b.w_.size() || c; ++j) {
        std::uint64_t cur = r.w_[i + j] + c + std::uint64_t(a.w_[i]) * b.at(j);
        r.w_[i + j] = std::uint32_t(cur);
        c = cur >> 32;
      }
    }
    r.trim();
    return r;
  }
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  friend cpp_int operator*(const cpp_int& a, T b) { return a * cpp_int((unsigned long long)b); }
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  friend cpp_int operator-(const cpp_int& a, T b) { return a - cpp_int((unsigned long long)b); }
  friend cpp_int operator<<(const cpp_int& a, std::size_t s) {
    cpp_int r;
    r.w_.assign(s / 32, 0);
    std::uint64_t c = 0;
    for (std::size_t i = 0; i < a.w_.size(); ++i) {
      std::uint64_t v = (std::uint64_t(a.w_[i]) << (s % 32)) | c;
      r.w_.push_back(std::uint32_t(v));
      c = v >> 32;
    }
    if (c) r.w_.push_back(std::uint32_t(c));
    r.trim();
    return r;
  }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return cmp(a, b) < 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return cmp(a, b) >= 0; }

 private:
  std::vector<std::uint32_t> w_;
  void set(unsigned long long v) {
    w_.clear();
    while (v) {
      w_.push_back(std::uint32_t(v));
      v >>= 32;
    }
  }
  std::uint32_t at(std::size_t i) const { return i < w_.size() ? w_[i] : 0; }
  void trim() {
    while (!w_.empty() && w_.back() == 0) w_.pop_back();
  }
  static int cmp(const cpp_int& a, const cpp_int& b) {
    if (a.w_.size() != b.w_.size()) return a.w_.size() < b.w_.size() ? -1 : 1;
    for (std::size_t i = a.w_.size(); i-- > 0;)
      if (a.w_[i] != b.w_[i]) return a.w_[i] < b.w_[i] ? -1 : 1;
    return 0;
  }
};

}  // namespace multiprecision
}  // namespace boost
