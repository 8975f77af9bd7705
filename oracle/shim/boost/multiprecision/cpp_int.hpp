// Minimal stand-in for <boost/multiprecision/cpp_int.hpp> — TEST INFRASTRUCTURE ONLY.
//
// Boost is not installed in this image. The reference's seqpar sources use
// `cpp_int` only as `actplan::BigInt` (rational.hpp:29) for the CommLog ring-element counters
// and the per-layer comm-byte model (collectives.cpp:30-38, 75-87). Those values stay far
// below 2^127, so a checked __int128 is an exact substitute: every operation that would leave
// the __int128 range throws std::overflow_error instead of wrapping.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace boost::multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  template <class I, std::enable_if_t<std::is_integral_v<I>, int> = 0>
  cpp_int(I v) : v_(static_cast<__int128>(v)) {}  // NOLINT: implicit like boost

  template <class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
  explicit operator T() const { return static_cast<T>(v_); }

  std::string str() const {
    if (v_ == 0) return "0";
    unsigned __int128 m = v_ < 0 ? static_cast<unsigned __int128>(-(v_ + 1)) + 1
                                 : static_cast<unsigned __int128>(v_);
    std::string s;
    while (m) { s.insert(s.begin(), static_cast<char>('0' + static_cast<int>(m % 10))); m /= 10; }
    return v_ < 0 ? "-" + s : s;
  }

  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    cpp_int r; if (__builtin_add_overflow(a.v_, b.v_, &r.v_)) overflow(); return r;
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
    cpp_int r; if (__builtin_sub_overflow(a.v_, b.v_, &r.v_)) overflow(); return r;
  }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    cpp_int r; if (__builtin_mul_overflow(a.v_, b.v_, &r.v_)) overflow(); return r;
  }
  // Truncating division and remainder, as boost's cpp_int.
  friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
    if (b.v_ == 0) throw std::overflow_error("cpp_int shim: division by zero");
    cpp_int r; r.v_ = a.v_ / b.v_; return r;
  }
  friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
    if (b.v_ == 0) throw std::overflow_error("cpp_int shim: division by zero");
    cpp_int r; r.v_ = a.v_ % b.v_; return r;
  }
  cpp_int operator-() const { return cpp_int(0) - *this; }
  cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
  cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
  cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
  cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }
  cpp_int& operator++() { return *this += 1; }
  cpp_int& operator--() { return *this -= 1; }

  friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v_ == b.v_; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v_ != b.v_; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v_ < b.v_; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v_ > b.v_; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return a.v_ <= b.v_; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return a.v_ >= b.v_; }

 private:
  [[noreturn]] static void overflow() { throw std::overflow_error("cpp_int shim: __int128 overflow"); }
  __int128 v_ = 0;
};

}  // namespace boost::multiprecision
