// Minimal stand-in for <boost/rational.hpp> — TEST INFRASTRUCTURE ONLY.
//
// The reference includes it for `actplan::Rational` (rational.hpp:30). The seqpar sources
// compiled into oracle/_ref use only the inline helpers of rational.hpp:32-49 (numerator(),
// denominator()); this class keeps boost's invariants (reduced, positive denominator).
#pragma once

#include <stdexcept>

namespace boost {

template <class T>
class rational {
 public:
  rational() : n_(0), d_(1) {}
  rational(const T& n) : n_(n), d_(1) {}  // NOLINT
  rational(const T& n, const T& d) : n_(n), d_(d) { normalize(); }
  const T& numerator() const { return n_; }
  const T& denominator() const { return d_; }

  friend rational operator+(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_ + b.n_ * a.d_, a.d_ * b.d_);
  }
  friend rational operator-(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_ - b.n_ * a.d_, a.d_ * b.d_);
  }
  friend rational operator*(const rational& a, const rational& b) {
    return rational(a.n_ * b.n_, a.d_ * b.d_);
  }
  friend rational operator/(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_, a.d_ * b.n_);
  }
  friend bool operator==(const rational& a, const rational& b) {
    return a.n_ == b.n_ && a.d_ == b.d_;
  }
  friend bool operator<(const rational& a, const rational& b) {
    return a.n_ * b.d_ < b.n_ * a.d_;
  }

 private:
  static T gcd(T a, T b) {
    if (a < T(0)) a = -a;
    if (b < T(0)) b = -b;
    while (b != T(0)) { T r = a % b; a = b; b = r; }
    return a;
  }
  void normalize() {
    if (d_ == T(0)) throw std::domain_error("rational shim: zero denominator");
    if (d_ < T(0)) { n_ = -n_; d_ = -d_; }
    T g = gcd(n_, d_);
    if (g != T(0) && g != T(1)) { n_ = n_ / g; d_ = d_ / g; }
  }
  T n_, d_;
};

}  // namespace boost
