// TEST INFRASTRUCTURE (oracle) — never linked into the product path.
//
// Minimal arbitrary-precision integer and dyadic rational, written for two
// uses:
//   1. the oracle's exact predicate fallback (restating the reference's
//      scaled-integer method, /root/reference/proj/src/geometry.cpp:21-146);
//   2. a stand-in for boost::multiprecision::{cpp_int,cpp_rational}
//      (oracle/shim/boost/multiprecision/cpp_int.hpp), so the reference's own
//      geometry.cpp and test support headers compile by path here. Boost is
//      not installed; only the operations those files use are
//      provided: construction from int/long long/double, <<=, + - *, += -=,
//      comparisons, sign().
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace sbdt_bigint {

class BigInt {
 public:
  BigInt() = default;
  BigInt(long long v) { set_ll(v); }
  BigInt(int v) { set_ll(v); }
  BigInt(long v) { set_ll(v); }
  BigInt(unsigned long long v) {
    neg_ = false;
    while (v) {
      mag_.push_back(static_cast<std::uint32_t>(v));
      v >>= 32;
    }
  }

  int sign() const { return mag_.empty() ? 0 : (neg_ ? -1 : 1); }
  bool is_zero() const { return mag_.empty(); }

  BigInt& operator<<=(long long s) {
    if (mag_.empty() || s <= 0) return *this;
    const std::size_t words = static_cast<std::size_t>(s / 32);
    const unsigned bits = static_cast<unsigned>(s % 32);
    std::vector<std::uint32_t> r(mag_.size() + words + 1, 0);
    for (std::size_t i = 0; i < mag_.size(); ++i) {
      const std::uint64_t v = std::uint64_t(mag_[i]) << bits;
      r[i + words] |= static_cast<std::uint32_t>(v);
      r[i + words + 1] |= static_cast<std::uint32_t>(v >> 32);
    }
    mag_ = std::move(r);
    trim();
    return *this;
  }

  friend BigInt operator+(const BigInt& a, const BigInt& b) {
    if (a.neg_ == b.neg_) return make(add_mag(a.mag_, b.mag_), a.neg_);
    const int c = cmp_mag(a.mag_, b.mag_);
    if (c == 0) return BigInt();
    if (c > 0) return make(sub_mag(a.mag_, b.mag_), a.neg_);
    return make(sub_mag(b.mag_, a.mag_), b.neg_);
  }
  friend BigInt operator-(const BigInt& a) {
    BigInt r = a;
    if (!r.mag_.empty()) r.neg_ = !r.neg_;
    return r;
  }
  friend BigInt operator-(const BigInt& a, const BigInt& b) { return a + (-b); }
  friend BigInt operator*(const BigInt& a, const BigInt& b) {
    if (a.mag_.empty() || b.mag_.empty()) return BigInt();
    std::vector<std::uint32_t> r(a.mag_.size() + b.mag_.size(), 0);
    for (std::size_t i = 0; i < a.mag_.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < b.mag_.size(); ++j) {
        const std::uint64_t cur = std::uint64_t(a.mag_[i]) * b.mag_[j] + r[i + j] + carry;
        r[i + j] = static_cast<std::uint32_t>(cur);
        carry = cur >> 32;
      }
      std::size_t k = i + b.mag_.size();
      while (carry) {
        const std::uint64_t cur = std::uint64_t(r[k]) + carry;
        r[k] = static_cast<std::uint32_t>(cur);
        carry = cur >> 32;
        ++k;
      }
    }
    return make(std::move(r), a.neg_ != b.neg_);
  }
  BigInt& operator+=(const BigInt& o) { return *this = *this + o; }
  BigInt& operator-=(const BigInt& o) { return *this = *this - o; }
  BigInt& operator*=(const BigInt& o) { return *this = *this * o; }

  friend int compare(const BigInt& a, const BigInt& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    const int c = cmp_mag(a.mag_, b.mag_);
    return a.neg_ ? -c : c;
  }
  friend bool operator==(const BigInt& a, const BigInt& b) { return compare(a, b) == 0; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return compare(a, b) != 0; }
  friend bool operator<(const BigInt& a, const BigInt& b) { return compare(a, b) < 0; }
  friend bool operator>(const BigInt& a, const BigInt& b) { return compare(a, b) > 0; }
  friend bool operator<=(const BigInt& a, const BigInt& b) { return compare(a, b) <= 0; }
  friend bool operator>=(const BigInt& a, const BigInt& b) { return compare(a, b) >= 0; }

 private:
  void set_ll(long long v) {
    mag_.clear();
    neg_ = v < 0;
    unsigned long long u = neg_ ? (~static_cast<unsigned long long>(v) + 1ULL) : static_cast<unsigned long long>(v);
    while (u) {
      mag_.push_back(static_cast<std::uint32_t>(u));
      u >>= 32;
    }
  }
  void trim() {
    while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
    if (mag_.empty()) neg_ = false;
  }
  static BigInt make(std::vector<std::uint32_t> m, bool neg) {
    BigInt r;
    r.mag_ = std::move(m);
    r.neg_ = neg;
    r.trim();
    return r;
  }
  static int cmp_mag(const std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static std::vector<std::uint32_t> add_mag(const std::vector<std::uint32_t>& a,
                                            const std::vector<std::uint32_t>& b) {
    const auto& x = a.size() >= b.size() ? a : b;
    const auto& y = a.size() >= b.size() ? b : a;
    std::vector<std::uint32_t> r(x.size() + 1, 0);
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < x.size(); ++i) {
      const std::uint64_t cur = std::uint64_t(x[i]) + (i < y.size() ? y[i] : 0) + carry;
      r[i] = static_cast<std::uint32_t>(cur);
      carry = cur >> 32;
    }
    r[x.size()] = static_cast<std::uint32_t>(carry);
    return r;
  }
  // |a| >= |b|
  static std::vector<std::uint32_t> sub_mag(const std::vector<std::uint32_t>& a,
                                            const std::vector<std::uint32_t>& b) {
    std::vector<std::uint32_t> r(a.size(), 0);
    std::int64_t borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::int64_t cur = std::int64_t(a[i]) - (i < b.size() ? b[i] : 0) - borrow;
      borrow = cur < 0;
      if (cur < 0) cur += (std::int64_t(1) << 32);
      r[i] = static_cast<std::uint32_t>(cur);
    }
    return r;
  }

  std::vector<std::uint32_t> mag_;
  bool neg_ = false;
};

// Exact dyadic rational m * 2^e (every finite binary64 is one). Closed under
// + - *, which is all the reference's rational test oracle uses
// (/root/reference/proj/tests/support/exact_ref.hpp:18-85).
class Dyadic {
 public:
  Dyadic() = default;
  Dyadic(int v) : m_(v), e_(0) {}
  Dyadic(long long v) : m_(v), e_(0) {}
  Dyadic(double v) {
    if (!std::isfinite(v)) throw std::domain_error("non-finite value in Dyadic");
    if (v == 0.0) return;
    int ex;
    const double fr = std::frexp(v, &ex);  // v = fr * 2^ex, 0.5 <= |fr| < 1
    const long long mant = static_cast<long long>(std::ldexp(fr, 53));
    m_ = BigInt(mant);
    e_ = ex - 53;
  }
  int sign() const { return m_.sign(); }
  friend Dyadic operator*(const Dyadic& a, const Dyadic& b) {
    Dyadic r;
    r.m_ = a.m_ * b.m_;
    r.e_ = a.e_ + b.e_;
    return r;
  }
  friend Dyadic operator+(const Dyadic& a, const Dyadic& b) {
    if (a.m_.is_zero()) return b;
    if (b.m_.is_zero()) return a;
    Dyadic r;
    if (a.e_ <= b.e_) {
      BigInt t = b.m_;
      t <<= (b.e_ - a.e_);
      r.m_ = a.m_ + t;
      r.e_ = a.e_;
    } else {
      BigInt t = a.m_;
      t <<= (a.e_ - b.e_);
      r.m_ = t + b.m_;
      r.e_ = b.e_;
    }
    return r;
  }
  friend Dyadic operator-(const Dyadic& a) {
    Dyadic r = a;
    r.m_ = -r.m_;
    return r;
  }
  friend Dyadic operator-(const Dyadic& a, const Dyadic& b) { return a + (-b); }
  Dyadic& operator+=(const Dyadic& o) { return *this = *this + o; }
  Dyadic& operator-=(const Dyadic& o) { return *this = *this - o; }
  Dyadic& operator*=(const Dyadic& o) { return *this = *this * o; }
  friend bool operator==(const Dyadic& a, const Dyadic& b) { return (a - b).sign() == 0; }
  friend bool operator!=(const Dyadic& a, const Dyadic& b) { return (a - b).sign() != 0; }
  friend bool operator<(const Dyadic& a, const Dyadic& b) { return (a - b).sign() < 0; }
  friend bool operator>(const Dyadic& a, const Dyadic& b) { return (a - b).sign() > 0; }
  friend bool operator<=(const Dyadic& a, const Dyadic& b) { return (a - b).sign() <= 0; }
  friend bool operator>=(const Dyadic& a, const Dyadic& b) { return (a - b).sign() >= 0; }

 private:
  BigInt m_;
  long long e_ = 0;
};

}  // namespace sbdt_bigint
