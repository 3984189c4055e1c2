// TEST INFRASTRUCTURE ONLY (oracle build shim).
//
// A small, non-expression-template stand-in for GMP's C++ interface
// (<gmpxx.h>), which the image does not ship.  It provides the value classes
// `mpz_class` / `mpq_class` with the operators the reference sources use
// (`using BigInt = mpz_class; using BigRat = mpq_class;` at
// proj/include/curvetop/numeric.hpp:12-13) on top of the system libgmp.so.10.
// Semantics follow gmpxx: `/` and `%` truncate, `>>` floors, the (num, den)
// constructor does not canonicalise, integral/double constructors are
// implicit.  Because there are no expression templates, a few more
// temporaries are created than with the real header; CPU timings taken with
// this shim say so.
//
// Nothing in the product (paper_1103_4697_b200/) includes this file.
#ifndef CTG_ORACLE_SHIM_GMPXX_H
#define CTG_ORACLE_SHIM_GMPXX_H

#include <gmp.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>

class mpq_class;

class mpz_class {
 public:
  mpz_class() { __gmpz_init(z_); }
  mpz_class(const mpz_class& o) { __gmpz_init_set(z_, o.z_); }
  mpz_class(mpz_class&& o) noexcept {
    __gmpz_init(z_);
    __gmpz_swap(z_, o.z_);
  }
  mpz_class(int v) { __gmpz_init_set_si(z_, v); }
  mpz_class(unsigned int v) { __gmpz_init_set_ui(z_, v); }
  mpz_class(long v) { __gmpz_init_set_si(z_, v); }
  mpz_class(unsigned long v) { __gmpz_init_set_ui(z_, v); }
  mpz_class(long long v) { __gmpz_init_set_si(z_, static_cast<long>(v)); }
  mpz_class(unsigned long long v) { __gmpz_init_set_ui(z_, static_cast<unsigned long>(v)); }
  mpz_class(double v) { __gmpz_init_set_d(z_, v); }
  explicit mpz_class(const char* s, int base = 10) {
    if (__gmpz_init_set_str(z_, s, base) != 0) {
      __gmpz_clear(z_);
      throw std::invalid_argument("mpz_set_str");
    }
  }
  explicit mpz_class(const std::string& s, int base = 10) : mpz_class(s.c_str(), base) {}
  explicit mpz_class(mpz_srcptr z) { __gmpz_init_set(z_, z); }
  explicit mpz_class(const mpq_class& q);
  ~mpz_class() { __gmpz_clear(z_); }

  mpz_class& operator=(const mpz_class& o) {
    if (this != &o) __gmpz_set(z_, o.z_);
    return *this;
  }
  mpz_class& operator=(mpz_class&& o) noexcept {
    __gmpz_swap(z_, o.z_);
    return *this;
  }

  mpz_ptr get_mpz_t() { return z_; }
  mpz_srcptr get_mpz_t() const { return z_; }

  std::string get_str(int base = 10) const {
    char* s = __gmpz_get_str(nullptr, base, z_);
    std::string r(s);
    std::free(s);
    return r;
  }
  double get_d() const { return __gmpz_get_d(z_); }
  long get_si() const { return __gmpz_get_si(z_); }
  unsigned long get_ui() const { return __gmpz_get_ui(z_); }
  bool fits_slong_p() const { return __gmpz_fits_slong_p(z_) != 0; }

  mpz_class& operator+=(const mpz_class& o) { __gmpz_add(z_, z_, o.z_); return *this; }
  mpz_class& operator-=(const mpz_class& o) { __gmpz_sub(z_, z_, o.z_); return *this; }
  mpz_class& operator*=(const mpz_class& o) { __gmpz_mul(z_, z_, o.z_); return *this; }
  mpz_class& operator/=(const mpz_class& o) { __gmpz_tdiv_q(z_, z_, o.z_); return *this; }
  mpz_class& operator%=(const mpz_class& o) { __gmpz_tdiv_r(z_, z_, o.z_); return *this; }
  mpz_class& operator<<=(mp_bitcnt_t k) { __gmpz_mul_2exp(z_, z_, k); return *this; }
  mpz_class& operator>>=(mp_bitcnt_t k) { __gmpz_fdiv_q_2exp(z_, z_, k); return *this; }
  mpz_class& operator++() { __gmpz_add_ui(z_, z_, 1); return *this; }
  mpz_class& operator--() { __gmpz_sub_ui(z_, z_, 1); return *this; }

 private:
  mpz_t z_;
};

inline mpz_class operator+(const mpz_class& a, const mpz_class& b) {
  mpz_class r; __gmpz_add(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator-(const mpz_class& a, const mpz_class& b) {
  mpz_class r; __gmpz_sub(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator*(const mpz_class& a, const mpz_class& b) {
  mpz_class r; __gmpz_mul(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator/(const mpz_class& a, const mpz_class& b) {
  mpz_class r; __gmpz_tdiv_q(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator%(const mpz_class& a, const mpz_class& b) {
  mpz_class r; __gmpz_tdiv_r(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator-(const mpz_class& a) {
  mpz_class r; __gmpz_neg(r.get_mpz_t(), a.get_mpz_t()); return r;
}
inline mpz_class operator+(const mpz_class& a) { return a; }
inline mpz_class operator<<(const mpz_class& a, mp_bitcnt_t k) {
  mpz_class r; __gmpz_mul_2exp(r.get_mpz_t(), a.get_mpz_t(), k); return r;
}
inline mpz_class operator>>(const mpz_class& a, mp_bitcnt_t k) {
  mpz_class r; __gmpz_fdiv_q_2exp(r.get_mpz_t(), a.get_mpz_t(), k); return r;
}
inline int cmp(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.get_mpz_t(), b.get_mpz_t()); }
inline bool operator==(const mpz_class& a, const mpz_class& b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) != 0; }
inline bool operator<(const mpz_class& a, const mpz_class& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpz_class& a, const mpz_class& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) >= 0; }
inline int sgn(const mpz_class& a) { return mpz_sgn(a.get_mpz_t()); }
inline mpz_class abs(const mpz_class& a) {
  mpz_class r; __gmpz_abs(r.get_mpz_t(), a.get_mpz_t()); return r;
}
inline mpz_class gcd(const mpz_class& a, const mpz_class& b) {
  mpz_class r; __gmpz_gcd(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline std::ostream& operator<<(std::ostream& os, const mpz_class& a) { return os << a.get_str(); }

class mpq_class {
 public:
  mpq_class() { __gmpq_init(q_); }
  mpq_class(const mpq_class& o) { __gmpq_init(q_); __gmpq_set(q_, o.q_); }
  mpq_class(mpq_class&& o) noexcept { __gmpq_init(q_); __gmpq_swap(q_, o.q_); }
  mpq_class(const mpz_class& z) { __gmpq_init(q_); __gmpq_set_z(q_, z.get_mpz_t()); }
  mpq_class(int v) { __gmpq_init(q_); __gmpq_set_si(q_, v, 1); }
  mpq_class(unsigned int v) : mpq_class(mpz_class(v)) {}
  mpq_class(long v) { __gmpq_init(q_); __gmpq_set_si(q_, v, 1); }
  mpq_class(unsigned long v) : mpq_class(mpz_class(v)) {}
  mpq_class(long long v) : mpq_class(mpz_class(v)) {}
  mpq_class(unsigned long long v) : mpq_class(mpz_class(v)) {}
  mpq_class(double v) { __gmpq_init(q_); __gmpq_set_d(q_, v); }
  // (num, den) without canonicalisation, as gmpxx.
  mpq_class(const mpz_class& n, const mpz_class& d) {
    __gmpq_init(q_);
    __gmpz_set(mpq_numref(q_), n.get_mpz_t());
    __gmpz_set(mpq_denref(q_), d.get_mpz_t());
  }
  ~mpq_class() { __gmpq_clear(q_); }

  mpq_class& operator=(const mpq_class& o) {
    if (this != &o) __gmpq_set(q_, o.q_);
    return *this;
  }
  mpq_class& operator=(mpq_class&& o) noexcept {
    __gmpq_swap(q_, o.q_);
    return *this;
  }

  mpq_ptr get_mpq_t() { return q_; }
  mpq_srcptr get_mpq_t() const { return q_; }
  const mpz_class& get_num() const { return *reinterpret_cast<const mpz_class*>(mpq_numref(q_)); }
  const mpz_class& get_den() const { return *reinterpret_cast<const mpz_class*>(mpq_denref(q_)); }
  mpz_class& get_num() { return *reinterpret_cast<mpz_class*>(mpq_numref(q_)); }
  mpz_class& get_den() { return *reinterpret_cast<mpz_class*>(mpq_denref(q_)); }
  void canonicalize() { __gmpq_canonicalize(q_); }
  double get_d() const { return __gmpq_get_d(q_); }
  std::string get_str(int base = 10) const {
    char* s = __gmpq_get_str(nullptr, base, q_);
    std::string r(s);
    std::free(s);
    return r;
  }

  mpq_class& operator+=(const mpq_class& o) { __gmpq_add(q_, q_, o.q_); return *this; }
  mpq_class& operator-=(const mpq_class& o) { __gmpq_sub(q_, q_, o.q_); return *this; }
  mpq_class& operator*=(const mpq_class& o) { __gmpq_mul(q_, q_, o.q_); return *this; }
  mpq_class& operator/=(const mpq_class& o) { __gmpq_div(q_, q_, o.q_); return *this; }

 private:
  mpq_t q_;
};

static_assert(sizeof(mpz_class) == sizeof(__mpz_struct), "mpz_class must wrap exactly one mpz_t");

inline mpz_class::mpz_class(const mpq_class& q) {
  __gmpz_init(z_);
  __gmpz_tdiv_q(z_, q.get_num().get_mpz_t(), q.get_den().get_mpz_t());
}

inline mpq_class operator+(const mpq_class& a, const mpq_class& b) {
  mpq_class r; __gmpq_add(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator-(const mpq_class& a, const mpq_class& b) {
  mpq_class r; __gmpq_sub(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator*(const mpq_class& a, const mpq_class& b) {
  mpq_class r; __gmpq_mul(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator/(const mpq_class& a, const mpq_class& b) {
  mpq_class r; __gmpq_div(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator-(const mpq_class& a) {
  mpq_class r; __gmpq_neg(r.get_mpq_t(), a.get_mpq_t()); return r;
}
inline mpq_class operator+(const mpq_class& a) { return a; }
inline int cmp(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(a.get_mpq_t(), b.get_mpq_t()); }
inline bool operator==(const mpq_class& a, const mpq_class& b) {
  return __gmpq_equal(a.get_mpq_t(), b.get_mpq_t()) != 0;
}
inline bool operator!=(const mpq_class& a, const mpq_class& b) { return !(a == b); }
inline bool operator<(const mpq_class& a, const mpq_class& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpq_class& a, const mpq_class& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpq_class& a, const mpq_class& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpq_class& a, const mpq_class& b) { return cmp(a, b) >= 0; }
inline int sgn(const mpq_class& a) { return mpq_sgn(a.get_mpq_t()); }
inline mpq_class abs(const mpq_class& a) {
  mpq_class r; __gmpq_abs(r.get_mpq_t(), a.get_mpq_t()); return r;
}
inline std::ostream& operator<<(std::ostream& os, const mpq_class& a) { return os << a.get_str(); }

#endif  // CTG_ORACLE_SHIM_GMPXX_H
