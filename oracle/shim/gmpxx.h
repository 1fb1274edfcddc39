// TEST INFRASTRUCTURE ONLY (oracle/_ref build). A minimal stand-in for GMP's C++ layer.
//
// The reference core (/root/reference/proj/core) is written against gmpxx (rational.hpp:3,
// highprec.hpp:3: Integer = mpz_class, Rational = mpq_class, BigFloat = mpf_class). This image
// has libgmp.so.10 but neither gmpxx.h nor libgmpxx, so this header supplies value classes with
// the gmpxx member/operator surface the reference uses, over the C entry points declared in
// ./gmp.h. Semantics that matter for the reference's results:
//   * mpz/mpq arithmetic is exact, exactly as in gmpxx (every operation is one GMP call);
//   * mpq_class(n, d) and mpq_class(const char*) do NOT canonicalise (gmpxx behaviour, relied on
//     by methods.cpp:14 and rational.cpp:40-41, which canonicalise explicitly);
//   * string constructors use base 0 (gmpxx's default for mpz/mpq) and throw
//     std::invalid_argument on malformed text;
//   * mpf_class: gmpxx evaluates a whole expression at the precision of the assignment target;
//     here each binary operation rounds to max(operand precisions) and assignment rounds to the
//     target's precision. Every BigFloat the reference creates carries an explicit precision
//     (bounds.cpp:104-108 uses 256 bits throughout), so intermediate precision is never lower
//     than gmpxx's; only the FP64 path (dense.cpp, action.cpp) is used for parity pinning, and
//     it touches GMP only through to_double_nearest (exact).
#ifndef PF_SHIM_GMPXX_H
#define PF_SHIM_GMPXX_H

#include <cstring>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "gmp.h"

class mpz_class {
 public:
  mpz_t mp;

  mpz_class() { mpz_init(mp); }
  mpz_class(const mpz_class& o) { mpz_init_set(mp, o.mp); }
  mpz_class(mpz_class&& o) noexcept {
    mpz_init(mp);
    mpz_swap(mp, o.mp);
  }
  template <class T, std::enable_if_t<std::is_integral_v<T> && std::is_signed_v<T>, int> = 0>
  mpz_class(T v) {
    mpz_init_set_si(mp, long(v));
  }
  template <class T, std::enable_if_t<std::is_integral_v<T> && !std::is_signed_v<T>, int> = 0>
  mpz_class(T v) {
    mpz_init_set_ui(mp, (unsigned long)(v));
  }
  mpz_class(double d) { mpz_init_set_d(mp, d); }
  explicit mpz_class(const char* s, int base = 0) {
    if (mpz_init_set_str(mp, s, base) != 0) {
      mpz_clear(mp);
      throw std::invalid_argument("mpz_set_str");
    }
  }
  explicit mpz_class(const std::string& s, int base = 0) : mpz_class(s.c_str(), base) {}
  ~mpz_class() { mpz_clear(mp); }

  mpz_class& operator=(const mpz_class& o) {
    if (this != &o) mpz_set(mp, o.mp);
    return *this;
  }
  mpz_class& operator=(mpz_class&& o) noexcept {
    mpz_swap(mp, o.mp);
    return *this;
  }

  mpz_ptr get_mpz_t() { return mp; }
  mpz_srcptr get_mpz_t() const { return mp; }
  long get_si() const { return mpz_get_si(mp); }
  unsigned long get_ui() const { return mpz_get_ui(mp); }
  double get_d() const { return mpz_get_d(mp); }
  bool fits_slong_p() const { return mpz_fits_slong_p(mp) != 0; }
  std::string get_str(int base = 10) const {
    std::vector<char> buf(mpz_sizeinbase(mp, base) + 2);
    mpz_get_str(buf.data(), base, mp);
    return std::string(buf.data());
  }
  void swap(mpz_class& o) { mpz_swap(mp, o.mp); }

  mpz_class& operator+=(const mpz_class& o) { mpz_add(mp, mp, o.mp); return *this; }
  mpz_class& operator-=(const mpz_class& o) { mpz_sub(mp, mp, o.mp); return *this; }
  mpz_class& operator*=(const mpz_class& o) { mpz_mul(mp, mp, o.mp); return *this; }
  mpz_class& operator/=(const mpz_class& o) { mpz_tdiv_q(mp, mp, o.mp); return *this; }
  mpz_class& operator%=(const mpz_class& o) { mpz_tdiv_r(mp, mp, o.mp); return *this; }
  mpz_class operator-() const { mpz_class r; mpz_neg(r.mp, mp); return r; }
  mpz_class operator+() const { return *this; }

  friend mpz_class operator+(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_add(r.mp, a.mp, b.mp); return r; }
  friend mpz_class operator-(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_sub(r.mp, a.mp, b.mp); return r; }
  friend mpz_class operator*(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_mul(r.mp, a.mp, b.mp); return r; }
  friend mpz_class operator/(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_tdiv_q(r.mp, a.mp, b.mp); return r; }
  friend mpz_class operator%(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_tdiv_r(r.mp, a.mp, b.mp); return r; }
  friend bool operator==(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.mp, b.mp) == 0; }
  friend bool operator!=(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.mp, b.mp) != 0; }
  friend bool operator<(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.mp, b.mp) < 0; }
  friend bool operator<=(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.mp, b.mp) <= 0; }
  friend bool operator>(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.mp, b.mp) > 0; }
  friend bool operator>=(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.mp, b.mp) >= 0; }
  friend mpz_class abs(const mpz_class& a) { mpz_class r; mpz_abs(r.mp, a.mp); return r; }
  friend int sgn(const mpz_class& a) { return mpz_sgn(a.mp); }
  friend mpz_class gcd(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_gcd(r.mp, a.mp, b.mp); return r; }
  friend std::ostream& operator<<(std::ostream& os, const mpz_class& a) { return os << a.get_str(); }
};

class mpq_class {
 public:
  mpq_t mp;

  mpq_class() { mpq_init(mp); }
  mpq_class(const mpq_class& o) { mpq_init(mp); mpq_set(mp, o.mp); }
  mpq_class(mpq_class&& o) noexcept { mpq_init(mp); mpq_swap(mp, o.mp); }
  template <class T, std::enable_if_t<std::is_integral_v<T> && std::is_signed_v<T>, int> = 0>
  mpq_class(T v) {
    mpq_init(mp);
    mpq_set_si(mp, long(v), 1);
  }
  template <class T, std::enable_if_t<std::is_integral_v<T> && !std::is_signed_v<T>, int> = 0>
  mpq_class(T v) {
    mpq_init(mp);
    mpq_set_ui(mp, (unsigned long)(v), 1);
  }
  mpq_class(double d) { mpq_init(mp); mpq_set_d(mp, d); }
  mpq_class(const mpz_class& z) { mpq_init(mp); mpq_set_z(mp, z.mp); }
  // gmpxx: numerator/denominator pair, stored as given (no canonicalisation).
  mpq_class(const mpz_class& n, const mpz_class& d) {
    mpq_init(mp);
    mpz_set(mpq_numref(mp), n.mp);
    mpz_set(mpq_denref(mp), d.mp);
  }
  template <class N, class D,
            std::enable_if_t<std::is_integral_v<N> && std::is_integral_v<D>, int> = 0>
  mpq_class(N n, D d) : mpq_class(mpz_class(n), mpz_class(d)) {}
  explicit mpq_class(const char* s, int base = 0) {
    mpq_init(mp);
    if (mpq_set_str(mp, s, base) != 0) {
      mpq_clear(mp);
      throw std::invalid_argument("mpq_set_str");
    }
  }
  explicit mpq_class(const std::string& s, int base = 0) : mpq_class(s.c_str(), base) {}
  ~mpq_class() { mpq_clear(mp); }

  mpq_class& operator=(const mpq_class& o) {
    if (this != &o) mpq_set(mp, o.mp);
    return *this;
  }
  mpq_class& operator=(mpq_class&& o) noexcept {
    mpq_swap(mp, o.mp);
    return *this;
  }

  mpq_ptr get_mpq_t() { return mp; }
  mpq_srcptr get_mpq_t() const { return mp; }
  // gmpxx returns the numerator/denominator in place; mpz_class is layout-identical to mpz_t.
  mpz_class& get_num() { return *reinterpret_cast<mpz_class*>(mpq_numref(mp)); }
  const mpz_class& get_num() const { return *reinterpret_cast<const mpz_class*>(mpq_numref(mp)); }
  mpz_class& get_den() { return *reinterpret_cast<mpz_class*>(mpq_denref(mp)); }
  const mpz_class& get_den() const { return *reinterpret_cast<const mpz_class*>(mpq_denref(mp)); }
  mpz_ptr get_num_mpz_t() { return mpq_numref(mp); }
  mpz_srcptr get_num_mpz_t() const { return mpq_numref(mp); }
  mpz_ptr get_den_mpz_t() { return mpq_denref(mp); }
  mpz_srcptr get_den_mpz_t() const { return mpq_denref(mp); }
  void canonicalize() { mpq_canonicalize(mp); }
  double get_d() const { return mpq_get_d(mp); }
  std::string get_str(int base = 10) const {
    std::vector<char> buf(mpz_sizeinbase(mpq_numref(mp), base) + mpz_sizeinbase(mpq_denref(mp), base) + 3);
    mpq_get_str(buf.data(), base, mp);
    return std::string(buf.data());
  }
  void swap(mpq_class& o) { mpq_swap(mp, o.mp); }

  mpq_class& operator+=(const mpq_class& o) { mpq_add(mp, mp, o.mp); return *this; }
  mpq_class& operator-=(const mpq_class& o) { mpq_sub(mp, mp, o.mp); return *this; }
  mpq_class& operator*=(const mpq_class& o) { mpq_mul(mp, mp, o.mp); return *this; }
  mpq_class& operator/=(const mpq_class& o) { mpq_div(mp, mp, o.mp); return *this; }
  mpq_class operator-() const { mpq_class r; mpq_neg(r.mp, mp); return r; }
  mpq_class operator+() const { return *this; }

  friend mpq_class operator+(const mpq_class& a, const mpq_class& b) { mpq_class r; mpq_add(r.mp, a.mp, b.mp); return r; }
  friend mpq_class operator-(const mpq_class& a, const mpq_class& b) { mpq_class r; mpq_sub(r.mp, a.mp, b.mp); return r; }
  friend mpq_class operator*(const mpq_class& a, const mpq_class& b) { mpq_class r; mpq_mul(r.mp, a.mp, b.mp); return r; }
  friend mpq_class operator/(const mpq_class& a, const mpq_class& b) { mpq_class r; mpq_div(r.mp, a.mp, b.mp); return r; }
  friend bool operator==(const mpq_class& a, const mpq_class& b) { return mpq_equal(a.mp, b.mp) != 0; }
  friend bool operator!=(const mpq_class& a, const mpq_class& b) { return mpq_equal(a.mp, b.mp) == 0; }
  friend bool operator<(const mpq_class& a, const mpq_class& b) { return mpq_cmp(a.mp, b.mp) < 0; }
  friend bool operator<=(const mpq_class& a, const mpq_class& b) { return mpq_cmp(a.mp, b.mp) <= 0; }
  friend bool operator>(const mpq_class& a, const mpq_class& b) { return mpq_cmp(a.mp, b.mp) > 0; }
  friend bool operator>=(const mpq_class& a, const mpq_class& b) { return mpq_cmp(a.mp, b.mp) >= 0; }
  friend mpq_class abs(const mpq_class& a) { mpq_class r; mpq_abs(r.mp, a.mp); return r; }
  friend int sgn(const mpq_class& a) { return mpq_sgn(a.mp); }
  friend std::ostream& operator<<(std::ostream& os, const mpq_class& a) { return os << a.get_str(); }
};

class mpf_class {
 public:
  mpf_t mp;

  mpf_class() { mpf_init2(mp, mpf_get_default_prec()); }
  mpf_class(const mpf_class& o) { mpf_init2(mp, mpf_get_prec(o.mp)); mpf_set(mp, o.mp); }
  mpf_class(mpf_class&& o) noexcept { mpf_init2(mp, mpf_get_prec(o.mp)); mpf_swap(mp, o.mp); }
  mpf_class(const mpf_class& o, mp_bitcnt_t prec) { mpf_init2(mp, prec); mpf_set(mp, o.mp); }
  template <class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
  mpf_class(T v) {
    mpf_init2(mp, mpf_get_default_prec());
    assign(v);
  }
  template <class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
  mpf_class(T v, mp_bitcnt_t prec) {
    mpf_init2(mp, prec);
    assign(v);
  }
  mpf_class(const mpq_class& q, mp_bitcnt_t prec) { mpf_init2(mp, prec); mpf_set_q(mp, q.mp); }
  explicit mpf_class(const mpq_class& q) { mpf_init2(mp, mpf_get_default_prec()); mpf_set_q(mp, q.mp); }
  explicit mpf_class(const mpz_class& z) { mpf_init2(mp, mpf_get_default_prec()); mpf_set_z(mp, z.mp); }
  explicit mpf_class(const char* s, mp_bitcnt_t prec = 0, int base = 10) {
    mpf_init2(mp, prec ? prec : mpf_get_default_prec());
    if (mpf_set_str(mp, s, base) != 0) {
      mpf_clear(mp);
      throw std::invalid_argument("mpf_set_str");
    }
  }
  ~mpf_class() { mpf_clear(mp); }

  // Assignment keeps the target's precision (gmpxx semantics).
  mpf_class& operator=(const mpf_class& o) {
    if (this != &o) mpf_set(mp, o.mp);
    return *this;
  }
  mpf_class& operator=(mpf_class&& o) noexcept {
    if (mpf_get_prec(mp) == mpf_get_prec(o.mp))
      mpf_swap(mp, o.mp);
    else
      mpf_set(mp, o.mp);
    return *this;
  }
  template <class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
  mpf_class& operator=(T v) {
    assign(v);
    return *this;
  }

  mpf_ptr get_mpf_t() { return mp; }
  mpf_srcptr get_mpf_t() const { return mp; }
  mp_bitcnt_t get_prec() const { return mpf_get_prec(mp); }
  void set_prec(mp_bitcnt_t prec) { mpf_set_prec(mp, prec); }
  double get_d() const { return mpf_get_d(mp); }
  long get_si() const { return mpf_get_si(mp); }
  void swap(mpf_class& o) { mpf_swap(mp, o.mp); }

  mpf_class& operator+=(const mpf_class& o) { mpf_add(mp, mp, o.mp); return *this; }
  mpf_class& operator-=(const mpf_class& o) { mpf_sub(mp, mp, o.mp); return *this; }
  mpf_class& operator*=(const mpf_class& o) { mpf_mul(mp, mp, o.mp); return *this; }
  mpf_class& operator/=(const mpf_class& o) { mpf_div(mp, mp, o.mp); return *this; }
  mpf_class operator-() const { mpf_class r(0, get_prec()); mpf_neg(r.mp, mp); return r; }
  mpf_class operator+() const { return *this; }

  static mp_bitcnt_t join(const mpf_class& a, const mpf_class& b) {
    mp_bitcnt_t pa = mpf_get_prec(a.mp), pb = mpf_get_prec(b.mp);
    return pa > pb ? pa : pb;
  }
  friend mpf_class operator+(const mpf_class& a, const mpf_class& b) { mpf_class r(0, join(a, b)); mpf_add(r.mp, a.mp, b.mp); return r; }
  friend mpf_class operator-(const mpf_class& a, const mpf_class& b) { mpf_class r(0, join(a, b)); mpf_sub(r.mp, a.mp, b.mp); return r; }
  friend mpf_class operator*(const mpf_class& a, const mpf_class& b) { mpf_class r(0, join(a, b)); mpf_mul(r.mp, a.mp, b.mp); return r; }
  friend mpf_class operator/(const mpf_class& a, const mpf_class& b) { mpf_class r(0, join(a, b)); mpf_div(r.mp, a.mp, b.mp); return r; }
  friend bool operator==(const mpf_class& a, const mpf_class& b) { return mpf_cmp(a.mp, b.mp) == 0; }
  friend bool operator!=(const mpf_class& a, const mpf_class& b) { return mpf_cmp(a.mp, b.mp) != 0; }
  friend bool operator<(const mpf_class& a, const mpf_class& b) { return mpf_cmp(a.mp, b.mp) < 0; }
  friend bool operator<=(const mpf_class& a, const mpf_class& b) { return mpf_cmp(a.mp, b.mp) <= 0; }
  friend bool operator>(const mpf_class& a, const mpf_class& b) { return mpf_cmp(a.mp, b.mp) > 0; }
  friend bool operator>=(const mpf_class& a, const mpf_class& b) { return mpf_cmp(a.mp, b.mp) >= 0; }
  friend mpf_class abs(const mpf_class& a) { mpf_class r(0, a.get_prec()); mpf_abs(r.mp, a.mp); return r; }
  friend mpf_class sqrt(const mpf_class& a) { mpf_class r(0, a.get_prec()); mpf_sqrt(r.mp, a.mp); return r; }
  friend mpf_class floor(const mpf_class& a) { mpf_class r(0, a.get_prec()); mpf_floor(r.mp, a.mp); return r; }
  friend mpf_class ceil(const mpf_class& a) { mpf_class r(0, a.get_prec()); mpf_ceil(r.mp, a.mp); return r; }
  friend mpf_class trunc(const mpf_class& a) { mpf_class r(0, a.get_prec()); mpf_trunc(r.mp, a.mp); return r; }
  friend int sgn(const mpf_class& a) { return mpf_sgn(a.mp); }

 private:
  template <class T>
  void assign(T v) {
    if constexpr (std::is_floating_point_v<T>)
      mpf_set_d(mp, double(v));
    else if constexpr (std::is_signed_v<T>)
      mpf_set_si(mp, long(v));
    else
      mpf_set_ui(mp, (unsigned long)(v));
  }
};

#endif  // PF_SHIM_GMPXX_H
