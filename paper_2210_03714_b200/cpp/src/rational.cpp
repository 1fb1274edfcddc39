// Exact rationals over the GMP runtime (see gmp_runtime.h), the reference's mpq_class semantics.
#include "parfrac/rational.hpp"

#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "gmp_runtime.h"
#include "parfrac/error.hpp"

namespace parfrac {

static_assert(sizeof(pf_mpq) == 32 && alignof(pf_mpq) <= 8, "mpq_t layout (LP64)");

namespace {
inline pf_mpq* Q(void* p) { return static_cast<pf_mpq*>(p); }
inline const pf_mpq* Q(const void* p) { return static_cast<const pf_mpq*>(p); }

bool all_digits(std::string_view s) {
  if (!s.empty() && (s[0] == '+' || s[0] == '-')) s.remove_prefix(1);
  if (s.empty()) return false;
  for (char c : s)
    if (!std::isdigit(static_cast<unsigned char>(c))) return false;
  return true;
}
}  // namespace

Rational::Rational() { __gmpq_init(Q(q_)); }
Rational::Rational(long value) {
  __gmpq_init(Q(q_));
  __gmpq_set_si(Q(q_), value, 1);
}
Rational::Rational(long num, long den) {
  if (den == 0) raise(Errc::BadArgument, "zero denominator");
  __gmpq_init(Q(q_));
  __gmpq_set_si(Q(q_), den < 0 ? -num : num, (unsigned long)(den < 0 ? -den : den));
  __gmpq_canonicalize(Q(q_));
}
Rational::Rational(const Rational& o) {
  __gmpq_init(Q(q_));
  __gmpq_set(Q(q_), Q(o.q_));
}
Rational::Rational(Rational&& o) noexcept {
  __gmpq_init(Q(q_));
  __gmpq_set(Q(q_), Q(o.q_));
}
Rational& Rational::operator=(const Rational& o) {
  if (this != &o) __gmpq_set(Q(q_), Q(o.q_));
  return *this;
}
Rational& Rational::operator=(Rational&& o) noexcept {
  if (this != &o) __gmpq_set(Q(q_), Q(o.q_));
  return *this;
}
Rational::~Rational() { __gmpq_clear(Q(q_)); }

Rational Rational::from_double(double x) {
  if (!std::isfinite(x)) raise(Errc::BadArgument, "non-finite value has no rational form");
  Rational r;
  __gmpq_set_d(Q(r.q_), x);  // exact
  return r;
}

Rational& Rational::operator+=(const Rational& o) {
  __gmpq_add(Q(q_), Q(q_), Q(o.q_));
  return *this;
}
Rational& Rational::operator-=(const Rational& o) {
  __gmpq_sub(Q(q_), Q(q_), Q(o.q_));
  return *this;
}
Rational& Rational::operator*=(const Rational& o) {
  __gmpq_mul(Q(q_), Q(q_), Q(o.q_));
  return *this;
}
Rational& Rational::operator/=(const Rational& o) {
  if (o.is_zero()) raise(Errc::BadArgument, "division by zero");
  __gmpq_div(Q(q_), Q(q_), Q(o.q_));
  return *this;
}
Rational Rational::operator-() const {
  Rational r;
  __gmpq_neg(Q(r.q_), Q(q_));
  return r;
}
int Rational::compare(const Rational& o) const {
  const int c = __gmpq_cmp(Q(q_), Q(o.q_));
  return c < 0 ? -1 : (c > 0 ? 1 : 0);
}
int Rational::sign() const {
  const int s = Q(q_)->num.size;
  return s < 0 ? -1 : (s > 0 ? 1 : 0);
}
Rational Rational::abs() const {
  Rational r;
  __gmpq_abs(Q(r.q_), Q(q_));
  return r;
}
Rational Rational::pow(unsigned k) const {
  Rational r(1), b(*this);
  while (k) {  // square and multiply: exact
    if (k & 1u) r *= b;
    k >>= 1;
    if (k) b *= b;
  }
  return r;
}

Rational rational_from_string(std::string_view text) {
  std::string s(text);
  while (!s.empty() && std::isspace(static_cast<unsigned char>(s.front()))) s.erase(s.begin());
  while (!s.empty() && std::isspace(static_cast<unsigned char>(s.back()))) s.pop_back();
  if (s.empty()) raise(Errc::BadArgument, "empty rational literal");
  Rational q;
  const auto slash = s.find('/');
  const auto dot = s.find('.');
  if (slash != std::string::npos) {
    const std::string num = s.substr(0, slash), den = s.substr(slash + 1);
    if (!all_digits(num) || !all_digits(den)) raise(Errc::BadArgument, "malformed rational literal: " + s);
    std::string canon = (num[0] == '+' ? num.substr(1) : num) + "/" + (den[0] == '+' ? den.substr(1) : den);
    if (__gmpq_set_str(Q(q.raw()), canon.c_str(), 10) != 0) raise(Errc::BadArgument, "malformed rational literal: " + s);
    if (Q(q.raw())->den.size == 0) raise(Errc::BadArgument, "zero denominator in: " + s);
    __gmpq_canonicalize(Q(q.raw()));
    return q;
  }
  if (dot != std::string::npos) {  // decimal: digits / 10^fraction_length, exactly
    std::string digits = s.substr(0, dot) + s.substr(dot + 1);
    if (!all_digits(digits)) raise(Errc::BadArgument, "malformed decimal literal: " + s);
    std::string den = "1" + std::string(s.size() - dot - 1, '0');
    std::string canon = (digits[0] == '+' ? digits.substr(1) : digits) + "/" + den;
    if (__gmpq_set_str(Q(q.raw()), canon.c_str(), 10) != 0) raise(Errc::BadArgument, "malformed decimal literal: " + s);
    __gmpq_canonicalize(Q(q.raw()));
    return q;
  }
  if (!all_digits(s)) raise(Errc::BadArgument, "malformed rational literal: " + s);
  std::string canon = s[0] == '+' ? s.substr(1) : s;
  if (__gmpq_set_str(Q(q.raw()), canon.c_str(), 10) != 0) raise(Errc::BadArgument, "malformed rational literal: " + s);
  return q;
}

double to_double_nearest(const Rational& q) {
  // mpq_get_d truncates toward zero; the nearest double is that value or its neighbour away from
  // zero, decided by exact comparison of the two errors (a tie goes to the even significand)
  const double t = __gmpq_get_d(Q(q.raw()));
  if (!std::isfinite(t)) return t;
  const double away = std::nextafter(t, q.sign() >= 0 ? std::numeric_limits<double>::infinity()
                                                      : -std::numeric_limits<double>::infinity());
  if (!std::isfinite(away)) return t;
  const Rational et = (q - Rational::from_double(t)).abs();
  const Rational ea = (q - Rational::from_double(away)).abs();
  const int c = ea.compare(et);
  if (c < 0) return away;
  if (c > 0) return t;
  std::uint64_t bt, ba;
  std::memcpy(&bt, &t, 8);
  std::memcpy(&ba, &away, 8);
  return (ba & 1u) == 0 && (bt & 1u) != 0 ? away : t;
}

std::string to_fraction_string(const Rational& q) {
  const pf_mpq* m = Q(q.raw());
  std::vector<char> buf(__gmpz_sizeinbase(&m->num, 10) + __gmpz_sizeinbase(&m->den, 10) + 3);
  __gmpq_get_str(buf.data(), 10, m);
  return std::string(buf.data());
}

}  // namespace parfrac
