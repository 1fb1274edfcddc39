#pragma once
// Exact rationals of the host layer (the reference's Rational = mpq_class, rational.hpp:10-16):
// always canonical (lowest terms, positive denominator), value semantics, GMP runtime underneath.
// Every coefficient of the method layer is one of these; the kernels receive to_double_nearest.

#include <string>
#include <string_view>

namespace parfrac {

class Rational {
 public:
  Rational();
  Rational(long value);  // NOLINT: integers convert implicitly, as with mpq_class
  Rational(long num, long den);
  Rational(const Rational& o);
  Rational(Rational&& o) noexcept;
  Rational& operator=(const Rational& o);
  Rational& operator=(Rational&& o) noexcept;
  ~Rational();

  /// Exact binary value of a finite double (rational_from_double, rational.cpp:62-64).
  static Rational from_double(double x);

  Rational& operator+=(const Rational& o);
  Rational& operator-=(const Rational& o);
  Rational& operator*=(const Rational& o);
  Rational& operator/=(const Rational& o);  // BadArgument on division by zero
  Rational operator-() const;

  friend Rational operator+(Rational a, const Rational& b) { return a += b; }
  friend Rational operator-(Rational a, const Rational& b) { return a -= b; }
  friend Rational operator*(Rational a, const Rational& b) { return a *= b; }
  friend Rational operator/(Rational a, const Rational& b) { return a /= b; }
  friend bool operator==(const Rational& a, const Rational& b) { return a.compare(b) == 0; }
  friend bool operator!=(const Rational& a, const Rational& b) { return a.compare(b) != 0; }
  friend bool operator<(const Rational& a, const Rational& b) { return a.compare(b) < 0; }
  friend bool operator<=(const Rational& a, const Rational& b) { return a.compare(b) <= 0; }
  friend bool operator>(const Rational& a, const Rational& b) { return a.compare(b) > 0; }
  friend bool operator>=(const Rational& a, const Rational& b) { return a.compare(b) >= 0; }

  int compare(const Rational& o) const;
  int sign() const;
  bool is_zero() const { return sign() == 0; }
  Rational abs() const;
  Rational pow(unsigned k) const;

  const void* raw() const { return q_; }  // the mpq_t (host layer internals)
  void* raw() { return q_; }

 private:
  alignas(8) unsigned char q_[32];
};

inline Rational abs(const Rational& q) { return q.abs(); }

/// "num/den", "num", or a plain decimal such as "-2.5" (rational_from_string, rational.cpp:26-59);
/// BadArgument on malformed text or a zero denominator.
Rational rational_from_string(std::string_view text);

/// Nearest double, ties to even (rational.cpp:66-88): the double handed to the kernels.
double to_double_nearest(const Rational& q);

/// "num/den", or "num" when the denominator is 1 (rational.cpp:90-93).
std::string to_fraction_string(const Rational& q);

}  // namespace parfrac
