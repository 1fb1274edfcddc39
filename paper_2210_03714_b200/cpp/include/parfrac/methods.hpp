#pragma once
// Method model of the reference (proj/core/include/parfrac/methods.hpp:16-114, series.hpp:12-68,
// bounds.hpp:17-62): exact rational coefficients (Rational, GMP runtime), the moment solve that
// builds a method from any shift set, the published catalog, and the certified theta bound.
// The doubles the kernels see are to_double_nearest of these exact values.

#include <functional>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "parfrac/rational.hpp"

namespace parfrac {

enum class EvalForm { Plain, Residual };

/// Target function (series.hpp:14-36); phi(0) is canonicalised to exp.
struct FunctionId {
  enum class Tag { Exp, Phi, LogOneMinus, Cos, Sin };
  Tag tag = Tag::Exp;
  unsigned phi_order = 0;
  static FunctionId exp() { return {Tag::Exp, 0}; }
  static FunctionId phi(unsigned m) { return m == 0 ? exp() : FunctionId{Tag::Phi, m}; }
  static FunctionId log_one_minus() { return {Tag::LogOneMinus, 0}; }
  static FunctionId cosine() { return {Tag::Cos, 0}; }
  static FunctionId sine() { return {Tag::Sin, 0}; }
  bool operator==(const FunctionId&) const = default;
  /// "exp", "phi1", ..., "log1m", "cos", "sin"
  std::string name() const;
  /// inverse of name(); "phi" means phi1 (BadArgument otherwise)
  static FunctionId parse(std::string_view name);
};

/// Exact Taylor coefficients a_k of a target function (series.hpp:38-57), cached per function.
class CoeffSeries {
 public:
  explicit CoeffSeries(FunctionId fn);
  FunctionId function() const { return fn_; }
  Rational coeff(int k) const;
  std::vector<Rational> prefix(int k_max) const;

 private:
  FunctionId fn_;
};

/// r(x) = d_0 + d_1 x + d_2 x^2 + sum_i b_i / (1 - c_i x)   (methods.hpp:20-48)
struct FractionMethod {
  std::string name;
  FunctionId function = FunctionId::exp();
  std::vector<Rational> shifts;   // c_i, pairwise distinct, at most one zero
  std::vector<Rational> weights;  // b_i
  std::vector<Rational> poly;     // d_0, d_1, d_2 (size 0 or 3)
  int order = 0;
  EvalForm form = EvalForm::Plain;
  std::vector<std::string> notes;
  double theta_u53 = 0.0;  // tabulated theta(2^-53) of the catalog sets (0: compute with theta())

  /// nonzero shifts = linear solves (methods.cpp:67-72)
  int processors() const;
  /// alpha_k = d_k + sum_i b_i c_i^k, 0^0 = 1 (methods.cpp:74-78)
  Rational taylor_coeff(int k) const;
  /// a_0 = d_0 + sum_i b_i, the residual form's constant (methods.cpp:80)
  Rational constant_term() const { return taylor_coeff(0); }
  Rational max_coefficient() const;
  /// max_i |c_i| (0 when every shift is zero)
  Rational max_abs_shift() const;
};

/// Moment system sum_i b_i c_i^k = a_k, k = 0..order, solved exactly (methods.cpp:95-111).
/// LengthMismatch unless shifts.size() == order + 1; DuplicateShift for repeated shifts.
std::vector<Rational> solve_weights(std::span<const Rational> shifts, const CoeffSeries& series, int order);

/// Pure fraction method from a shift set (methods.cpp:121-131); the sum rules are re-verified.
FractionMethod build_plain(std::span<const Rational> shifts, const CoeffSeries& series, int order, std::string name);

/// Hybrid with a quadratic polynomial part (methods.cpp:133-186): `free_weights` fixes 1-based
/// weights, the others solve the moments k = 3..order, then d_k = a_k - sum b_i c_i^k, k = 0..2.
FractionMethod build_hybrid(std::span<const Rational> shifts, const std::map<int, Rational>& free_weights,
                            const CoeffSeries& series, int order, std::string name);

/// LengthMismatch if d_k + sum b_i c_i^k != a_k for some k <= order (methods.hpp:111).
void verify_sum_rules(const FractionMethod& method, const CoeffSeries& series);

/// Shift patterns parameterised by alpha (methods.hpp:85-94).
struct MethodTemplate {
  std::string name;
  std::function<std::vector<Rational>(const Rational& alpha)> shift_pattern;
};
MethodTemplate frac4_template();  // (0, 1/a, -1/a, 1/(2a), -1/(2a))
MethodTemplate frac8_template();  // (0, +-1/a, +-2/(3a), +-1/(2a), +-2/(5a))

/// Published sets R4, R4_phi1, R5, R8, R10star, R10 (methods.cpp:298-369), cached for the process.
/// Built from the generated exact table and cross-checked against the moment solve.
const FractionMethod& catalog(std::string_view name);
std::vector<std::string> catalog_names();

/// phi1 weights on the R4 / R8 shifts ("R4_phi1set", "R8_phi1set"; derived, not in the reference).
const FractionMethod& derived_set(std::string_view name);

FractionMethod to_residual_form(const FractionMethod& method);
FractionMethod to_plain_form(const FractionMethod& method);

/// cos/sin pair set of a method with shifts symmetric about 0 (conjugate shifts +-ic merged).
struct PairMethod {
  std::string name;
  std::vector<Rational> c2, cw, sw;
  Rational a0, a1;
};
const PairMethod& pair_method(std::string_view base);

// ---- certified forward bound and theta (bounds.hpp:17-62)

struct ThetaResult {
  double theta = 0;
  bool saturated = false;  // the bound stays below tol on the whole domain
};

/// Certified upper bound on |f(x) - r(x)| for 0 <= x below the convergence domain
/// (bounds.cpp:97-167: exact per-term coefficients, 256-bit summation, geometric tail majorants,
/// outward rounding). OutOfConvergenceRadius outside the domain.
double forward_bound(const FractionMethod& method, const CoeffSeries& series, double x);

/// Largest x with forward_bound(x) <= tol, bisected to 1e-6 relative width (bounds.cpp:175-201, 252).
ThetaResult theta(const FractionMethod& method, const CoeffSeries& series, double tol);

/// theta of the degree-m Taylor polynomial of exp (bounds.cpp:256-258).
double theta_taylor(int degree, double tol);

/// theta at u = 2^-53: the tabulated value of a catalog / derived set, else theta(method, its
/// function's series, 2^-53) computed once per method name and cached.
double theta_u53(const FractionMethod& method);

}  // namespace parfrac
