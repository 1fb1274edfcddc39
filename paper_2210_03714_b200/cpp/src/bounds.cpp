// Certified forward error bound and theta of the C++ host layer (proj/core/include/parfrac/bounds.hpp:
// 17-62; algorithm of bounds.cpp:97-201): eps(x) = sum_{k>s} |a_k - alpha_k| x^k with the exact
// coefficient differences, summed in 256-bit binary floating point until the terms are negligible,
// plus geometric majorants of the fraction and series tails, rounded outward. theta(tol) is the
// bisection point where eps crosses tol. Profiles are built on demand and their thetas cached.
#include <cmath>
#include <limits>
#include <map>
#include <mutex>
#include <optional>
#include <sstream>

#include "gmp_runtime.h"
#include "parfrac/error.hpp"
#include "parfrac/methods.hpp"

namespace parfrac {

namespace {

constexpr int kBits = 256;        // >= 75 decimal digits
constexpr int kMaxTerms = 1500;   // summed terms; the tail majorant covers the rest
constexpr double kDomainCap = 500.0;

// 256-bit float with value semantics (only what the bound needs)
class Big {
 public:
  Big() { __gmpf_init2(&f_, kBits); }
  explicit Big(double x) : Big() { __gmpf_set_d(&f_, x); }
  explicit Big(const Rational& q) : Big() { __gmpf_set_q(&f_, static_cast<const pf_mpq*>(q.raw())); }
  Big(const Big& o) : Big() { __gmpf_set(&f_, &o.f_); }
  Big& operator=(const Big& o) {
    __gmpf_set(&f_, &o.f_);
    return *this;
  }
  ~Big() { __gmpf_clear(&f_); }
  Big& operator+=(const Big& o) {
    __gmpf_add(&f_, &f_, &o.f_);
    return *this;
  }
  Big& operator*=(const Big& o) {
    __gmpf_mul(&f_, &f_, &o.f_);
    return *this;
  }
  friend Big operator*(const Big& a, const Big& b) {
    Big r;
    __gmpf_mul(&r.f_, &a.f_, &b.f_);
    return r;
  }
  friend Big operator/(const Big& a, const Big& b) {
    Big r;
    __gmpf_div(&r.f_, &a.f_, &b.f_);
    return r;
  }
  friend Big operator+(const Big& a, const Big& b) {
    Big r;
    __gmpf_add(&r.f_, &a.f_, &b.f_);
    return r;
  }
  friend Big operator-(const Big& a, const Big& b) {
    Big r;
    __gmpf_sub(&r.f_, &a.f_, &b.f_);
    return r;
  }
  Big pow(unsigned long k) const {
    Big r;
    __gmpf_pow_ui(&r.f_, &f_, k);
    return r;
  }
  int cmp(const Big& o) const { return __gmpf_cmp(&f_, &o.f_); }
  bool is_zero() const { return f_.size == 0; }
  double to_double_toward_zero() const { return __gmpf_get_d(&f_); }

 private:
  pf_mpf f_;
};

std::optional<Rational> series_radius(FunctionId fn) {
  if (fn.tag == FunctionId::Tag::LogOneMinus) return Rational(1);
  return std::nullopt;
}

// sum_{k>K} |a_k| x^k majorant, exact (series.cpp:142-167's families)
Rational series_tail(FunctionId fn, int K, const Rational& x) {
  if (x.sign() < 0) raise(Errc::BadArgument, "tail bound needs x >= 0");
  if (fn.tag == FunctionId::Tag::LogOneMinus) {
    if (x >= Rational(1)) raise(Errc::OutOfConvergenceRadius, "log(1-x) series needs x < 1");
    return x.pow(unsigned(K + 1)) / Rational(K + 1) / (Rational(1) - x);
  }
  const long m = fn.tag == FunctionId::Tag::Phi ? long(fn.phi_order) : 0;
  const Rational ratio = x / Rational(K + m + 2);
  if (ratio >= Rational(1)) raise(Errc::OutOfConvergenceRadius, "tail bound needs K + 2 > x");
  Rational fact(1);
  for (long i = 2; i <= K + 1 + m; ++i) fact *= Rational(i);
  return x.pow(unsigned(K + 1)) / fact / (Rational(1) - ratio);
}

class Profile {
 public:
  Profile(const FractionMethod* method, FunctionId fn, int first_error_order)
      : method_(method ? std::optional<FractionMethod>(*method) : std::nullopt), fn_(fn), s1_(first_error_order) {}

  double domain_hi() const {
    const auto lim = limit();
    if (!lim) return kDomainCap;
    return std::min(kDomainCap, to_double_nearest(*lim) * (1 - 1e-9));
  }

  double bound(double x) {
    if (x < 0) raise(Errc::BadArgument, "forward bound needs x >= 0");
    if (x == 0) return 0.0;
    const Rational xq = Rational::from_double(x);
    const auto lim = limit();
    if (lim && xq >= *lim) raise(Errc::OutOfConvergenceRadius, "x outside the convergence domain");
    const long m_extra = fn_.tag == FunctionId::Tag::Phi ? long(fn_.phi_order) : 0;
    const Big xf(x), cutoff(1e-40);
    Big sum, xpow(xq.pow(unsigned(s1_)));
    int k = s1_;
    for (; k < s1_ + kMaxTerms; ++k) {
      const Big term = Big(err(k)) * xpow;
      sum += term;
      // stop at a negligible nonzero term once the analytic tail ratio is below 1/2
      if (!term.is_zero() && term.cmp(sum * cutoff) < 0 && k >= s1_ + 4 && Rational(k + m_extra) >= Rational(2) * xq)
        break;
      xpow *= xf;
    }
    const int K = std::min(k, s1_ + kMaxTerms - 1);
    Big tail;
    if (method_) {
      for (size_t i = 0; i < method_->shifts.size(); ++i) {
        if (method_->shifts[i].is_zero()) continue;
        const Big cx(abs(method_->shifts[i]) * xq);
        tail += Big(abs(method_->weights[i])) * cx.pow(unsigned(K + 1)) / (Big(1.0) - cx);
      }
    }
    tail += Big(series_tail(fn_, K, xq));
    sum += tail;
    sum *= Big(1.0) + Big(1e-25);  // outward slack for the summation's roundings
    return std::nextafter(sum.to_double_toward_zero(), std::numeric_limits<double>::infinity());
  }

  ThetaResult theta(double tol) {
    if (!(tol > 0)) raise(Errc::BadArgument, "tolerance must be positive");
    double hi = domain_hi();
    if (bound(hi) <= tol) return {hi, true};
    double lo = 0;
    for (int it = 0; it < 200; ++it) {
      const double mid = lo > 0 ? 0.5 * (lo + hi) : hi / 2;
      if (bound(mid) <= tol)
        lo = mid;
      else
        hi = mid;
      if (lo > 0 && (hi - lo) <= 1e-6 * lo && bound(lo) >= tol * (1 - 1e-4)) break;
    }
    return {lo, false};
  }

 private:
  std::optional<Rational> limit() const {
    std::optional<Rational> lim;
    if (method_) {
      const Rational cmax = method_->max_abs_shift();
      if (cmax.sign() > 0) lim = Rational(1) / cmax;
    }
    if (auto r = series_radius(fn_))
      if (!lim || *r < *lim) lim = *r;
    return lim;
  }

  // |a_k - alpha_k|, exact, cached
  const Rational& err(int k) {
    const CoeffSeries series(fn_);
    while (int(errs_.size()) <= k - s1_) {
      const int kk = s1_ + int(errs_.size());
      const Rational alpha = method_ ? method_->taylor_coeff(kk) : Rational(0);
      errs_.push_back(abs(series.coeff(kk) - alpha));
    }
    return errs_[size_t(k - s1_)];
  }

  std::optional<FractionMethod> method_;
  FunctionId fn_;
  int s1_;
  std::vector<Rational> errs_;
};

std::string method_key(const FractionMethod& m, FunctionId fn) {
  std::ostringstream os;
  os << fn.name() << '|' << m.order;
  for (const auto& c : m.shifts) os << '|' << to_fraction_string(c);
  for (const auto& b : m.weights) os << '|' << to_fraction_string(b);
  for (const auto& d : m.poly) os << '|' << to_fraction_string(d);
  return os.str();
}

std::mutex g_theta_mu;
std::map<std::pair<std::string, double>, ThetaResult> g_thetas;

}  // namespace

double forward_bound(const FractionMethod& method, const CoeffSeries& series, double x) {
  return Profile(&method, series.function(), method.order + 1).bound(x);
}

ThetaResult theta(const FractionMethod& method, const CoeffSeries& series, double tol) {
  const auto key = std::make_pair(method_key(method, series.function()), tol);
  {
    std::lock_guard<std::mutex> lock(g_theta_mu);
    auto it = g_thetas.find(key);
    if (it != g_thetas.end()) return it->second;
  }
  const ThetaResult r = Profile(&method, series.function(), method.order + 1).theta(tol);
  std::lock_guard<std::mutex> lock(g_theta_mu);
  g_thetas.emplace(key, r);
  return r;
}

double theta_taylor(int degree, double tol) {
  if (degree < 1) raise(Errc::BadArgument, "taylor degree must be >= 1");
  return Profile(nullptr, FunctionId::exp(), degree + 1).theta(tol).theta;
}

double theta_u53(const FractionMethod& method) {
  if (method.theta_u53 > 0) return method.theta_u53;
  return theta(method, CoeffSeries(method.function), std::ldexp(1.0, -53)).theta;
}

}  // namespace parfrac
