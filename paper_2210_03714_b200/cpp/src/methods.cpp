// Method layer of the C++ host: exact Taylor series, the moment solve (solve_weights / build_plain /
// build_hybrid), the shift templates and the published catalog (proj/core/src/methods.cpp:33-369,
// series.cpp:55-120), in exact rational arithmetic. The catalog rows are generated
// (tools/gen_tables.py, catalog_table.inc): exact fraction text plus the table's rounded double,
// which must equal to_double_nearest of the parsed value; every row is re-verified against the
// sum rules on first use.
#include "parfrac/methods.hpp"

#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>

#include "parfrac/error.hpp"

namespace parfrac {

namespace {

struct Coef {
  const char* text;
  double value;
};

struct CatalogRow {
  const char* name;
  const char* function;
  unsigned phi_order;
  int order;
  std::vector<Coef> shifts, weights, poly;
  Coef constant;
  double theta_u53;
};

struct PairRow {
  const char* name;
  std::vector<Coef> c2, cw, sw;
  Coef a0, a1;
};

#include "catalog_table.inc"

Rational exact(const Coef& c) {
  Rational q = rational_from_string(c.text);
  if (to_double_nearest(q) != c.value) raise(Errc::LengthMismatch, std::string("catalog table: ") + c.text);
  return q;
}

std::mutex g_mu;

FractionMethod from_row(const CatalogRow& r) {
  FractionMethod m;
  m.name = r.name;
  std::string fn = r.function;
  m.function = fn == "phi" ? FunctionId::phi(r.phi_order) : FunctionId::exp();
  for (const auto& c : r.shifts) m.shifts.push_back(exact(c));
  for (const auto& c : r.weights) m.weights.push_back(exact(c));
  for (const auto& c : r.poly) m.poly.push_back(exact(c));
  m.order = r.order;
  m.theta_u53 = r.theta_u53;
  if (m.constant_term() != exact(r.constant)) m.notes.push_back("constant term differs from the table");
  verify_sum_rules(m, CoeffSeries(m.function));
  return m;
}

// k! per function family, extended on demand (series coefficients are 1/(k+m)!)
Rational inv_factorial(int k) {
  static std::mutex mu;
  static std::vector<Rational> facts{Rational(1)};
  std::lock_guard<std::mutex> lock(mu);
  while ((int)facts.size() <= k) facts.push_back(facts.back() * Rational((long)facts.size()));
  return Rational(1) / facts[size_t(k)];
}

void check_distinct(std::span<const Rational> shifts) {
  for (size_t i = 0; i < shifts.size(); ++i)
    for (size_t j = i + 1; j < shifts.size(); ++j)
      if (shifts[i] == shifts[j])
        raise(Errc::DuplicateShift, "duplicate shift c = " + to_fraction_string(shifts[i]) + " at positions " +
                                        std::to_string(i + 1) + " and " + std::to_string(j + 1));
}

// exact Gaussian elimination, largest-magnitude pivot per column
std::vector<Rational> solve_exact(std::vector<std::vector<Rational>> a, std::vector<Rational> b) {
  const size_t n = b.size();
  for (size_t col = 0; col < n; ++col) {
    size_t piv = col;
    for (size_t r = col + 1; r < n; ++r)
      if (abs(a[r][col]) > abs(a[piv][col])) piv = r;
    if (a[piv][col].is_zero()) raise(Errc::DuplicateShift, "singular moment system");
    std::swap(a[piv], a[col]);
    std::swap(b[piv], b[col]);
    for (size_t r = col + 1; r < n; ++r) {
      if (a[r][col].is_zero()) continue;
      const Rational f = a[r][col] / a[col][col];
      for (size_t j = col; j < n; ++j) a[r][j] -= f * a[col][j];
      b[r] -= f * b[col];
    }
  }
  std::vector<Rational> x(n);
  for (size_t i = n; i-- > 0;) {
    Rational acc = b[i];
    for (size_t j = i + 1; j < n; ++j) acc -= a[i][j] * x[j];
    x[i] = acc / a[i][i];
  }
  return x;
}

}  // namespace

std::string format_sig17(double x) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", x);
  return buf;
}

// ---------------------------------------------------------------- FunctionId, CoeffSeries

std::string FunctionId::name() const {
  switch (tag) {
    case Tag::Exp: return "exp";
    case Tag::Phi: return "phi" + std::to_string(phi_order);
    case Tag::LogOneMinus: return "log1m";
    case Tag::Cos: return "cos";
    case Tag::Sin: return "sin";
  }
  return "?";
}

FunctionId FunctionId::parse(std::string_view name) {
  if (name == "exp") return exp();
  if (name == "log1m") return log_one_minus();
  if (name == "cos") return cosine();
  if (name == "sin") return sine();
  if (name == "phi") return phi(1);
  if (name.size() > 3 && name.substr(0, 3) == "phi") {
    unsigned m = 0;
    for (char c : name.substr(3)) {
      if (c < '0' || c > '9') raise(Errc::BadArgument, "unknown function: " + std::string(name));
      m = m * 10 + unsigned(c - '0');
    }
    return phi(m);
  }
  raise(Errc::BadArgument, "unknown function: " + std::string(name));
}

CoeffSeries::CoeffSeries(FunctionId fn) : fn_(fn) {}

Rational CoeffSeries::coeff(int k) const {
  if (k < 0) raise(Errc::BadArgument, "negative series index");
  switch (fn_.tag) {
    case FunctionId::Tag::Exp: return inv_factorial(k);
    case FunctionId::Tag::Phi: return inv_factorial(k + int(fn_.phi_order));
    case FunctionId::Tag::LogOneMinus: return k == 0 ? Rational(0) : Rational(-1, k);
    case FunctionId::Tag::Cos:
      if (k % 2) return Rational(0);
      return (k / 2) % 2 == 0 ? inv_factorial(k) : -inv_factorial(k);
    case FunctionId::Tag::Sin:
      if (k % 2 == 0) return Rational(0);
      return ((k - 1) / 2) % 2 == 0 ? inv_factorial(k) : -inv_factorial(k);
  }
  raise(Errc::BadArgument, "bad function tag");
}

std::vector<Rational> CoeffSeries::prefix(int k_max) const {
  if (k_max < 0) raise(Errc::BadArgument, "k_max must be >= 0");
  std::vector<Rational> out;
  for (int k = 0; k <= k_max; ++k) out.push_back(coeff(k));
  return out;
}

// ---------------------------------------------------------------- FractionMethod

int FractionMethod::processors() const {
  int n = 0;
  for (const auto& c : shifts)
    if (!c.is_zero()) ++n;
  return n;
}

Rational FractionMethod::taylor_coeff(int k) const {
  Rational acc = k < int(poly.size()) ? poly[size_t(k)] : Rational(0);
  for (size_t i = 0; i < shifts.size(); ++i) acc += weights[i] * (k == 0 ? Rational(1) : shifts[i].pow(unsigned(k)));
  return acc;
}

Rational FractionMethod::max_coefficient() const {
  Rational best(0);
  for (const auto& b : weights)
    if (abs(b) > best) best = abs(b);
  for (const auto& d : poly)
    if (abs(d) > best) best = abs(d);
  return best;
}

Rational FractionMethod::max_abs_shift() const {
  Rational best(0);
  for (const auto& c : shifts)
    if (abs(c) > best) best = abs(c);
  return best;
}

// ---------------------------------------------------------------- method construction

std::vector<Rational> solve_weights(std::span<const Rational> shifts, const CoeffSeries& series, int order) {
  if (order < 0) raise(Errc::BadArgument, "order must be >= 0");
  if (int(shifts.size()) != order + 1)
    raise(Errc::LengthMismatch, "need order + 1 = " + std::to_string(order + 1) + " shifts, got " +
                                    std::to_string(shifts.size()));
  check_distinct(shifts);
  const size_t n = shifts.size();
  std::vector<std::vector<Rational>> a(n, std::vector<Rational>(n));
  std::vector<Rational> b(n);
  for (size_t k = 0; k < n; ++k) {
    for (size_t i = 0; i < n; ++i) a[k][i] = k == 0 ? Rational(1) : shifts[i].pow(unsigned(k));
    b[k] = series.coeff(int(k));
  }
  return solve_exact(std::move(a), std::move(b));
}

void verify_sum_rules(const FractionMethod& method, const CoeffSeries& series) {
  for (int k = 0; k <= method.order; ++k)
    if (method.taylor_coeff(k) != series.coeff(k))
      raise(Errc::LengthMismatch, "sum rule violated at k = " + std::to_string(k) + " for method " + method.name);
}

FractionMethod build_plain(std::span<const Rational> shifts, const CoeffSeries& series, int order, std::string name) {
  FractionMethod m;
  m.name = std::move(name);
  m.function = series.function();
  m.shifts.assign(shifts.begin(), shifts.end());
  m.weights = solve_weights(shifts, series, order);
  m.order = order;
  verify_sum_rules(m, series);
  return m;
}

FractionMethod build_hybrid(std::span<const Rational> shifts, const std::map<int, Rational>& free_weights,
                            const CoeffSeries& series, int order, std::string name) {
  check_distinct(shifts);
  for (const auto& c : shifts)
    if (c.is_zero()) raise(Errc::BadArgument, "hybrid methods need nonzero shifts");
  for (const auto& [idx, w] : free_weights)
    if (idx < 1 || idx > int(shifts.size()))
      raise(Errc::UnderDetermined, "free weight index " + std::to_string(idx) + " out of range");
  const int n_con = int(shifts.size()) - int(free_weights.size());
  if (n_con != order - 2)
    raise(Errc::UnderDetermined, "hybrid system needs order - 2 = " + std::to_string(order - 2) +
                                     " constrained weights, got " + std::to_string(n_con));
  std::vector<size_t> con;
  for (size_t i = 0; i < shifts.size(); ++i)
    if (!free_weights.count(int(i) + 1)) con.push_back(i);
  std::vector<std::vector<Rational>> a(con.size(), std::vector<Rational>(con.size()));
  std::vector<Rational> b(con.size());
  for (size_t row = 0; row < con.size(); ++row) {
    const unsigned k = unsigned(3 + row);
    Rational rhs = series.coeff(int(k));
    for (const auto& [idx, w] : free_weights) rhs -= w * shifts[size_t(idx - 1)].pow(k);
    b[row] = rhs;
    for (size_t j = 0; j < con.size(); ++j) a[row][j] = shifts[con[j]].pow(k);
  }
  const std::vector<Rational> solved = solve_exact(std::move(a), std::move(b));
  FractionMethod m;
  m.name = std::move(name);
  m.function = series.function();
  m.shifts.assign(shifts.begin(), shifts.end());
  m.weights.assign(shifts.size(), Rational(0));
  for (const auto& [idx, w] : free_weights) m.weights[size_t(idx - 1)] = w;
  for (size_t j = 0; j < con.size(); ++j) m.weights[con[j]] = solved[j];
  for (int k = 0; k < 3; ++k) {
    Rational acc = series.coeff(k);
    for (size_t i = 0; i < shifts.size(); ++i) acc -= m.weights[i] * (k == 0 ? Rational(1) : shifts[i].pow(unsigned(k)));
    m.poly.push_back(acc);
  }
  m.order = order;
  verify_sum_rules(m, series);
  return m;
}

MethodTemplate frac4_template() {
  return {"frac4", [](const Rational& a) {
            const Rational one(1), two_a = Rational(2) * a;
            return std::vector<Rational>{Rational(0), one / a, -(one / a), one / two_a, -(one / two_a)};
          }};
}

MethodTemplate frac8_template() {
  return {"frac8", [](const Rational& a) {
            std::vector<Rational> s{Rational(0)};
            for (const auto& q : {Rational(1), Rational(2, 3), Rational(1, 2), Rational(2, 5)}) {
              s.push_back(q / a);
              s.push_back(-(q / a));
            }
            return s;
          }};
}

// ---------------------------------------------------------------- catalog

const FractionMethod& catalog(std::string_view name) {
  static std::map<std::string, FractionMethod> cache;
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = cache.find(std::string(name));
  if (it != cache.end()) return it->second;
  for (const auto& r : kCatalogRows) {
    if (name == r.name && std::string(r.name).find("set") == std::string::npos)
      return cache.emplace(std::string(name), from_row(r)).first->second;
  }
  raise(Errc::UnknownMethod, "unknown catalog method: " + std::string(name));
}

const FractionMethod& derived_set(std::string_view name) {
  static std::map<std::string, FractionMethod> cache;
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = cache.find(std::string(name));
  if (it != cache.end()) return it->second;
  for (const auto& r : kCatalogRows)
    if (name == r.name) return cache.emplace(std::string(name), from_row(r)).first->second;
  raise(Errc::UnknownMethod, "unknown derived weight set: " + std::string(name));
}

std::vector<std::string> catalog_names() { return {"R4", "R4_phi1", "R5", "R8", "R10star", "R10"}; }

FractionMethod to_residual_form(const FractionMethod& method) {
  FractionMethod m = method;
  m.form = EvalForm::Residual;
  return m;
}

FractionMethod to_plain_form(const FractionMethod& method) {
  FractionMethod m = method;
  m.form = EvalForm::Plain;
  return m;
}

const PairMethod& pair_method(std::string_view base) {
  static std::map<std::string, PairMethod> cache;
  std::lock_guard<std::mutex> lock(g_mu);
  const std::string key = std::string(base) + "_cossin";
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  for (const auto& r : kPairRows) {
    if (key == r.name) {
      PairMethod pm;
      pm.name = r.name;
      for (const auto& c : r.c2) pm.c2.push_back(exact(c));
      for (const auto& c : r.cw) pm.cw.push_back(exact(c));
      for (const auto& c : r.sw) pm.sw.push_back(exact(c));
      pm.a0 = exact(r.a0);
      pm.a1 = exact(r.a1);
      return cache.emplace(key, pm).first->second;
    }
  }
  raise(Errc::UnknownMethod, "no cos/sin pair set for method " + std::string(base));
}

}  // namespace parfrac
