// Catalog and method helpers of the C++ host layer (proj/core/src/methods.cpp:298-369 restated
// as generated tables; exact values checked by tests/test_cpp_tables.py).
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

Rational rat(const Coef& c) { return Rational{c.text, c.value}; }

FractionMethod from_row(const CatalogRow& r) {
  FractionMethod m;
  m.name = r.name;
  std::string fn = r.function;
  m.function = fn == "phi" ? FunctionId::phi(r.phi_order) : FunctionId::exp();
  for (const auto& c : r.shifts) m.shifts.push_back(rat(c));
  for (const auto& c : r.weights) m.weights.push_back(rat(c));
  for (const auto& c : r.poly) m.poly.push_back(rat(c));
  m.order = r.order;
  m.constant = rat(r.constant);
  m.theta_u53 = r.theta_u53;
  return m;
}

std::mutex g_mu;

}  // namespace

std::string format_sig17(double x) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", x);
  return buf;
}

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

int FractionMethod::processors() const {
  int n = 0;
  for (const auto& c : shifts)
    if (c.nearest != 0.0) ++n;
  return n;
}

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
      for (const auto& c : r.c2) pm.c2.push_back(rat(c));
      for (const auto& c : r.cw) pm.cw.push_back(rat(c));
      for (const auto& c : r.sw) pm.sw.push_back(rat(c));
      pm.a0 = rat(r.a0);
      pm.a1 = rat(r.a1);
      return cache.emplace(key, pm).first->second;
    }
  }
  raise(Errc::UnknownMethod, "no cos/sin pair set for method " + std::string(base));
}

double theta_u53(const FractionMethod& method) {
  if (method.theta_u53 > 0) return method.theta_u53;
  raise(Errc::BadArgument, "no theta(2^-53) tabulated for method " + method.name);
}

}  // namespace parfrac
