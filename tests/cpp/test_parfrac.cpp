// C++ parity tests of the drop-in host layer (namespace parfrac) on the B200, written like the
// reference's own suites (proj/tests/test_dense.cpp, test_methods.cpp) so a maintainer can read them
// side by side. Built by __graft_entry__.build(); run by tests/test_cpp_host.py (-m gpu).
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "parfrac/action.hpp"
#include "parfrac/dense.hpp"
#include "parfrac/error.hpp"
#include "parfrac/methods.hpp"
#include "parfrac/rng.hpp"

using namespace parfrac;

static int g_fail = 0, g_checks = 0;
static bool g_host_only = false;  // --host-only: the method layer only (no GPU needed)
#define CHECK(cond)                                                         \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(cond)) {                                                          \
      ++g_fail;                                                             \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
    }                                                                       \
  } while (0)
#define CHECK_THROWS(expr)                                                  \
  do {                                                                      \
    ++g_checks;                                                             \
    bool thrown_ = false;                                                   \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const Error&) {                                                \
      thrown_ = true;                                                       \
    }                                                                       \
    if (!thrown_) {                                                         \
      ++g_fail;                                                             \
      std::printf("FAIL %s:%d: no throw: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                       \
  } while (0)

namespace {

DenseMatrix random_matrix(int d, std::uint64_t seed) {  // make_dense_matrix randn (cli.cpp:40-45)
  DenseMatrix m(d);
  NormalSampler normal(seed);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) m.at(i, j) = normal.next();
  return m;
}

DenseMatrix scaled_to_one_norm(DenseMatrix m, double target) {
  m.scale(target / m.one_norm());
  return m;
}

double rel_diff_1norm(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix diff = a;
  diff.axpy(-1.0, b);
  return diff.one_norm() / std::max(b.one_norm(), 1e-300);
}

// CPU reference of the residual evaluator in the reference's operation order (the oracle's
// algorithm, small sizes only), used as the parity referee inside this binary.
DenseMatrix host_eval(const FractionMethod& m, const DenseMatrix& b, EvalForm form) {
  const int d = b.dim();
  DenseMatrix acc(d);
  for (size_t i = 0; i < m.shifts.size(); ++i) {
    const double c = to_double_nearest(m.shifts[i]), w = to_double_nearest(m.weights[i]);
    if (c == 0.0) {
      if (form == EvalForm::Plain) acc.add_scaled_identity(w);
      continue;
    }
    DenseMatrix mm = b;
    mm.scale(-c);
    mm.add_scaled_identity(1.0);
    // Gauss-Jordan with partial pivoting on [M | RHS] (small sizes)
    DenseMatrix rhs(d);
    if (form == EvalForm::Plain)
      rhs = DenseMatrix::identity(d);
    else {
      rhs = b;
      rhs.scale(c);
    }
    for (int col = 0; col < d; ++col) {
      int p = col;
      for (int r = col + 1; r < d; ++r)
        if (std::abs(mm.at(r, col)) > std::abs(mm.at(p, col))) p = r;
      for (int j = 0; j < d; ++j) {
        std::swap(mm.at(p, j), mm.at(col, j));
        std::swap(rhs.at(p, j), rhs.at(col, j));
      }
      for (int r = 0; r < d; ++r) {
        if (r == col) continue;
        const double f = mm.at(r, col) / mm.at(col, col);
        for (int j = 0; j < d; ++j) {
          mm.at(r, j) -= f * mm.at(col, j);
          rhs.at(r, j) -= f * rhs.at(col, j);
        }
      }
    }
    for (int r = 0; r < d; ++r)
      for (int j = 0; j < d; ++j) rhs.at(r, j) = rhs.at(r, j) / mm.at(r, r) * w;
    acc.axpy(1.0, rhs);
  }
  if (form == EvalForm::Residual) acc.add_scaled_identity(to_double_nearest(m.constant_term()));
  return acc;
}

void test_lu_solve_and_singular() {  // test_dense.cpp:34-53
  DenseMatrix a(3);
  a.at(0, 0) = 2;
  a.at(0, 1) = 1;
  a.at(1, 1) = 3;
  a.at(1, 2) = -1;
  a.at(2, 0) = 1;
  a.at(2, 2) = 4;
  DenseLu lu(a);
  std::vector<double> x = lu.solve(std::vector<double>{3, 2, 5});
  std::vector<double> r = a.matvec(x);
  CHECK(std::abs(r[0] - 3) <= 1e-14 * 3);
  CHECK(std::abs(r[1] - 2) <= 1e-14 * 2);
  CHECK(std::abs(r[2] - 5) <= 1e-14 * 5);
  DenseMatrix singular(2);
  singular.at(0, 0) = 1;
  singular.at(1, 0) = 1;
  CHECK_THROWS(DenseLu{singular});
}

void test_solve_shifted() {  // test_dense.cpp:55-83
  DenseMatrix zero(4);
  CHECK(rel_diff_1norm(solve_shifted(zero, 0.3), DenseMatrix::identity(4)) == 0.0);
  DenseMatrix diag(3);
  diag.at(0, 0) = 1.0;
  diag.at(1, 1) = -2.0;
  diag.at(2, 2) = 0.5;
  DenseMatrix di = solve_shifted(diag, 0.25);
  for (int i = 0; i < 3; ++i) {
    const double expect = 1.0 / (1.0 - 0.25 * diag.at(i, i));
    CHECK(std::abs(di.at(i, i) - expect) <= 1e-15 * std::abs(expect));
  }
  DenseMatrix b = random_matrix(8, 3);
  const double c = 1.0 / 5.0;
  DenseMatrix x = solve_shifted(b, c);
  DenseMatrix shifted = b;
  shifted.scale(-c);
  shifted.add_scaled_identity(1.0);
  DenseMatrix residual = shifted.mul(x);
  residual.add_scaled_identity(-1.0);
  CHECK(residual.one_norm() <= 1e-13 * x.one_norm());
  CHECK_THROWS(solve_shifted(DenseMatrix::identity(5), 1.0));
}

void test_eval_dense_trivial_and_diagonal() {  // test_dense.cpp:85-106
  const FractionMethod& r4 = catalog("R4");
  const FractionMethod& r10 = catalog("R10");
  DenseMatrix zero(5);
  DenseMatrix expect = DenseMatrix::identity(5);
  CHECK(rel_diff_1norm(eval_dense(r4, zero), expect) <= 1e-12);
  CHECK(rel_diff_1norm(eval_dense(r10, zero), expect) <= 1e-9);
  DenseMatrix diag(3);
  for (int i = 0; i < 3; ++i) diag.at(i, i) = 0.1;
  DenseMatrix v = eval_dense(r4, diag);
  double scalar = 0;
  for (size_t i = 0; i < r4.shifts.size(); ++i)
    scalar += to_double_nearest(r4.weights[i]) * (1.0 / (1 - to_double_nearest(r4.shifts[i]) * 0.1));
  for (int i = 0; i < 3; ++i) CHECK(std::abs(v.at(i, i) - scalar) <= 10 * std::abs(scalar) * 2.23e-16);
}

void test_workers_bit_identical() {  // test_dense.cpp:108-119
  const FractionMethod& r8 = catalog("R8");
  DenseMatrix b = scaled_to_one_norm(random_matrix(24, 5), 0.7);
  DenseMatrix w1 = eval_dense(r8, b, {.workers = 1});
  DenseMatrix w2 = eval_dense(r8, b, {.workers = 2});
  DenseMatrix w8 = eval_dense(r8, b, {.workers = 8});
  bool same = true;
  for (int i = 0; i < b.dim(); ++i)
    for (int j = 0; j < b.dim(); ++j) same = same && w1.at(i, j) == w2.at(i, j) && w1.at(i, j) == w8.at(i, j);
  CHECK(same);
  CHECK_THROWS(eval_dense(r8, b, {.workers = 0}));
  CHECK_THROWS(eval_dense(r8, b, {.fixed_order = false}));
}

void test_plain_and_residual_and_message() {  // test_dense.cpp:121-140
  const FractionMethod& r10 = catalog("R10");
  DenseMatrix b = scaled_to_one_norm(random_matrix(24, 7), 1.0);
  DenseMatrix plain = eval_dense(r10, b, {.form = EvalForm::Plain});
  DenseMatrix residual = eval_dense(r10, b, {.form = EvalForm::Residual});
  CHECK(rel_diff_1norm(plain, residual) <= 1e-8);
  DenseMatrix bad = DenseMatrix::identity(4);
  bad.scale(8.0);
  bool ok = false;
  try {
    eval_dense(r10, bad);
  } catch (const Error& e) {
    ok = e.code() == Errc::SingularShift && std::string(e.what()).find("shift") != std::string::npos &&
         std::string(e.what()).find("singular system: pivot magnitude") != std::string::npos && e.is_numerical();
  }
  CHECK(ok);
}

void test_residual_parity_vs_host_reference() {
  for (const char* name : {"R4", "R8"}) {
    const FractionMethod& m = catalog(name);
    DenseMatrix b = scaled_to_one_norm(random_matrix(40, 9), 0.09);
    DenseMatrix got = eval_dense(m, b, {.form = EvalForm::Residual});
    DenseMatrix ref = host_eval(m, b, EvalForm::Residual);
    CHECK(rel_diff_1norm(got, ref) <= 1e-12);
  }
}

void test_expm_and_friends() {
  DenseMatrix a = scaled_to_one_norm(random_matrix(64, 1), 2.0);  // cfg1
  int j = -1;
  DenseMatrix e4 = expm(catalog("R4"), a, EvalForm::Residual, &j);
  CHECK(j == 10);
  DenseMatrix e8 = expm(catalog("R8"), a);
  CHECK(rel_diff_1norm(e4, e8) <= 1e-12);
  DenseMatrix minus = a;
  minus.scale(-1.0);
  DenseMatrix prod = e8.mul(expm(catalog("R8"), minus));
  CHECK(rel_diff_1norm(prod, DenseMatrix::identity(64)) <= 1e-12);
  auto [ex, phi] = expm_phi1(catalog("R8"), a);
  DenseMatrix lhs = phi.mul(a);
  DenseMatrix rhs = ex;
  rhs.add_scaled_identity(-1.0);
  CHECK(rel_diff_1norm(lhs, rhs) <= 1e-11);
  DenseMatrix sym = a;
  for (int i = 0; i < 64; ++i)
    for (int k = 0; k < 64; ++k) sym.at(i, k) = 0.5 * (a.at(i, k) + a.at(k, i));
  auto [c, s] = cossin(catalog("R8"), sym);
  DenseMatrix py = c.mul(c);
  py.axpy(1.0, s.mul(s));
  CHECK(rel_diff_1norm(py, DenseMatrix::identity(64)) <= 1e-12);
  std::vector<double> v(64 * 2);
  NormalSampler ns(11);
  for (auto& x : v) x = ns.next();
  std::vector<double> av = substep_action(catalog("R8"), a, v, 2, 0, {.form = EvalForm::Residual});
  // column 0 of exp(A) V against e8 V
  double err = 0, nrm = 0;
  for (int i = 0; i < 64; ++i) {
    double ref = 0;
    for (int k = 0; k < 64; ++k) ref += e8.at(i, k) * v[size_t(k) * 2];
    err += std::abs(av[size_t(i) * 2] - ref);
    nrm += std::abs(ref);
  }
  CHECK(err <= 1e-11 * nrm);
}

void test_catalog() {  // test_methods.cpp:50-110: exact rationals, correctly rounded doubles
  CHECK(to_fraction_string(catalog("R4").weights[3]) == "-515/9");
  CHECK(to_fraction_string(catalog("R8").weights[0]) == "-9979069/32256");
  CHECK(to_fraction_string(catalog("R10star").poly[0]) == "-34244933704346617/14676708556800");
  CHECK(catalog("R4").processors() == 4);
  CHECK(catalog("R4").constant_term() == Rational(1));
  CHECK(to_double_nearest(catalog("R4").shifts[1]) == 0.2);
  CHECK(to_double_nearest(catalog("R8").weights[5]) == -0x1.182875d1dc706p+11);  // SURVEY Appendix A hex
  CHECK_THROWS(catalog("R99"));
  CHECK(&catalog("R4") == &catalog("R4"));
  // rational_from_string / to_double_nearest (test_rational.cpp:30-46)
  CHECK(rational_from_string(" 6/4 ") == Rational(3, 2));
  CHECK(rational_from_string("-2.5") == Rational(-5, 2));
  CHECK_THROWS(rational_from_string("1/0"));
  CHECK_THROWS(rational_from_string("abc"));
  CHECK(to_double_nearest(Rational(1, 3)) == 1.0 / 3.0);
  CHECK(to_double_nearest(Rational(-2, 3)) == -2.0 / 3.0);
}

// ---- f3: methods from any shift set, exactly (methods.cpp:95-186), and theta (bounds.cpp:97-254)
void test_method_construction_and_theta() {
  // the catalog sets rebuilt from their shifts by the moment solve (test_methods.cpp:50-110)
  for (const char* name : {"R4", "R5", "R8", "R4_phi1"}) {
    const FractionMethod& m = catalog(name);
    FractionMethod b = build_plain(m.shifts, CoeffSeries(m.function), m.order, name);
    bool same = b.weights.size() == m.weights.size();
    for (size_t i = 0; same && i < b.weights.size(); ++i) same = b.weights[i] == m.weights[i];
    CHECK(same);
  }
  // R10 / R10star: hybrids from their free weights
  for (const char* name : {"R10", "R10star"}) {
    const FractionMethod& m = catalog(name);
    std::map<int, Rational> free;
    free[9] = m.weights[8];
    free[10] = m.weights[9];
    FractionMethod h = build_hybrid(m.shifts, free, CoeffSeries(FunctionId::exp()), 10, name);
    bool same = true;
    for (size_t i = 0; i < m.weights.size(); ++i) same = same && h.weights[i] == m.weights[i];
    for (size_t k = 0; k < 3; ++k) same = same && h.poly[k] == m.poly[k];
    CHECK(same);
  }
  // phi1 weights on the R8 shifts = the derived table (frac8_template(5))
  FractionMethod phi = build_plain(frac8_template().shift_pattern(Rational(5)), CoeffSeries(FunctionId::phi(1)), 8,
                                   "R8_phi1");
  const FractionMethod& tab = derived_set("R8_phi1set");
  bool same = true;
  for (size_t i = 0; i < tab.weights.size(); ++i) same = same && phi.weights[i] == tab.weights[i];
  CHECK(same);
  CHECK(phi.constant_term() == Rational(1));
  // errors: duplicate shifts, wrong counts
  std::vector<Rational> dup{Rational(0), Rational(1, 5), Rational(1, 5)};
  CHECK_THROWS(build_plain(dup, CoeffSeries(FunctionId::exp()), 2, "dup"));
  CHECK_THROWS(solve_weights(dup, CoeffSeries(FunctionId::exp()), 3));
  // theta KATs (test_bounds.cpp:59-71) and the 2^-53 table
  const double u24 = std::ldexp(1.0, -24), u53 = std::ldexp(1.0, -53);
  CHECK(std::abs(theta_taylor(5, u24) - 0.186) <= 0.002);
  CHECK(std::abs(theta_taylor(10, u24) - 1.073) <= 0.005);
  CHECK(std::abs(theta(catalog("R5"), CoeffSeries(FunctionId::exp()), u24).theta - 0.298) <= 0.002);
  CHECK(std::abs(theta(catalog("R10star"), CoeffSeries(FunctionId::exp()), u24).theta - 1.734) <= 0.005);
  for (const char* name : {"R4", "R8", "R10"}) {
    const double t = theta(catalog(name), CoeffSeries(FunctionId::exp()), u53).theta;
    CHECK(std::abs(t - catalog(name).theta_u53) <= 2e-6 * t);
  }
  const double tp = theta(phi, CoeffSeries(FunctionId::phi(1)), u53).theta;
  CHECK(std::abs(tp - tab.theta_u53) <= 2e-6 * tp);
  // a method built here drives the evaluator like a catalog one (theta computed on demand)
  FractionMethod r4b = build_plain(frac4_template().shift_pattern(Rational(5)), CoeffSeries(FunctionId::exp()), 4, "R4b");
  CHECK(std::abs(theta_u53(r4b) - catalog("R4").theta_u53) <= 2e-6 * catalog("R4").theta_u53);
  if (g_host_only) return;
  DenseMatrix a = scaled_to_one_norm(random_matrix(40, 3), 1.5);
  CHECK(rel_diff_1norm(expm(r4b, a), expm(catalog("R4"), a)) <= 1e-13);
}

// ---- banded action (proj/tests/test_action.cpp:49-188)

double vec_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double n = 0, d = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    n += b[i] * b[i];
  }
  return std::sqrt(d) / std::max(std::sqrt(n), 1e-300);
}

TridiagMatrix random_tridiag(int d, std::uint64_t seed, double dom) {
  TridiagMatrix t = TridiagMatrix::zero(d);
  NormalSampler ns(seed);
  for (auto& x : t.sub) x = ns.next();
  for (auto& x : t.diag) x = ns.next() + dom;
  for (auto& x : t.super) x = ns.next();
  return t;
}

void test_thomas() {  // test_action.cpp:49-92
  const int d = 50;
  TridiagMatrix eye = TridiagMatrix::zero(d);
  std::fill(eye.diag.begin(), eye.diag.end(), 1.0);
  std::vector<double> v(d);
  NormalSampler ns(3);
  for (auto& x : v) x = ns.next();
  CHECK(thomas_solve(eye, v) == v);
  TridiagMatrix t = random_tridiag(d, 5, 4.0);
  std::vector<double> x = thomas_solve(t, v);
  CHECK(vec_rel(x, DenseLu(t.to_dense()).solve(v)) <= 1e-13);
  std::vector<double> back = t.matvec(x);
  CHECK(vec_rel(back, v) <= 1e-12);
  TridiagFactor factor(t);
  for (int s = 0; s < 4; ++s) {
    std::vector<double> r(d);
    NormalSampler rs(100 + s);
    for (auto& e : r) e = rs.next();
    CHECK(factor.solve(r) == thomas_solve(t, r));
  }
  TridiagMatrix z = TridiagMatrix::zero(d);
  std::fill(z.sub.begin(), z.sub.end(), 1.0);
  bool got = false;
  try {
    thomas_solve(z, v);
  } catch (const Error& e) {
    got = e.code() == Errc::ZeroPivot && std::string(e.what()).find("zero pivot at row 0") != std::string::npos;
  }
  CHECK(got);
  CHECK_THROWS(TridiagFactor(z));
}

void test_pentadiag() {  // test_action.cpp:95-121
  const int d = 40;
  PentadiagMatrix p;
  p.d = d;
  NormalSampler ns(9);
  p.sub2.resize(d - 2);
  p.sub1.resize(d - 1);
  p.diag.resize(d);
  p.super1.resize(d - 1);
  p.super2.resize(d - 2);
  for (auto* band : {&p.sub2, &p.sub1, &p.super1, &p.super2})
    for (auto& e : *band) e = ns.next();
  for (auto& e : p.diag) e = ns.next() + 6.0;
  std::vector<double> rhs(d);
  for (auto& e : rhs) e = ns.next();
  CHECK(vec_rel(pentadiag_solve(p, rhs), DenseLu(p.to_dense()).solve(rhs)) <= 1e-12);
  PentadiagMatrix zero;
  zero.d = 2;
  zero.sub1 = {0.0};
  zero.diag = {0.0, 0.0};
  zero.super1 = {0.0};
  CHECK_THROWS(pentadiag_solve(zero, std::vector<double>{1, 1}));
}

void test_action() {  // test_action.cpp:124-188
  const int d = 64;
  TridiagMatrix a = TridiagMatrix::trid121(d);
  for (auto* band : {&a.sub, &a.diag, &a.super})
    for (auto& e : *band) e *= -0.25;
  std::vector<double> v(d);
  NormalSampler ns(21);
  for (auto& x : v) x = ns.next();
  for (const char* name : {"R4", "R8", "R10"}) {
    const FractionMethod& m = catalog(name);
    EvalOptions res{.form = EvalForm::Residual};
    std::vector<double> by_action = action_eval(m, a, v, res);
    std::vector<double> by_dense = substep_action(m, a.to_dense(), v, 1, 1, res);
    CHECK(vec_rel(by_action, by_dense) <= 1e-11);
    ActionOperator op(m, a);
    CHECK(op.apply(v, res) == by_action);  // :171-188 identical results
    std::vector<double> s4 = substep_action(m, a, v, 4, res);
    CHECK(s4 == substep_action_block(m, a, v, 1, 4, res));
  }
  std::vector<double> z = action_eval(catalog("R8"), TridiagMatrix::zero(d), v, {.form = EvalForm::Residual});
  CHECK(z == v);  // :149-157 (a0 = 1)
  CHECK_THROWS(action_eval(catalog("R8"), a, v, {.fixed_order = false}));
  CHECK_THROWS(action_eval(catalog("R8"), a, v, {.workers = 0}));
  // "shift i: zero pivot at row r": 1 - c a_00 = 0 for the second shift of R4
  const double c = to_double_nearest(catalog("R4").shifts[1]);
  TridiagMatrix bad = TridiagMatrix::zero(4);
  bad.diag = {1.0 / c, 1.0, 1.0, 1.0};
  bool got = false;
  try {
    action_eval(catalog("R4"), bad, std::vector<double>(4, 1.0), {.form = EvalForm::Residual});
  } catch (const Error& e) {
    got = e.code() == Errc::ZeroPivot && std::string(e.what()).rfind("shift ", 0) == 0;
  }
  CHECK(got);
}

// ---- multi-GPU through EvalOptions (pf_context_create_multi / pf_eval_multi_gpu). One GPU here:
// {0} is a one-rank NCCL communicator; {0, 0, ...} runs the same partition with peer copies.
// fixed_order => bit-identical for any device count (test_dense.cpp:108-119's contract).
void test_multi_device() {
  DenseMatrix b = scaled_to_one_norm(random_matrix(96, 41), 0.6);
  for (const char* name : {"R4", "R8", "R10"}) {
    const FractionMethod& m = catalog(name);
    EvalOptions one{.form = EvalForm::Residual, .device_ids = {0}};
    DenseMatrix ref = eval_dense(m, b, one);
    for (int g : {2, 3, 8}) {
      EvalOptions opts{.form = EvalForm::Residual, .device_ids = std::vector<int>(size_t(g), 0)};
      CHECK(rel_diff_1norm(eval_dense(m, b, opts), ref) == 0.0);
    }
    CHECK(rel_diff_1norm(ref, eval_dense(m, b, {.form = EvalForm::Residual})) <= 1e-12);
  }
  DenseMatrix a = scaled_to_one_norm(random_matrix(160, 42), 4.0);
  int j1 = -1, j4 = -1;
  DenseMatrix e1 = expm(catalog("R8"), a, EvalOptions{.devices = 1, .device_ids = {0}}, &j1);
  DenseMatrix e4 = expm(catalog("R8"), a, EvalOptions{.device_ids = {0, 0, 0, 0}}, &j4);
  CHECK(j1 == j4 && j1 > 0);
  CHECK(rel_diff_1norm(e1, e4) == 0.0);
  CHECK(rel_diff_1norm(e1, expm(catalog("R8"), a)) <= 1e-12);
  auto [pe, pp] = expm_phi1(catalog("R8"), a, EvalOptions{.device_ids = {0, 0}});
  auto [qe, qp] = expm_phi1(catalog("R8"), a);
  CHECK(rel_diff_1norm(pe, qe) <= 1e-12 && rel_diff_1norm(pp, qp) <= 1e-12);
  // SingularShift keeps the reference message with the global shift index
  bool got = false;
  try {
    DenseMatrix five = DenseMatrix::identity(6);
    five.scale(5.0);
    eval_dense(catalog("R4"), five, {.form = EvalForm::Plain, .device_ids = {0, 0, 0}});
  } catch (const Error& e) {
    got = e.code() == Errc::SingularShift && std::string(e.what()).rfind("shift 2: singular system", 0) == 0;
  }
  CHECK(got);
}

// ---- device-resident factors: DenseLu, TridiagFactor, ActionOperator reuse them across calls
void test_resident_factors() {
  DenseMatrix m = random_matrix(70, 7);
  m.add_scaled_identity(12.0);
  DenseLu lu(m);
  DenseLu copy = lu;  // shares the device factors
  DenseMatrix r1 = scaled_to_one_norm(random_matrix(70, 8), 1.0);
  DenseMatrix x1 = lu.solve_matrix(r1), x2 = copy.solve_matrix(r1);
  CHECK(rel_diff_1norm(x1, x2) == 0.0);
  DenseMatrix back = m.mul(x1);
  CHECK(rel_diff_1norm(back, r1) <= 1e-12);
  std::vector<double> col(70);
  for (int i = 0; i < 70; ++i) col[size_t(i)] = r1.at(i, 3);
  std::vector<double> xc = lu.solve(col);
  for (int i = 0; i < 70; ++i) CHECK(std::abs(xc[size_t(i)] - x1.at(i, 3)) <= 1e-13 * (1.0 + std::abs(x1.at(i, 3))));
  TridiagMatrix t = random_tridiag(300, 9, 4.0);
  TridiagFactor f(t);
  std::vector<double> rhs(300);
  NormalSampler ns(10);
  for (auto& e : rhs) e = ns.next();
  CHECK(f.solve(rhs) == thomas_solve(t, rhs));
  CHECK(f.solve(rhs) == f.solve(rhs));
  TridiagMatrix a = TridiagMatrix::trid121(300);
  for (auto* band : {&a.sub, &a.diag, &a.super})
    for (auto& e : *band) e *= -0.3;
  ActionOperator op(catalog("R8"), a);
  for (EvalForm form : {EvalForm::Residual, EvalForm::Plain}) {  // apply's opts.form may change per call
    EvalOptions o{.form = form};
    CHECK(op.apply(rhs, o) == action_eval(catalog("R8"), a, rhs, o));
  }
  std::vector<double> block(300 * 5);
  for (auto& e : block) e = ns.next();
  std::vector<double> ob = op.apply_block(block, 5, {.form = EvalForm::Residual});
  CHECK(ob == substep_action_block(catalog("R8"), a, block, 5, 1, {.form = EvalForm::Residual}));
}

}  // namespace

int main(int argc, char** argv) {
  g_host_only = argc > 1 && std::string(argv[1]) == "--host-only";
  const std::vector<std::pair<const char*, std::function<void()>>> host_tests = {
      {"catalog", test_catalog},
      {"method construction (f3) and theta", test_method_construction_and_theta},
  };
  const std::vector<std::pair<const char*, std::function<void()>>> all_tests = {
      {"lu solve and singularity detection", test_lu_solve_and_singular},
      {"solve_shifted", test_solve_shifted},
      {"eval_dense on trivial and diagonal inputs", test_eval_dense_trivial_and_diagonal},
      {"eval_dense is bit identical across worker counts", test_workers_bit_identical},
      {"plain and residual forms agree to rounding", test_plain_and_residual_and_message},
      {"residual parity vs host reference", test_residual_parity_vs_host_reference},
      {"expm / phi1 / cos-sin / action", test_expm_and_friends},
      {"catalog", test_catalog},
      {"method construction (f3) and theta", test_method_construction_and_theta},
      {"thomas solve and factor reuse", test_thomas},
      {"pentadiagonal solve", test_pentadiag},
      {"tridiagonal action, operator, substeps", test_action},
      {"multi-device evaluation (EvalOptions::devices / device_ids)", test_multi_device},
      {"device-resident DenseLu / TridiagFactor / ActionOperator", test_resident_factors},
  };
  for (auto& [name, fn] : g_host_only ? host_tests : all_tests) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("FAIL %s: exception %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
