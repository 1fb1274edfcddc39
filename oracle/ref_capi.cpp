// TEST INFRASTRUCTURE ONLY -- C entry points over the REFERENCE ITSELF (oracle/_ref).
//
// oracle/Makefile compiles /root/reference/proj/core/src/*.cpp unmodified (against the GMP/gmpxx
// shims in oracle/shim/) together with this file into oracle/_ref/libparfrac_ref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's CPU legs load it; the product path never does.
//
// Everything below calls the reference's own code: catalog()/build_plain()/to_residual_form()
// (methods.cpp), theta() (bounds.cpp), eval_dense()/DenseLu/solve_shifted()/DenseMatrix::mul
// (dense.cpp), action_eval()/substep_action()/ActionOperator/thomas_solve()/TridiagFactor/
// pentadiag_solve() (action.cpp), make_dense_matrix()/random_unit_vector() (cli.cpp),
// SplitMix64/NormalSampler (rng.hpp, rng.cpp), pade4()/taylor8()/... (dense.cpp). Where SURVEY
// §8(a) defines a composition the reference does not have (a10 scaling and squaring, a12 phi1
// doubling, a13 dense block action), it is written here from those reference primitives only,
// in the order the compositions are specified.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

// DenseLu keeps its factors private (dense.hpp:55-58); the parity tests compare pivots and
// factors, so this translation unit (test infrastructure) reads them through a layout-identical
// mirror instead of modifying the reference.
#include "parfrac/action.hpp"
#include "parfrac/bounds.hpp"
#include "parfrac/cli.hpp"
#include "parfrac/dense.hpp"
#include "parfrac/error.hpp"
#include "parfrac/methods.hpp"
#include "parfrac/rng.hpp"
#include "worker_pool.hpp"

using namespace parfrac;

namespace {

struct DenseLuMirror {  // same members, same order as DenseLu (dense.hpp:55-58)
  int d_;
  std::vector<double> lu_;
  std::vector<int> piv_;
};
static_assert(sizeof(DenseLuMirror) == sizeof(DenseLu));

int fail(const Error& e, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), size_t(errlen) - 1);
    err[errlen - 1] = 0;
  }
  return int(e.code()) + 1;
}

int fail_other(const std::exception& e, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), size_t(errlen) - 1);
    err[errlen - 1] = 0;
  }
  return 1000;
}

#define PFR_TRY(...)                               \
  try {                                            \
    __VA_ARGS__;                                   \
    return 0;                                      \
  } catch (const Error& e) {                       \
    return fail(e, err, errlen);                   \
  } catch (const std::exception& e) {              \
    return fail_other(e, err, errlen);             \
  }

DenseMatrix load(int n, const double* a) {
  DenseMatrix m(n);
  std::copy(a, a + size_t(n) * size_t(n), m.data().begin());
  return m;
}

void store(const DenseMatrix& m, double* out) { std::copy(m.data().begin(), m.data().end(), out); }

std::optional<EvalForm> form_of(int form) {
  if (form == 0) return EvalForm::Plain;
  if (form == 1) return EvalForm::Residual;
  return std::nullopt;
}

TridiagMatrix tridiag(int d, const double* sub, const double* diag, const double* sup) {
  TridiagMatrix t = TridiagMatrix::zero(d);
  std::copy(diag, diag + d, t.diag.begin());
  if (d > 1) {
    std::copy(sub, sub + d - 1, t.sub.begin());
    std::copy(sup, sup + d - 1, t.super.begin());
  }
  return t;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------------ methods (methods.cpp)
typedef struct pfr_method pfr_method;

pfr_method* pfr_catalog(const char* name, char* err, int errlen) {
  try {
    return reinterpret_cast<pfr_method*>(new FractionMethod(catalog(name)));
  } catch (const Error& e) {
    fail(e, err, errlen);
    return nullptr;
  }
}

// build_plain over frac4_template/frac8_template(alpha) for `function` ("exp", "phi1", "cos", ...).
pfr_method* pfr_build_plain(int tmpl, const char* alpha, const char* function, int order, char* err,
                            int errlen) {
  try {
    MethodTemplate t = tmpl == 4 ? frac4_template() : frac8_template();
    std::vector<Rational> shifts = t.shift_pattern(rational_from_string(alpha));
    CoeffSeries series(FunctionId::parse(function));
    return reinterpret_cast<pfr_method*>(
        new FractionMethod(build_plain(shifts, series, order, std::string(function))));
  } catch (const Error& e) {
    fail(e, err, errlen);
    return nullptr;
  }
}

pfr_method* pfr_with_form(const pfr_method* h, int form) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  return reinterpret_cast<pfr_method*>(
      new FractionMethod(form == 1 ? to_residual_form(m) : to_plain_form(m)));
}

void pfr_method_free(pfr_method* h) { delete reinterpret_cast<FractionMethod*>(h); }

// Correctly rounded doubles (rational.cpp:66-88) of the method's coefficients; a0 is
// constant_term() (methods.cpp:80). Buffers hold >= 16 entries.
int pfr_method_doubles(const pfr_method* h, int* n_terms, double* shifts, double* weights, int* n_poly,
                       double* poly, double* a0, int* form) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  *n_terms = int(m.shifts.size());
  for (size_t i = 0; i < m.shifts.size(); ++i) {
    shifts[i] = to_double_nearest(m.shifts[i]);
    weights[i] = to_double_nearest(m.weights[i]);
  }
  *n_poly = int(m.poly.size());
  for (size_t i = 0; i < m.poly.size(); ++i) poly[i] = to_double_nearest(m.poly[i]);
  *a0 = to_double_nearest(m.constant_term());
  *form = m.form == EvalForm::Residual ? 1 : 0;
  return 0;
}

// Exact "num/den" text of every coefficient, '\n'-separated: shifts, then weights, then poly.
int pfr_method_text(const pfr_method* h, char* out, int outlen) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  std::string s;
  for (const auto& q : m.shifts) s += to_fraction_string(q) + "\n";
  for (const auto& q : m.weights) s += to_fraction_string(q) + "\n";
  for (const auto& q : m.poly) s += to_fraction_string(q) + "\n";
  if (int(s.size()) + 1 > outlen) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

// bounds.cpp:252 theta(method, series-of-the-method's-function, tol)
int pfr_theta(const pfr_method* h, double tol, double* theta_out, int* saturated, char* err, int errlen) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  PFR_TRY({
    ThetaResult r = theta(m, CoeffSeries(m.function), tol);
    *theta_out = r.theta;
    if (saturated) *saturated = r.saturated ? 1 : 0;
  });
}

int pfr_theta_taylor(int degree, double tol, double* theta_out, char* err, int errlen) {
  PFR_TRY(*theta_out = theta_taylor(degree, tol));
}

// ------------------------------------------------------------------------ dense.cpp primitives
void pfr_mul(int n, const double* a, const double* b, double* c) { store(load(n, a).mul(load(n, b)), c); }

double pfr_one_norm(int n, const double* a) { return load(n, a).one_norm(); }

int pfr_lu(int n, const double* a, double rel_tol, double* lu, int* piv, char* err, int errlen) {
  PFR_TRY({
    DenseLu f(load(n, a), rel_tol);
    const auto& mir = reinterpret_cast<const DenseLuMirror&>(f);
    std::copy(mir.lu_.begin(), mir.lu_.end(), lu);
    std::copy(mir.piv_.begin(), mir.piv_.end(), piv);
  });
}

int pfr_lu_solve_matrix(int n, const double* a, const double* rhs, double* out, char* err, int errlen) {
  PFR_TRY(store(DenseLu(load(n, a)).solve_matrix(load(n, rhs)), out));
}

int pfr_solve_shifted(int n, const double* b, double c, double* out, char* err, int errlen) {
  PFR_TRY(store(solve_shifted(load(n, b), c), out));
}

int pfr_eval_dense(const pfr_method* h, int form, int n, const double* b, int workers, double* out, char* err,
                   int errlen) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  EvalOptions opts;
  opts.workers = workers;
  opts.form = form_of(form);
  PFR_TRY(store(eval_dense(m, load(n, b), opts), out));
}

// Comparators (dense.cpp:254-332) used by the experiment drivers.
int pfr_baseline(const char* which, int n, const double* b, double* out, char* err, int errlen) {
  PFR_TRY({
    std::string w(which);
    DenseMatrix x = load(n, b);
    if (w == "pade4")
      store(pade4(x), out);
    else if (w == "pade4_phi1")
      store(pade4_phi1(x), out);
    else if (w == "taylor8")
      store(taylor8(x), out);
    else if (w == "pade10")
      store(pade10(x), out);
    else
      raise(Errc::BadArgument, "unknown baseline " + w);
  });
}

// a10 composition from reference primitives: j = smallest j >= 0 with ||A||_1 2^-j <= theta
// (or j_fixed >= 0); B = 2^-j A (DenseMatrix::scale, exact); E = eval_dense(B); E <- E.mul(E).
int pfr_expm(const pfr_method* h, int form, int n, const double* a, double theta, int j_fixed, int workers,
             double* out, int* j_out, char* err, int errlen) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  PFR_TRY({
    DenseMatrix b = load(n, a);
    int j = j_fixed;
    if (j < 0) {
      const double nrm = b.one_norm();
      j = 0;
      while (std::ldexp(nrm, -j) > theta && j < 2000) ++j;
    }
    b.scale(std::ldexp(1.0, -j));
    EvalOptions opts;
    opts.workers = workers;
    opts.form = form_of(form);
    DenseMatrix e = eval_dense(m, b, opts);
    for (int s = 0; s < j; ++s) e = e.mul(e);
    store(e, out);
    if (j_out) *j_out = j;
  });
}

// Batched a10, parallel over the batch with workers = 1 inside (cli.cpp:314 / :228 pattern),
// through the reference's own worker pool (worker_pool.hpp:16-44).
int pfr_expm_batched(const pfr_method* h, int form, int n, int batch, const double* a, double theta, int threads,
                     double* out, int* j_out, int* first_bad, char* err, int errlen) {
  std::vector<int> codes(size_t(std::max(batch, 1)), 0);
  std::vector<std::string> msgs(size_t(std::max(batch, 1)));
  const size_t nn = size_t(n) * size_t(n);
  detail::parallel_for_index(batch, threads, [&](int i) {
    char e[256] = {0};
    codes[size_t(i)] = pfr_expm(h, form, n, a + size_t(i) * nn, theta, -1, 1, out + size_t(i) * nn,
                                j_out ? j_out + i : nullptr, e, sizeof e);
    msgs[size_t(i)] = e;
  });
  for (int i = 0; i < batch; ++i)
    if (codes[size_t(i)]) {
      if (first_bad) *first_bad = i;
      if (err && errlen > 0) {
        std::strncpy(err, msgs[size_t(i)].c_str(), size_t(errlen) - 1);
        err[errlen - 1] = 0;
      }
      return codes[size_t(i)];
    }
  return 0;
}

// a11 + a12 from reference primitives: both weight sets evaluated on the same B (two eval_dense
// calls: the solves are deterministic, so this equals one solve feeding two sums), then
// j times: T = E + I (copy + add_scaled_identity), Phi = 0.5 * (T.mul(Phi)) (scale), E = E.mul(E).
int pfr_expm_phi1(const pfr_method* h_exp, const pfr_method* h_phi, int form, int n, const double* a,
                  double theta, int j_fixed, int workers, double* out_e, double* out_phi, int* j_out, char* err,
                  int errlen) {
  const auto& me = *reinterpret_cast<const FractionMethod*>(h_exp);
  const auto& mp = *reinterpret_cast<const FractionMethod*>(h_phi);
  PFR_TRY({
    DenseMatrix b = load(n, a);
    int j = j_fixed;
    if (j < 0) {
      const double nrm = b.one_norm();
      j = 0;
      while (std::ldexp(nrm, -j) > theta && j < 2000) ++j;
    }
    b.scale(std::ldexp(1.0, -j));
    EvalOptions opts;
    opts.workers = workers;
    opts.form = form_of(form);
    DenseMatrix e = eval_dense(me, b, opts);
    DenseMatrix phi = eval_dense(mp, b, opts);
    for (int s = 0; s < j; ++s) {
      DenseMatrix t = e;
      t.add_scaled_identity(1.0);
      DenseMatrix u = t.mul(phi);
      u.scale(0.5);
      phi = std::move(u);
      e = e.mul(e);
    }
    store(e, out_e);
    store(phi, out_phi);
    if (j_out) *j_out = j;
  });
}

// a13 dense block action from reference primitives, following assemble_action
// (action.cpp:224-284) column by column with DenseLu in place of the Thomas factor:
// B = A * (1.0/substeps) (action.cpp:330-334); every (I - c_i B) factored once
// (ActionOperator, action.cpp:300-312); per substep and column: av = B.matvec(v), residual rhs
// c*av, x = lu.solve(rhs), term = w*x, acc = sum in ascending shift order, + a0*v (+ d1 Av + d2 A^2 v).
int pfr_dense_action(const pfr_method* h, int form, int n, int k, const double* a, const double* v,
                     int substeps, int workers, double* out, char* err, int errlen) {
  const auto& m = *reinterpret_cast<const FractionMethod*>(h);
  PFR_TRY({
    if (substeps < 1 || workers < 1) raise(Errc::BadArgument, "substeps and workers must be >= 1");
    const EvalForm fm = form_of(form).value_or(m.form);
    DenseMatrix b = load(n, a);
    const double inv = 1.0 / substeps;
    for (auto& e : b.data()) e *= inv;
    const int ns = int(m.shifts.size());
    std::vector<std::unique_ptr<DenseLu>> lus(static_cast<size_t>(ns));
    detail::parallel_for_index(ns, workers, [&](int i) {
      const double c = to_double_nearest(m.shifts[size_t(i)]);
      if (c == 0.0) return;
      DenseMatrix mm = b;
      mm.scale(-c);
      mm.add_scaled_identity(1.0);
      try {
        lus[size_t(i)] = std::make_unique<DenseLu>(mm);
      } catch (const Error& e) {
        raise(e.code(), "shift " + std::to_string(i + 1) + ": " + e.what());
      }
    });
    const double constant = fm == EvalForm::Residual ? to_double_nearest(m.constant_term())
                                                     : (m.poly.size() == 3 ? to_double_nearest(m.poly[0]) : 0.0);
    std::vector<double> x(v, v + size_t(n) * size_t(k));
    std::vector<double> col(static_cast<size_t>(n));
    for (int step = 0; step < substeps; ++step) {
      std::vector<double> next(x.size());
      for (int cidx = 0; cidx < k; ++cidx) {
        for (int r = 0; r < n; ++r) col[size_t(r)] = x[size_t(r) * size_t(k) + size_t(cidx)];
        std::vector<double> av;
        if (fm == EvalForm::Residual || m.poly.size() == 3) av = b.matvec(col);
        std::vector<std::vector<double>> terms(static_cast<size_t>(ns));
        detail::parallel_for_index(ns, workers, [&](int i) {
          const double c = to_double_nearest(m.shifts[size_t(i)]);
          const double w = to_double_nearest(m.weights[size_t(i)]);
          std::vector<double> term;
          if (fm == EvalForm::Plain) {
            term = c == 0.0 ? col : lus[size_t(i)]->solve(col);
            for (double& t : term) t *= w;
          } else if (c == 0.0) {
            term.assign(size_t(n), 0.0);
          } else {
            std::vector<double> rhs(static_cast<size_t>(n));
            for (int j = 0; j < n; ++j) rhs[size_t(j)] = c * av[size_t(j)];
            term = lus[size_t(i)]->solve(rhs);
            for (double& t : term) t *= w;
          }
          terms[size_t(i)] = std::move(term);
        });
        std::vector<double> acc(static_cast<size_t>(n), 0.0);
        for (int i = 0; i < ns; ++i)
          for (int j = 0; j < n; ++j) acc[size_t(j)] += terms[size_t(i)][size_t(j)];
        if (fm == EvalForm::Residual || m.poly.size() == 3) {
          for (int j = 0; j < n; ++j) acc[size_t(j)] += constant * col[size_t(j)];
          if (m.poly.size() == 3) {
            const double d1 = to_double_nearest(m.poly[1]), d2 = to_double_nearest(m.poly[2]);
            std::vector<double> a2v = b.matvec(av);
            for (int j = 0; j < n; ++j) acc[size_t(j)] += d1 * av[size_t(j)] + d2 * a2v[size_t(j)];
          }
        }
        for (int r = 0; r < n; ++r) next[size_t(r) * size_t(k) + size_t(cidx)] = acc[size_t(r)];
      }
      x.swap(next);
    }
    std::copy(x.begin(), x.end(), out);
  });
}

// ------------------------------------------------------------------------ action.cpp (banded)
int pfr_thomas_solve(int d, const double* sub, const double* diag, const double* sup, const double* rhs,
                     double* x, char* err, int errlen) {
  PFR_TRY({
    auto r = thomas_solve(tridiag(d, sub, diag, sup), std::span<const double>(rhs, size_t(d)));
    std::copy(r.begin(), r.end(), x);
  });
}

int pfr_tridiag_factor_solve(int d, const double* sub, const double* diag, const double* sup, const double* rhs,
                             double* x, char* err, int errlen) {
  PFR_TRY({
    TridiagFactor f(tridiag(d, sub, diag, sup));
    auto r = f.solve(std::span<const double>(rhs, size_t(d)));
    std::copy(r.begin(), r.end(), x);
  });
}

int pfr_pentadiag_solve(int d, const double* sub2, const double* sub1, const double* diag, const double* super1,
                        const double* super2, const double* rhs, double* x, char* err, int errlen) {
  PFR_TRY({
    PentadiagMatrix p;
    p.d = d;
    p.diag.assign(diag, diag + d);
    p.sub1.assign(sub1, sub1 + std::max(d - 1, 0));
    p.super1.assign(super1, super1 + std::max(d - 1, 0));
    p.sub2.assign(sub2, sub2 + std::max(d - 2, 0));
    p.super2.assign(super2, super2 + std::max(d - 2, 0));
    auto r = pentadiag_solve(p, std::span<const double>(rhs, size_t(d)));
    std::copy(r.begin(), r.end(), x);
  });
}

void pfr_tridiag_matvec(int d, const double* sub, const double* diag, const double* sup, const double* v,
                        double* out) {
  auto r = tridiag(d, sub, diag, sup).matvec(std::span<const double>(v, size_t(d)));
  std::copy(r.begin(), r.end(), out);
}

// mode 0: action_eval; 1: substep_action(substeps); 2: ActionOperator(method, A).apply (one step)
int pfr_tridiag_action(const pfr_method* h, int form, int mode, int d, const double* sub, const double* diag,
                       const double* sup, const double* v, int substeps, int workers, double* out, char* err,
                       int errlen) {
  const auto& m0 = *reinterpret_cast<const FractionMethod*>(h);
  PFR_TRY({
    EvalOptions opts;
    opts.workers = workers;
    opts.form = form_of(form);
    TridiagMatrix t = tridiag(d, sub, diag, sup);
    std::span<const double> vs(v, size_t(d));
    std::vector<double> r;
    if (mode == 0)
      r = action_eval(m0, t, vs, opts);
    else if (mode == 1)
      r = substep_action(m0, t, vs, substeps, opts);
    else
      r = ActionOperator(m0, t).apply(vs, opts);
    std::copy(r.begin(), r.end(), out);
  });
}

// ------------------------------------------------------------------------ generators
void pfr_splitmix(uint64_t seed, int64_t count, uint64_t* out) {
  SplitMix64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next();
}

void pfr_uniform(uint64_t seed, int64_t count, double* out) {
  SplitMix64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.uniform();
}

void pfr_normal(uint64_t seed, int64_t count, double* out) {
  NormalSampler g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next();
}

// cli.cpp:35-56; kind 0 randn, 1 cauchy, 2 trid121
int pfr_make_dense_matrix(int kind, int dim, uint64_t seed, double* out, char* err, int errlen) {
  PFR_TRY({
    MatrixSpec spec;
    spec.kind = kind == 0 ? MatrixSpec::Kind::Randn : kind == 1 ? MatrixSpec::Kind::Cauchy : MatrixSpec::Kind::Trid121;
    spec.dim = dim;
    spec.seed = seed;
    store(make_dense_matrix(spec), out);
  });
}

int pfr_random_unit_vector(int dim, uint64_t seed, double* out, char* err, int errlen) {
  PFR_TRY({
    auto v = random_unit_vector(dim, seed);
    std::copy(v.begin(), v.end(), out);
  });
}

}  // extern "C"
