// Banded action of the C++ host layer: the reference's API (proj/core/src/action.cpp:15-339) with
// the solves on the B200 through the C ABI (pf_thomas_solve_batched, pf_pentadiag_solve_batched,
// pf_tridiag_action). ZeroPivot messages as the reference's ("shift i: zero pivot at row r").
#include "parfrac/action.hpp"

#include <algorithm>
#include <cmath>

#include "engine.hpp"
#include "parfrac/error.hpp"
#include "pf_b200.h"

namespace parfrac {

using namespace engine;

namespace {

// device copy of the three bands (the off-diagonals of a 1 x 1 matrix are empty: point at diag)
struct DevBand {
  Buf sub, diag, sup;
  DevBand(Device& dev, const TridiagMatrix& t)
      : sub(dev, size_t(std::max(t.d - 1, 1))), diag(dev, size_t(std::max(t.d, 1))),
        sup(dev, size_t(std::max(t.d - 1, 1))) {
    if (int(t.diag.size()) != t.d || int(t.sub.size()) != std::max(t.d - 1, 0) ||
        int(t.super.size()) != std::max(t.d - 1, 0))
      raise(Errc::LengthMismatch, "band length mismatch");
    if (t.d > 1) {
      sub.put(t.sub.data(), size_t(t.d - 1));
      sup.put(t.super.data(), size_t(t.d - 1));
    }
    if (t.d > 0) diag.put(t.diag.data(), size_t(t.d));
  }
};

std::vector<double> tridiag_action_block(const FractionMethod& method, const TridiagMatrix& a,
                                         std::span<const double> v, int k, int substeps, const EvalOptions& opts) {
  if (opts.workers < 1) raise(Errc::BadArgument, "workers must be >= 1");
  if (!opts.fixed_order) raise(Errc::BadArgument, "only fixed-order reduction is supported");
  if (substeps < 1) raise(Errc::BadArgument, "substeps must be >= 1");
  if (k < 0 || v.size() != size_t(a.d) * size_t(k)) raise(Errc::LengthMismatch, "vector length mismatch");
  Packed pk({&method}, opts.form.value_or(method.form));
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  DevBand band(dev, a);
  const size_t n = std::max<size_t>(v.size(), 1);
  Buf in(dev, n), out(dev, n);
  if (!v.empty()) in.put(v.data(), v.size());
  pf_status st{};
  const int rc = pf_tridiag_action(dev.ctx, &pk.m, a.d, k, band.sub.d(), band.diag.d(), band.sup.d(), in.d(), k,
                                   substeps, out.d(), k, 0, &st);
  if (rc) rethrow(rc, st, true);
  std::vector<double> r(v.size());
  if (!r.empty()) out.get(r.data(), r.size());
  return r;
}

}  // namespace

TridiagMatrix TridiagMatrix::zero(int dim) {
  TridiagMatrix t;
  t.d = dim;
  t.sub.assign(size_t(std::max(0, dim - 1)), 0.0);
  t.diag.assign(size_t(dim), 0.0);
  t.super.assign(size_t(std::max(0, dim - 1)), 0.0);
  return t;
}

TridiagMatrix TridiagMatrix::trid121(int dim) {
  TridiagMatrix t = zero(dim);
  std::fill(t.sub.begin(), t.sub.end(), -1.0);
  std::fill(t.diag.begin(), t.diag.end(), 2.0);
  std::fill(t.super.begin(), t.super.end(), -1.0);
  return t;
}

std::vector<double> TridiagMatrix::matvec(std::span<const double> v) const {
  if (int(v.size()) != d) raise(Errc::LengthMismatch, "vector length mismatch");
  if (d == 0) return {};
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  DevBand band(dev, *this);
  Buf in(dev, size_t(d)), out(dev, size_t(d));
  in.put(v.data(), size_t(d));
  const int rc = pf_tridiag_matvec_batched(dev.ctx, d, 1, band.sub.d(), band.diag.d(), band.sup.d(), in.d(), 1,
                                           out.d(), 1);
  if (rc) rethrow(rc, pf_status{}, false);
  std::vector<double> r(static_cast<size_t>(d));
  out.get(r.data(), size_t(d));
  return r;
}

DenseMatrix TridiagMatrix::to_dense() const {
  DenseMatrix m(d);
  for (int i = 0; i < d; ++i) {
    m.at(i, i) = diag[size_t(i)];
    if (i > 0) m.at(i, i - 1) = sub[size_t(i - 1)];
    if (i + 1 < d) m.at(i, i + 1) = super[size_t(i)];
  }
  return m;
}

double TridiagMatrix::one_norm() const {
  double best = 0;
  for (int j = 0; j < d; ++j) {
    double col = std::abs(diag[size_t(j)]);
    if (j > 0) col += std::abs(super[size_t(j - 1)]);
    if (j + 1 < d) col += std::abs(sub[size_t(j)]);
    best = std::max(best, col);
  }
  return best;
}

std::vector<double> thomas_solve(const TridiagMatrix& t, std::span<const double> rhs) {
  if (int(rhs.size()) != t.d) raise(Errc::LengthMismatch, "rhs length mismatch");
  if (t.d == 0) return {};
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  DevBand band(dev, t);
  Buf in(dev, size_t(t.d)), out(dev, size_t(t.d));
  in.put(rhs.data(), size_t(t.d));
  pf_status st{};
  const int rc = pf_thomas_solve_batched(dev.ctx, t.d, 1, band.sub.d(), band.diag.d(), band.sup.d(), in.d(), 1,
                                         out.d(), 1, &st);
  if (rc) rethrow(rc, st, false);
  std::vector<double> r(static_cast<size_t>(t.d));
  out.get(r.data(), size_t(t.d));
  return r;
}

struct TridiagFactorDevice {
  pf_tridiag_factor* f = nullptr;
  ~TridiagFactorDevice() { pf_tridiag_factor_destroy(f); }
};

struct ActionOperatorDevice {
  pf_tridiag_op* op = nullptr;
  ~ActionOperatorDevice() { pf_tridiag_op_destroy(op); }
};

TridiagFactor::TridiagFactor(const TridiagMatrix& t) : d_(t.d) {
  if (t.d == 0) return;
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  DevBand band(dev, t);
  auto f = std::make_shared<TridiagFactorDevice>();
  pf_status st{};
  // factored once; ZeroPivot at construction (action.cpp:120-133)
  const int rc = pf_tridiag_factor_create(dev.ctx, t.d, band.sub.d(), band.diag.d(), band.sup.d(), &st, &f->f);
  if (rc) rethrow(rc, st, false);
  dev_ = std::move(f);
}

std::vector<double> TridiagFactor::solve(std::span<const double> rhs) const {
  if (int(rhs.size()) != d_) raise(Errc::LengthMismatch, "rhs length mismatch");
  if (d_ == 0) return {};
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  Buf in(dev, size_t(d_)), out(dev, size_t(d_));
  in.put(rhs.data(), size_t(d_));
  const int rc = pf_tridiag_factor_solve(dev_->f, 1, in.d(), 1, out.d(), 1);
  if (rc) rethrow(rc, pf_status{}, false);
  std::vector<double> r(static_cast<size_t>(d_));
  out.get(r.data(), size_t(d_));
  return r;
}

std::vector<double> PentadiagMatrix::matvec(std::span<const double> v) const {
  std::vector<double> out(size_t(d), 0.0);
  for (int i = 0; i < d; ++i) {
    double acc = diag[size_t(i)] * v[size_t(i)];
    if (i > 1) acc += sub2[size_t(i - 2)] * v[size_t(i - 2)];
    if (i > 0) acc += sub1[size_t(i - 1)] * v[size_t(i - 1)];
    if (i + 1 < d) acc += super1[size_t(i)] * v[size_t(i + 1)];
    if (i + 2 < d) acc += super2[size_t(i)] * v[size_t(i + 2)];
    out[size_t(i)] = acc;
  }
  return out;
}

DenseMatrix PentadiagMatrix::to_dense() const {
  DenseMatrix m(d);
  for (int i = 0; i < d; ++i) {
    m.at(i, i) = diag[size_t(i)];
    if (i > 1) m.at(i, i - 2) = sub2[size_t(i - 2)];
    if (i > 0) m.at(i, i - 1) = sub1[size_t(i - 1)];
    if (i + 1 < d) m.at(i, i + 1) = super1[size_t(i)];
    if (i + 2 < d) m.at(i, i + 2) = super2[size_t(i)];
  }
  return m;
}

std::vector<double> pentadiag_solve(const PentadiagMatrix& p, std::span<const double> rhs) {
  const int d = p.d;
  if (int(rhs.size()) != d) raise(Errc::LengthMismatch, "rhs length mismatch");
  if (d == 0) return {};
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  Buf s2(dev, std::max<size_t>(p.sub2.size(), 1)), s1(dev, std::max<size_t>(p.sub1.size(), 1)),
      dg(dev, size_t(d)), u1(dev, std::max<size_t>(p.super1.size(), 1)),
      u2(dev, std::max<size_t>(p.super2.size(), 1)), in(dev, size_t(d)), out(dev, size_t(d));
  if (!p.sub2.empty()) s2.put(p.sub2.data(), p.sub2.size());
  if (!p.sub1.empty()) s1.put(p.sub1.data(), p.sub1.size());
  dg.put(p.diag.data(), size_t(d));
  if (!p.super1.empty()) u1.put(p.super1.data(), p.super1.size());
  if (!p.super2.empty()) u2.put(p.super2.data(), p.super2.size());
  in.put(rhs.data(), size_t(d));
  pf_status st{};
  const int rc = pf_pentadiag_solve_batched(dev.ctx, d, 1, s2.d(), s1.d(), dg.d(), u1.d(), u2.d(), in.d(), 1, out.d(),
                                            1, &st);
  if (rc) rethrow(rc, st, false);
  std::vector<double> r(static_cast<size_t>(d));
  out.get(r.data(), size_t(d));
  return r;
}

std::vector<double> action_eval(const FractionMethod& method, const TridiagMatrix& a, std::span<const double> v,
                                const EvalOptions& opts) {
  return tridiag_action_block(method, a, v, 1, 1, opts);
}

std::vector<double> substep_action(const FractionMethod& method, const TridiagMatrix& a, std::span<const double> v,
                                   int substeps, const EvalOptions& opts) {
  if (substeps < 1) raise(Errc::BadArgument, "substeps must be >= 1");
  return tridiag_action_block(method, a, v, 1, substeps, opts);
}

std::vector<double> substep_action_block(const FractionMethod& method, const TridiagMatrix& a,
                                         std::span<const double> v, int k, int substeps, const EvalOptions& opts) {
  return tridiag_action_block(method, a, v, k, substeps, opts);
}

ActionOperator::ActionOperator(const FractionMethod& method, const TridiagMatrix& a) : method_(method), a_(a) {
  // every shifted system factored once, kept on the device: ZeroPivot at construction (action.cpp:300-312)
  if (a.d == 0) return;
  Packed pk({&method_}, method_.form);
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  DevBand band(dev, a);
  auto op = std::make_shared<ActionOperatorDevice>();
  pf_status st{};
  const int rc = pf_tridiag_op_create(dev.ctx, &pk.m, a.d, band.sub.d(), band.diag.d(), band.sup.d(), 1, &st, &op->op);
  if (rc) rethrow(rc, st, true);
  dev_ = std::move(op);
}

std::vector<double> ActionOperator::apply_block(std::span<const double> v, int k, const EvalOptions& opts) const {
  if (opts.workers < 1) raise(Errc::BadArgument, "workers must be >= 1");
  if (!opts.fixed_order) raise(Errc::BadArgument, "only fixed-order reduction is supported");
  if (k < 0 || v.size() != size_t(a_.d) * size_t(k)) raise(Errc::LengthMismatch, "vector length mismatch");
  std::vector<double> r(v.size());
  if (v.empty()) return r;
  Packed pk({&method_}, opts.form.value_or(method_.form));
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  Buf in(dev, v.size()), out(dev, v.size());
  in.put(v.data(), v.size());
  pf_status st{};
  const int rc = pf_tridiag_op_apply(dev_->op, &pk.m, in.d(), k, k, out.d(), k, &st);
  if (rc) rethrow(rc, st, true);
  out.get(r.data(), r.size());
  return r;
}

std::vector<double> ActionOperator::apply(std::span<const double> v, const EvalOptions& opts) const {
  return apply_block(v, 1, opts);
}

}  // namespace parfrac
