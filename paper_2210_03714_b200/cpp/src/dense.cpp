// Dense evaluator of the C++ host layer: the reference's API (proj/core/src/dense.cpp:11-252) with
// the numerical work on the B200 through the C ABI. Value semantics, parfrac::Error exceptions and
// the "shift i: singular system: ..." messages are preserved; exceptions never cross the ABI.
#include "parfrac/dense.hpp"

#include <algorithm>
#include <cmath>
#include <mutex>

#include "engine.hpp"
#include "parfrac/error.hpp"
#include "pf_b200.h"

namespace parfrac {

struct DenseLuDevice {
  engine::Buf lu, piv;
  DenseLuDevice(pf_context* ctx, int d) : lu(ctx, size_t(d) * d), piv(ctx, (size_t(d) + 1) / 2) {}
};

namespace {

using namespace engine;

DenseMatrix from_flat(int d, const double* p) {
  DenseMatrix m(d);
  std::copy(p, p + size_t(d) * d, m.data().begin());
  return m;
}

std::vector<int> device_list(const EvalOptions& opts) {
  if (!opts.device_ids.empty()) return opts.device_ids;
  if (opts.devices < 1) raise(Errc::BadArgument, "devices must be >= 1");
  std::vector<int> ids(size_t(opts.devices));
  for (int i = 0; i < opts.devices; ++i) ids[size_t(i)] = i;
  return ids;
}

bool multi_gpu(const EvalOptions& opts) { return opts.devices > 1 || !opts.device_ids.empty(); }

// ONE matrix over the devices `ids` (pf_eval_multi_gpu, deterministic: the reference's fixed-order
// contract); returns the output of every weight set of `sets`
std::vector<DenseMatrix> eval_multi(const std::vector<const FractionMethod*>& sets, EvalForm form, const DenseMatrix& a,
                                    int recurrence, double theta, const std::vector<int>& ids, int* squarings) {
  Packed pk(sets, form);
  MultiDevices& md = multi_devices();
  std::lock_guard<std::mutex> lock(md.mu);
  pf_context* ctx = md.get(ids);
  const int d = a.dim();
  const size_t nn = size_t(d) * d;
  std::vector<DenseMatrix> res(sets.size(), DenseMatrix(d));
  if (nn == 0) return res;
  Buf in(ctx, nn), o0(ctx, nn), o1(ctx, sets.size() > 1 ? nn : 1);
  in.put(a.data().data(), nn);
  pf_status st{};
  int j = 0;
  const int rc = pf_eval_multi_gpu(ctx, &pk.m, theta, recurrence, d, in.d(), d, o0.d(), sets.size() > 1 ? o1.d() : nullptr,
                                   d, 1, 0, &j, &st);
  if (rc) rethrow(rc, st, true);
  o0.get(res[0].data().data(), nn);
  if (sets.size() > 1) o1.get(res[1].data().data(), nn);
  if (squarings) *squarings = j;
  return res;
}

}  // namespace

DenseMatrix DenseMatrix::identity(int dim) {
  DenseMatrix m(dim);
  for (int i = 0; i < dim; ++i) m.at(i, i) = 1.0;
  return m;
}

DenseMatrix DenseMatrix::mul(const DenseMatrix& o) const {
  if (o.dim() != d_) raise(Errc::LengthMismatch, "matrix dimension mismatch");
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const size_t nn = size_t(d_) * d_;
  DenseMatrix out(d_);
  if (nn == 0) return out;
  Buf a(dev, nn), b(dev, nn), c(dev, nn);
  a.put(a_.data(), nn);
  b.put(o.a_.data(), nn);
  const int rc = pf_gemm_batched(dev.ctx, d_, d_, d_, 1, 1.0, a.d(), d_, 0, b.d(), d_, 0, 0.0, c.d(), d_, 0, 0.0);
  if (rc) rethrow(rc, pf_status{}, false);
  c.get(out.a_.data(), nn);
  return out;
}

std::vector<double> DenseMatrix::matvec(std::span<const double> v) const {
  std::vector<double> out(size_t(d_), 0.0);
  for (int i = 0; i < d_; ++i) {
    double acc = 0;
    const double* row = &a_[size_t(i) * size_t(d_)];
    for (int j = 0; j < d_; ++j) acc += row[j] * v[size_t(j)];
    out[size_t(i)] = acc;
  }
  return out;
}

void DenseMatrix::axpy(double s, const DenseMatrix& x) {
  for (size_t i = 0; i < a_.size(); ++i) a_[i] += s * x.a_[i];
}

void DenseMatrix::add_scaled_identity(double s) {
  for (int i = 0; i < d_; ++i) at(i, i) += s;
}

void DenseMatrix::scale(double s) {
  for (auto& v : a_) v *= s;
}

double DenseMatrix::one_norm() const {
  double best = 0;
  for (int j = 0; j < d_; ++j) {
    double col = 0;
    for (int i = 0; i < d_; ++i) col += std::abs(at(i, j));
    best = std::max(best, col);
  }
  return best;
}

double DenseMatrix::max_abs() const {
  double best = 0;
  for (double v : a_) best = std::max(best, std::abs(v));
  return best;
}

DenseLu::DenseLu(const DenseMatrix& a, double pivot_rel_tol) : d_(a.dim()), lu_(a.data().begin(), a.data().end()) {
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const size_t nn = size_t(d_) * d_;
  piv_.resize(size_t(d_));
  if (nn == 0) return;
  auto f = std::make_shared<DenseLuDevice>(dev.ctx, d_);
  f->lu.put(lu_.data(), nn);
  pf_status st{};
  const int rc = pf_lu_factor_batched(dev.ctx, d_, 1, f->lu.d(), d_, 0, f->piv.i(), pivot_rel_tol, 0, &st);
  if (rc) rethrow(rc, st, false);
  f->lu.get(lu_.data(), nn);  // host copies for factors() / pivots(); the device keeps its own
  Buf::check(pf_copy_to_host(dev.ctx, piv_.data(), f->piv.d(), sizeof(int) * size_t(d_)));
  dev_ = std::move(f);
}

DenseMatrix DenseLu::solve_matrix(const DenseMatrix& rhs) const {
  if (rhs.dim() != d_) raise(Errc::LengthMismatch, "matrix dimension mismatch");
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const size_t nn = size_t(d_) * d_;
  DenseMatrix out = rhs;
  if (nn == 0) return out;
  Buf r(dev, nn);
  r.put(rhs.data().data(), nn);
  const int rc = pf_lu_solve_batched(dev.ctx, d_, d_, 1, dev_->lu.d(), d_, 0, dev_->piv.i(), r.d(), d_, 0);
  if (rc) rethrow(rc, pf_status{}, false);
  r.get(out.data().data(), nn);
  return out;
}

std::vector<double> DenseLu::solve(std::span<const double> rhs) const {
  if (int(rhs.size()) != d_) raise(Errc::LengthMismatch, "vector length mismatch");
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  std::vector<double> x(rhs.begin(), rhs.end());
  if (d_ == 0) return x;
  Buf r(dev, size_t(d_));
  r.put(x.data(), size_t(d_));
  const int rc = pf_lu_solve_batched(dev.ctx, d_, 1, 1, dev_->lu.d(), d_, 0, dev_->piv.i(), r.d(), 1, 0);
  if (rc) rethrow(rc, pf_status{}, false);
  r.get(x.data(), size_t(d_));
  return x;
}

DenseMatrix solve_shifted(const DenseMatrix& b, double c) {
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const int d = b.dim();
  const size_t nn = size_t(d) * d;
  if (nn == 0) return DenseMatrix(d);
  Buf in(dev, nn), out(dev, nn);
  in.put(b.data().data(), nn);
  pf_status st{};
  const int rc = pf_solve_shifted_batched(dev.ctx, d, 1, in.d(), d, 0, c, out.d(), d, 0, 0, &st);
  if (rc) rethrow(rc, st, false);
  DenseMatrix r(d);
  out.get(r.data().data(), nn);
  return r;
}

std::vector<DenseMatrix> eval_dense_batched(const FractionMethod& method, const std::vector<DenseMatrix>& bs,
                                            const EvalOptions& opts) {
  if (opts.workers < 1) raise(Errc::BadArgument, "workers must be >= 1");
  if (!opts.fixed_order) raise(Errc::BadArgument, "only fixed-order reduction is supported");
  std::vector<DenseMatrix> res;
  if (bs.empty()) return res;
  const int d = bs[0].dim();
  for (const auto& b : bs)
    if (b.dim() != d) raise(Errc::LengthMismatch, "batched matrices must share the dimension");
  const EvalForm form = opts.form.value_or(method.form);
  Packed pk({&method}, form);
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const size_t nn = size_t(d) * d, batch = bs.size();
  if (nn == 0) return std::vector<DenseMatrix>(batch, DenseMatrix(d));
  Buf in(dev, nn * batch), out(dev, nn * batch);
  std::vector<double> host(nn * batch);
  for (size_t k = 0; k < batch; ++k) std::copy(bs[k].data().begin(), bs[k].data().end(), host.begin() + k * nn);
  in.put(host.data(), nn * batch);
  double* outs[1] = {out.d()};
  pf_status st{};
  const int rc = pf_eval_dense_batched(dev.ctx, &pk.m, d, int(batch), in.d(), d, int64_t(nn), outs, d, int64_t(nn), 0, &st);
  if (rc) rethrow(rc, st, true);
  out.get(host.data(), nn * batch);
  for (size_t k = 0; k < batch; ++k) res.push_back(from_flat(d, host.data() + k * nn));
  return res;
}

DenseMatrix eval_dense(const FractionMethod& method, const DenseMatrix& b, const EvalOptions& opts) {
  if (multi_gpu(opts)) {
    if (opts.workers < 1) raise(Errc::BadArgument, "workers must be >= 1");
    if (!opts.fixed_order) raise(Errc::BadArgument, "only fixed-order reduction is supported");
    return eval_multi({&method}, opts.form.value_or(method.form), b, PF_REC_NONE, 0.0, device_list(opts), nullptr)[0];
  }
  return eval_dense_batched(method, {b}, opts)[0];
}

std::vector<DenseMatrix> expm_batched(const FractionMethod& method, const std::vector<DenseMatrix>& as, EvalForm form) {
  std::vector<DenseMatrix> res;
  if (as.empty()) return res;
  const int d = as[0].dim();
  Packed pk({&method}, form);
  const double th = theta_u53(method);
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const size_t nn = size_t(d) * d, batch = as.size();
  Buf in(dev, nn * batch), out(dev, nn * batch);
  std::vector<double> host(nn * batch);
  for (size_t k = 0; k < batch; ++k) std::copy(as[k].data().begin(), as[k].data().end(), host.begin() + k * nn);
  in.put(host.data(), nn * batch);
  pf_status st{};
  const int rc = pf_expm_batched(dev.ctx, &pk.m, th, d, int(batch), in.d(), d, int64_t(nn), nullptr, nullptr, out.d(),
                                 d, int64_t(nn), 0, &st);
  if (rc) rethrow(rc, st, true);
  out.get(host.data(), nn * batch);
  for (size_t k = 0; k < batch; ++k) res.push_back(from_flat(d, host.data() + k * nn));
  return res;
}

DenseMatrix expm(const FractionMethod& method, const DenseMatrix& a, EvalForm form, int* squarings) {
  DenseMatrix e = expm_batched(method, {a}, form)[0];
  if (squarings) {
    const double th = theta_u53(method);
    const double nrm = a.one_norm();
    int j = 0;
    while (std::ldexp(nrm, -j) > th && j < 2000) ++j;
    *squarings = j;
  }
  return e;
}

DenseMatrix expm(const FractionMethod& method, const DenseMatrix& a, const EvalOptions& opts, int* squarings) {
  if (opts.workers < 1) raise(Errc::BadArgument, "workers must be >= 1");
  if (!opts.fixed_order) raise(Errc::BadArgument, "only fixed-order reduction is supported");
  const EvalForm form = opts.form.value_or(EvalForm::Residual);
  if (!multi_gpu(opts)) return expm(method, a, form, squarings);
  return eval_multi({&method}, form, a, PF_REC_EXP, theta_u53(method), device_list(opts), squarings)[0];
}

std::pair<DenseMatrix, DenseMatrix> expm_phi1(const FractionMethod& method, const DenseMatrix& a,
                                              const EvalOptions& opts) {
  const FractionMethod& phi = derived_set(method.name + "_phi1set");
  const double th = std::min(theta_u53(method), phi.theta_u53);
  if (multi_gpu(opts)) {
    auto r = eval_multi({&method, &phi}, EvalForm::Residual, a, PF_REC_EXP_PHI1, th, device_list(opts), nullptr);
    return {r[0], r[1]};
  }
  Packed pk({&method, &phi}, EvalForm::Residual);
  const int d = a.dim();
  const size_t nn = size_t(d) * d;
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  Buf in(dev, nn), e(dev, nn), p(dev, nn);
  in.put(a.data().data(), nn);
  pf_status st{};
  const int rc = pf_expm_phi1_batched(dev.ctx, &pk.m, th, d, 1, in.d(), d, 0, nullptr, nullptr, e.d(), p.d(), d, 0, 0, &st);
  if (rc) rethrow(rc, st, true);
  DenseMatrix E(d), P(d);
  e.get(E.data().data(), nn);
  p.get(P.data().data(), nn);
  return {E, P};
}

std::pair<DenseMatrix, DenseMatrix> cossin(const FractionMethod& method, const DenseMatrix& a) {
  const PairMethod& pm = pair_method(method.name);
  std::vector<double> c2, cw, sw;
  for (size_t k = 0; k < pm.c2.size(); ++k) {
    c2.push_back(to_double_nearest(pm.c2[k]));
    cw.push_back(to_double_nearest(pm.cw[k]));
    sw.push_back(to_double_nearest(pm.sw[k]));
  }
  pf_pair_method p{int(c2.size()), c2.data(), cw.data(), sw.data(), to_double_nearest(pm.a0), to_double_nearest(pm.a1)};
  const int d = a.dim();
  const size_t nn = size_t(d) * d;
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  Buf in(dev, nn), c(dev, nn), s(dev, nn);
  in.put(a.data().data(), nn);
  pf_status st{};
  const int rc = pf_cossin_batched(dev.ctx, &p, theta_u53(method), d, 1, in.d(), d, 0, nullptr, nullptr, c.d(), s.d(),
                                   d, 0, 0, &st);
  if (rc) rethrow(rc, st, true);
  DenseMatrix C(d), S(d);
  c.get(C.data().data(), nn);
  s.get(S.data().data(), nn);
  return {C, S};
}

std::vector<double> substep_action(const FractionMethod& method, const DenseMatrix& a, std::span<const double> v,
                                   int k, int substeps, const EvalOptions& opts) {
  if (opts.workers < 1) raise(Errc::BadArgument, "workers must be >= 1");
  if (!opts.fixed_order) raise(Errc::BadArgument, "only fixed-order reduction is supported");
  const int d = a.dim();
  if (k < 1 || v.size() != size_t(d) * size_t(k)) raise(Errc::LengthMismatch, "vector length mismatch");
  if (substeps == 0) {
    const double nrm = a.one_norm(), th = theta_u53(method);
    substeps = nrm <= th ? 1 : int(std::ceil(nrm / th));
  }
  if (substeps < 1) raise(Errc::BadArgument, "substeps must be >= 1");
  Packed pk({&method}, opts.form.value_or(method.form));
  Device& dev = device();
  std::lock_guard<std::mutex> lock(dev.mu);
  const size_t nn = size_t(d) * d, nk = size_t(d) * k;
  Buf ad(dev, nn), vd(dev, nk), od(dev, nk);
  ad.put(a.data().data(), nn);
  vd.put(v.data(), nk);
  pf_status st{};
  const int rc = pf_action_block(dev.ctx, &pk.m, d, k, ad.d(), d, vd.d(), k, substeps, od.d(), k, 0, &st);
  if (rc) rethrow(rc, st, true);
  std::vector<double> out(nk);
  od.get(out.data(), nk);
  return out;
}

}  // namespace parfrac
