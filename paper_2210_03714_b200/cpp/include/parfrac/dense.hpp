#pragma once
// Dense evaluator surface of the reference (proj/core/include/parfrac/dense.hpp:12-75), kept
// source-compatible; the numerical work runs on the B200 through the C ABI (include/pf_b200.h).
// New entry points: expm / expm_phi1 / cossin with scaling and squaring, batched
// evaluation, and the dense block action.

#include <memory>
#include <optional>
#include <span>
#include <vector>

#include "parfrac/methods.hpp"

namespace parfrac {

/// Square row-major double-precision matrix (dense.hpp:13-38).
class DenseMatrix {
 public:
  DenseMatrix() = default;
  explicit DenseMatrix(int dim) : d_(dim), a_(size_t(dim) * size_t(dim), 0.0) {}

  static DenseMatrix identity(int dim);

  int dim() const { return d_; }
  double& at(int i, int j) { return a_[size_t(i) * size_t(d_) + size_t(j)]; }
  double at(int i, int j) const { return a_[size_t(i) * size_t(d_) + size_t(j)]; }
  std::span<const double> data() const { return a_; }
  std::span<double> data() { return a_; }

  DenseMatrix mul(const DenseMatrix& o) const;  // on the device (DMMA GEMM)
  std::vector<double> matvec(std::span<const double> v) const;
  void axpy(double s, const DenseMatrix& x);  // this += s x
  void add_scaled_identity(double s);
  void scale(double s);

  double one_norm() const;  // max column sum
  double max_abs() const;

 private:
  int d_ = 0;
  std::vector<double> a_;
};

struct DenseLuDevice;  // the factors and pivots kept in device memory (dense.cpp)

/// LU factors with partial pivoting (dense.hpp:44-59); factored on the device, and the factors STAY
/// there: every solve / solve_matrix reuses them (only the right-hand sides move). Copies share
/// the immutable device factors.
class DenseLu {
 public:
  DenseLu(const DenseMatrix& a, double pivot_rel_tol = 1e-14);

  std::vector<double> solve(std::span<const double> rhs) const;
  DenseMatrix solve_matrix(const DenseMatrix& rhs) const;
  /// The swap sequence (0-based, LAPACK style). The reference keeps it private (piv_).
  const std::vector<int>& pivots() const { return piv_; }
  const std::vector<double>& factors() const { return lu_; }

 private:
  int d_ = 0;
  std::vector<double> lu_;
  std::vector<int> piv_;
  std::shared_ptr<const DenseLuDevice> dev_;
};

/// (I - cB)^{-1} (dense.hpp:62)
DenseMatrix solve_shifted(const DenseMatrix& b, double c);

struct EvalOptions {
  int workers = 1;
  bool fixed_order = true;
  std::optional<EvalForm> form;
  /// New (B200): the reference's worker pool over shifts (dense.cpp:202) as GPUs. devices > 1 or a
  /// device_ids list partitions the shifts of ONE matrix over those GPUs (pf_eval_multi_gpu, one
  /// NCCL exchange); with fixed_order (always, as in the reference) the result is bit-identical
  /// for any device count. device_ids overrides devices (ids 0..devices-1).
  int devices = 1;
  std::vector<int> device_ids;
};

/// r(B) (dense.hpp:70-75)
DenseMatrix eval_dense(const FractionMethod& method, const DenseMatrix& b, const EvalOptions& opts = {});

/// Batched r(B_k): every matrix of `bs` must have the same dimension.
std::vector<DenseMatrix> eval_dense_batched(const FractionMethod& method, const std::vector<DenseMatrix>& bs,
                                            const EvalOptions& opts = {});

/// exp(A) = r(2^-j A)^(2^j), j = smallest j >= 0 with ||A||_1 2^-j <= theta (residual form by default).
DenseMatrix expm(const FractionMethod& method, const DenseMatrix& a, EvalForm form = EvalForm::Residual,
                 int* squarings = nullptr);
std::vector<DenseMatrix> expm_batched(const FractionMethod& method, const std::vector<DenseMatrix>& as,
                                      EvalForm form = EvalForm::Residual);

/// exp(A) with EvalOptions: form override, and devices / device_ids for the shift-partitioned
/// multi-GPU evaluation (one exchange, then the squaring on the first device).
DenseMatrix expm(const FractionMethod& method, const DenseMatrix& a, const EvalOptions& opts, int* squarings = nullptr);

/// (exp(A), phi1(A)) from one solve per shift, then phi1 doubling (multi-GPU with opts.devices).
std::pair<DenseMatrix, DenseMatrix> expm_phi1(const FractionMethod& method, const DenseMatrix& a,
                                              const EvalOptions& opts = {});

/// (cos(A), sin(A)) through merged conjugate shift pairs and C^2 - S^2 / 2SC.
std::pair<DenseMatrix, DenseMatrix> cossin(const FractionMethod& method, const DenseMatrix& a);

/// exp(A) V for an n x k block V (row-major), substeps V <- r(A/N) V with one LU per shift
/// (dense analogue of substep_action, action.hpp:61-66). N = 0 selects ceil(||A||_1 / theta).
std::vector<double> substep_action(const FractionMethod& method, const DenseMatrix& a, std::span<const double> v,
                                   int k, int substeps = 0, const EvalOptions& opts = {});

}  // namespace parfrac
