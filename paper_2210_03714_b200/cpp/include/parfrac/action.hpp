#pragma once
// Banded action surface of the reference (proj/core/include/parfrac/action.hpp:13-82), kept
// source-compatible; the solves run on the B200 through the C ABI (include/pf_b200.h, f2), every
// vector with exactly the reference's operation sequence. New: block variants over k vectors
// (d x k row-major), the shape the GPU is built for.

#include <memory>
#include <span>
#include <vector>

#include "parfrac/dense.hpp"
#include "parfrac/methods.hpp"

namespace parfrac {

/// Compact three-diagonal matrix (action.hpp:13-24).
struct TridiagMatrix {
  int d = 0;
  std::vector<double> sub, diag, super;  // lengths d-1, d, d-1

  static TridiagMatrix zero(int dim);
  /// trid{-1, 2, -1}
  static TridiagMatrix trid121(int dim);

  std::vector<double> matvec(std::span<const double> v) const;  // on the device
  DenseMatrix to_dense() const;
  double one_norm() const;
};

/// Thomas algorithm (action.hpp:29-31); ZeroPivot "zero pivot at row r" below 1e-300.
std::vector<double> thomas_solve(const TridiagMatrix& t, std::span<const double> rhs);

struct TridiagFactorDevice;
struct ActionOperatorDevice;

/// Thomas factorization reused across vectors (action.hpp:35-44): factored ONCE on the device at
/// construction (ZeroPivot there) and kept resident; solve() moves only the right-hand side and
/// performs the same floating-point operations as thomas_solve.
class TridiagFactor {
 public:
  explicit TridiagFactor(const TridiagMatrix& t);
  std::vector<double> solve(std::span<const double> rhs) const;

 private:
  int d_ = 0;
  std::shared_ptr<const TridiagFactorDevice> dev_;
};

/// Compact five-diagonal matrix (action.hpp:48-55).
struct PentadiagMatrix {
  int d = 0;
  std::vector<double> sub2, sub1, diag, super1, super2;

  std::vector<double> matvec(std::span<const double> v) const;
  DenseMatrix to_dense() const;
};

/// Banded LU without pivoting (action.hpp:57).
std::vector<double> pentadiag_solve(const PentadiagMatrix& p, std::span<const double> rhs);

/// r(A) v via shifted tridiagonal solves (action.hpp:63-64).
std::vector<double> action_eval(const FractionMethod& method, const TridiagMatrix& a, std::span<const double> v,
                                const EvalOptions& opts = {});

/// N-fold substepping v <- r(A/N) v (action.hpp:67-69).
std::vector<double> substep_action(const FractionMethod& method, const TridiagMatrix& a, std::span<const double> v,
                                   int substeps, const EvalOptions& opts = {});

/// One method bound to one tridiagonal matrix (action.hpp:73-82); results identical to action_eval.
/// The factored shifted systems live on the device from construction to destruction (factored
/// once, action.cpp:300-312); apply() moves only the vectors.
class ActionOperator {
 public:
  ActionOperator(const FractionMethod& method, const TridiagMatrix& a);
  std::vector<double> apply(std::span<const double> v, const EvalOptions& opts = {}) const;
  /// New: apply to each of the k columns of V (d x k row-major) in one device call.
  std::vector<double> apply_block(std::span<const double> v, int k, const EvalOptions& opts = {}) const;

 private:
  FractionMethod method_;
  TridiagMatrix a_;
  std::shared_ptr<ActionOperatorDevice> dev_;
};

/// New: substep_action on each of the k columns of V (d x k row-major), one device call.
std::vector<double> substep_action_block(const FractionMethod& method, const TridiagMatrix& a,
                                         std::span<const double> v, int k, int substeps, const EvalOptions& opts = {});

}  // namespace parfrac
