// C-ABI building blocks for shift-partitioned (multi-GPU) evaluation and for callers that drive the
// scaling-and-squaring stages themselves:
//   pf_squarings_batched       j_b from the 1-norm (K6)
//   pf_ordered_sum             ((t_0 + t_1) + t_2) + ...  -- the fixed ascending-shift reduction of
//                              eval_dense (dense.cpp:245-246), used by the deterministic multi-GPU mode
//   pf_square_chain / pf_phi1_doubling / pf_cossin_doubling   the recurrences
//   pf_action_create / _apply / _apply_terms / _destroy       ActionOperator (action.hpp:68-82) for a
//                              dense A: factor once, apply r(B) to many blocks; a shift mask lets every
//                              rank own a subset of the shifts (NCCL all-reduce between applies)
#include <algorithm>
#include <cstring>
#include <vector>

#include "pf_host.h"

namespace pf {

__global__ void ordered_sum_kernel(const double* const* terms, int count, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = terms[0][i];
    for (int t = 1; t < count; ++t) acc = __dadd_rn(acc, terms[t][i]);
    out[i] = acc;
  }
}

namespace host {

int square_chain(pf_context* ctx, int n, int batch, const int* dJ, double* E, double* spare) {
  int jmax = 0;
  int rc = max_j(ctx, dJ, batch, &jmax);
  if (rc) return rc;
  const int64_t nn = (int64_t)n * n;
  double* cur = E;
  double* nxt = spare;
  for (int s = 0; s < jmax; ++s) {
    gemm(ctx, n, n, n, batch, 1.0, cur, n, nn, cur, n, nn, 0.0, nxt, n, nn, 0.0, dJ, s, cur);
    std::swap(cur, nxt);
  }
  if (cur != E) cudaMemcpyAsync(E, cur, sizeof(double) * nn * batch, cudaMemcpyDeviceToDevice, ctx->stream);
  return cuda_fail(cudaGetLastError());
}

}  // namespace host
}  // namespace pf

using namespace pf::host;

extern "C" {

int pf_action_create(pf_context* ctx, const pf_method* m, int n, const double* dA, int64_t lda, int substeps,
                     const int* owned, int flags, pf_status* status, pf_action_op** out) {
  DeviceGuard device_guard(ctx);
  pf::SmallParams p{};
  if (!ctx || !out || !fill_method(m, p) || n < 1 || lda < n || substeps < 1 || !dA) return bad(status);
  *out = nullptr;
  const int rc = action_op_create(ctx, m, n, dA, lda, substeps, owned, flags, status, out);
  if (rc) return rc;
  return collect_status(ctx, 0, flags, status);
}

int pf_action_apply(pf_action_op* op, const double* dV, int64_t ldv, int k, double* dOut, int64_t ldo,
                    int include_poly, double* dTerms, pf_status* status) {
  if (!op || !dV || k < 1 || ldv < k || ldo < k || !dOut) return bad(status);
  DeviceGuard device_guard(op->ctx);
  const int rc = action_op_apply(op, dV, ldv, k, dOut, ldo, include_poly, dTerms);
  if (rc) return rc;
  return collect_status(op->ctx, 0, 0, status);
}

int pf_action_term_count(pf_action_op* op) { return op ? (int)op->term_index.size() : 0; }

int pf_action_destroy(pf_action_op* op) {
  if (!op) return PF_OK;
  DeviceGuard device_guard(op->ctx);
  action_op_destroy(op);
  return PF_OK;
}

int pf_squarings_batched(pf_context* ctx, int n, int batch, const double* dA, int64_t lda, int64_t strideA,
                         double theta, int* dJ) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || n < 0 || batch < 0 || lda < n || !(theta > 0) || !dJ) return PF_ERR_BAD_ARGUMENT;
  if (batch == 0) return PF_OK;
  double* norms = static_cast<double*>(workspace(ctx, kWsNorm, sizeof(double) * batch));
  if (!norms) return PF_ERR_CUDA;
  pf::launch_one_norm(n, batch, dA, lda, strideA, norms, ctx->stream);
  pf::launch_squarings(batch, norms, theta, dJ, ctx->stream);
  ctx->launches += 2;
  return cuda_fail(cudaGetLastError());
}

int pf_add_identity_rows(pf_context* ctx, int rows, int n, int r0, const double* dX, int64_t ldx, double* dY,
                         int64_t ldy) {
  DeviceGuard device_guard(ctx);
  if (!ctx || rows < 0 || n < 0 || r0 < 0 || ldx < n || ldy < n) return PF_ERR_BAD_ARGUMENT;
  if (rows == 0 || n == 0) return PF_OK;
  pf::launch_add_identity_rows(rows, n, r0, dX, ldx, dY, ldy, ctx->stream);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

int pf_sum_diff(pf_context* ctx, int64_t count, const double* dC, const double* dS, double* dDiff, double* dSum) {
  DeviceGuard device_guard(ctx);
  if (!ctx || count < 0 || (!dDiff && !dSum)) return PF_ERR_BAD_ARGUMENT;
  if (count == 0) return PF_OK;
  pf::launch_sum_diff(count, dC, dS, dDiff, dSum, ctx->stream);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

int pf_ordered_sum(pf_context* ctx, int count, const double* const* dTerms, int64_t n_elems, double* dOut) {
  DeviceGuard device_guard(ctx);
  if (!ctx || count < 1 || !dTerms || n_elems < 0 || !dOut) return PF_ERR_BAD_ARGUMENT;
  if (n_elems == 0) return PF_OK;
  auto** dptrs = static_cast<const double**>(workspace(ctx, kWsSmallArrays + 30, sizeof(double*) * count));
  if (!dptrs) return PF_ERR_CUDA;
  cudaMemcpyAsync(dptrs, dTerms, sizeof(double*) * count, cudaMemcpyHostToDevice, ctx->stream);
  const int64_t blocks = std::min<int64_t>((n_elems + 255) / 256, 4736);
  pf::ordered_sum_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(dptrs, count, n_elems, dOut);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

int pf_square_chain(pf_context* ctx, int n, int batch, const int* dJ, double* dE) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || n < 0 || batch < 0 || !dJ || !dE) return PF_ERR_BAD_ARGUMENT;
  if (batch == 0 || n == 0) return PF_OK;
  double* spare = static_cast<double*>(workspace(ctx, kWsT3, sizeof(double) * (size_t)n * n * batch));
  if (!spare) return PF_ERR_CUDA;
  int rc = square_chain(ctx, n, batch, dJ, dE, spare);
  if (rc) return rc;
  return collect_status(ctx, 0, 0, nullptr);
}

int pf_phi1_doubling(pf_context* ctx, int n, int batch, const int* dJ, double* dE, double* dPhi) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || n < 0 || batch < 0 || !dJ || !dE || !dPhi) return PF_ERR_BAD_ARGUMENT;
  if (batch == 0 || n == 0) return PF_OK;
  const int64_t nn = (int64_t)n * n;
  const size_t bytes = sizeof(double) * nn * batch;
  double* E = static_cast<double*>(workspace(ctx, kWsT1, bytes));
  double* Phi = static_cast<double*>(workspace(ctx, kWsT2, bytes));
  double* spare = static_cast<double*>(workspace(ctx, kWsT3, bytes));
  double* T = static_cast<double*>(workspace(ctx, kWsT4, bytes));
  if (!E || !Phi || !spare || !T) return PF_ERR_CUDA;
  int jmax = 0;
  int rc = max_j(ctx, dJ, batch, &jmax);
  if (rc) return rc;
  cudaMemcpyAsync(E, dE, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  cudaMemcpyAsync(Phi, dPhi, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  // Phi <- 0.5 (E + I) Phi ; E <- E E   (per-matrix step count j_b)
  for (int s = 0; s < jmax; ++s) {
    pf::launch_scale_add_identity(n, batch, 1.0, E, n, nn, 1.0, T, n, nn, ctx->stream);
    ctx->launches++;
    gemm(ctx, n, n, n, batch, 0.5, T, n, nn, Phi, n, nn, 0.0, spare, n, nn, 0.0, dJ, s, Phi);
    std::swap(Phi, spare);
    gemm(ctx, n, n, n, batch, 1.0, E, n, nn, E, n, nn, 0.0, spare, n, nn, 0.0, dJ, s, E);
    std::swap(E, spare);
  }
  cudaMemcpyAsync(dE, E, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  cudaMemcpyAsync(dPhi, Phi, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  return collect_status(ctx, 0, 0, nullptr);
}

int pf_cossin_doubling(pf_context* ctx, int n, int batch, const int* dJ, double* dC, double* dS) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || n < 0 || batch < 0 || !dJ || !dC || !dS) return PF_ERR_BAD_ARGUMENT;
  if (batch == 0 || n == 0) return PF_OK;
  const int64_t nn = (int64_t)n * n;
  const size_t bytes = sizeof(double) * nn * batch;
  double* C = static_cast<double*>(workspace(ctx, kWsT1, bytes));
  double* S = static_cast<double*>(workspace(ctx, kWsT2, bytes));
  double* C2 = static_cast<double*>(workspace(ctx, kWsT3, bytes));
  double* Sp = static_cast<double*>(workspace(ctx, kWsT4, bytes));
  if (!C || !S || !C2 || !Sp) return PF_ERR_CUDA;
  int jmax = 0;
  int rc = max_j(ctx, dJ, batch, &jmax);
  if (rc) return rc;
  cudaMemcpyAsync(C, dC, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  cudaMemcpyAsync(S, dS, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  // C <- C C - S S = (C - S)(C + S) ; S <- 2 (S C)  (same steps as pf_cossin_batched)
  // double angle: C <- C^2 - S^2 = (C - S)(C + S) (C and S are functions of the same matrix, so they
  // commute), S <- 2 S C: two GEMMs per step instead of three; matrices past their own j pass through
  double* D = jmax > 0 ? static_cast<double*>(workspace(ctx, kWsPairB, sizeof(double) * nn * batch)) : nullptr;
  double* Ep = jmax > 0 ? static_cast<double*>(workspace(ctx, kWsPairT, sizeof(double) * nn * batch)) : nullptr;
  if (jmax > 0 && (!D || !Ep)) return PF_ERR_CUDA;
  for (int s = 0; s < jmax; ++s) {  // D / E of the next step from the S GEMM's epilogue
    if (s == 0) {
      pf::launch_sum_diff(nn * batch, C, S, D, Ep, ctx->stream);
      ctx->launches++;
    }
    gemm(ctx, n, n, n, batch, 1.0, D, n, nn, Ep, n, nn, 0.0, C2, n, nn, 0.0, dJ, s, C);
    const bool more = s + 1 < jmax;
    gemm(ctx, n, n, n, batch, 2.0, S, n, nn, C, n, nn, 0.0, Sp, n, nn, 0.0, dJ, s, S, more ? C2 : nullptr,
         more ? D : nullptr, more ? Ep : nullptr);
    std::swap(C, C2);
    std::swap(S, Sp);
  }
  cudaMemcpyAsync(dC, C, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  cudaMemcpyAsync(dS, S, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
  return collect_status(ctx, 0, 0, nullptr);
}

}  // extern "C"
