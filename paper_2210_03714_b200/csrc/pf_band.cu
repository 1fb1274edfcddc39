// C ABI of the banded action (include/pf_b200.h, f2): host orchestration of band.cu's kernels.
// Replaces thomas_solve / TridiagFactor / pentadiag_solve / action_eval / ActionOperator /
// substep_action (proj/core/src/action.cpp:100-339) for blocks of vectors.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pf_host.h"

namespace pf {
__global__ void band_scale_kernel(int d, const double* sub, const double* diag, const double* super, double s,
                                  double* osub, double* odiag, double* osuper);
__global__ void band_factor_kernel(int d, int nsys, const double* sub, const double* diag, const double* super,
                                   const double* shifts, double* mult, double* fdiag, double* fsup, double* frcp,
                                   int* fail);
__global__ void band_solve_kernel(int d, int k, const double* mult, const double* fdiag, const double* fsup,
                                  const double* frcp, const double* src, int64_t lds, const double* rhs_scale,
                                  double* X, int64_t ldx, int64_t strideX);
__global__ void band_matvec_kernel(int d, int k, const double* sub, const double* diag, const double* super,
                                   const double* V, int64_t ldv, double* Out, int64_t ldo);
__global__ void band_accumulate_kernel(int d, int k, int n_terms, const int* slot, const double* w, const double* X,
                                       int64_t ldx, int64_t strideX, const double* V, int64_t ldv, int add_poly,
                                       double constant, int hybrid, double d1, double d2, const double* AV,
                                       const double* A2V, double* out, int64_t ldo);
__global__ void penta_factor_kernel(int d, const double* sub2, const double* sub1, const double* diag,
                                    const double* super1, const double* super2, double* W, double* F, int* fail);
__global__ void penta_solve_kernel(int d, int k, const double* W, const double* F, const double* rhs, int64_t ldr,
                                   double* X, int64_t ldx);
}  // namespace pf

using namespace pf::host;

namespace {

unsigned blocks_for(int64_t elems) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((elems + 255) / 256, 4736)); }

int zero_pivot(pf_status* st, int shift_index, int row) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->code = PF_ERR_ZERO_PIVOT;
    st->shift_index = shift_index;
    st->column = row;
  }
  return PF_ERR_ZERO_PIVOT;
}

// factor nsys systems (shifted by d_shifts when given); returns the first failing system or -1
int factor(pf_context* ctx, int d, int nsys, const double* sub, const double* diag, const double* super,
           const double* d_shifts, double* mult, double* fdiag, double* fsup, double* frcp, int* row, int* rc) {
  int* d_fail = static_cast<int*>(workspace(ctx, kWsSmallArrays + 40, sizeof(int) * std::max(nsys, 1)));
  if (!d_fail) {
    *rc = PF_ERR_CUDA;
    return -1;
  }
  pf::band_factor_kernel<<<(nsys + 31) / 32, 32, 0, ctx->stream>>>(d, nsys, sub, diag, super, d_shifts, mult, fdiag,
                                                                     fsup, frcp, d_fail);
  ctx->launches++;
  std::vector<int> fail(nsys);
  cudaMemcpyAsync(fail.data(), d_fail, sizeof(int) * nsys, cudaMemcpyDeviceToHost, ctx->stream);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    *rc = PF_ERR_CUDA;
    return -1;
  }
  *rc = PF_OK;
  for (int z = 0; z < nsys; ++z)
    if (fail[z] >= 0) {
      *row = fail[z];
      return z;
    }
  return -1;
}

// ---------------------------------------------------------------- banded ActionOperator
// Scaled bands (A / substeps), the P factored shifted systems and the bulk kernel's coefficient
// records, kept on the device between applies (ActionOperator, action.cpp:300-325: factored once).
// One-shot callers (pf_tridiag_action) build it in the context's workspace instead.
}  // namespace

struct pf_tridiag_op {
  pf_context* ctx = nullptr;
  int d = 0, P = 0, substeps = 1;
  bool owns = false;
  std::vector<double> sh;
  std::vector<int> sh_index;
  double* A3 = nullptr;   // ssub | sdiag | ssup
  double* F = nullptr;    // mult | fdiag | fsup | frcp  (P systems each)
  double* rec = nullptr;  // frec | brec
  double* d_sh = nullptr;
};

struct pf_tridiag_factor {
  pf_context* ctx = nullptr;
  int d = 0;
  double* F = nullptr;  // mult | fdiag | fsup | frcp
};

namespace {

void op_free(pf_tridiag_op* op) {
  if (!op->owns) return;
  cudaFree(op->A3);
  cudaFree(op->F);
  cudaFree(op->rec);
  cudaFree(op->d_sh);
  op->A3 = op->F = op->rec = op->d_sh = nullptr;
}

double* op_alloc(pf_tridiag_op* op, int slot, size_t bytes) {
  if (!op->owns) return static_cast<double*>(workspace(op->ctx, slot, bytes));
  void* p = nullptr;
  return cudaMalloc(&p, bytes) == cudaSuccess ? static_cast<double*>(p) : nullptr;
}

int op_build(pf_tridiag_op* op, pf_context* ctx, const pf_method* m, int d, const double* dSub, const double* dDiag,
             const double* dSuper, int substeps, bool one_shot, pf_status* status) {
  op->ctx = ctx;
  op->d = d;
  op->substeps = substeps;
  op->owns = !one_shot;
  const int64_t dm1 = std::max(d - 1, 1);
  for (int i = 0; i < m->n_terms; ++i)  // nonzero shifts in ascending index: one factored system each
    if (m->shifts[i] != 0.0) {
      op->sh.push_back(m->shifts[i]);
      op->sh_index.push_back(i);
    }
  const int P = op->P = (int)op->sh.size();
  op->A3 = op_alloc(op, kWsBandA, sizeof(double) * (size_t)(d + 2 * dm1));
  op->F = op_alloc(op, kWsBandF, sizeof(double) * (size_t)(2 * d + 2 * dm1) * std::max(P, 1));
  op->rec = op_alloc(op, kWsBandRec, sizeof(double) * 8 * (size_t)d * std::max(P, 1));
  op->d_sh = op_alloc(op, kWsSmallArrays + 41, sizeof(double) * std::max(P, 1));
  if (!op->A3 || !op->F || !op->rec || !op->d_sh) return PF_ERR_CUDA;
  double *ssub = op->A3, *sdiag = op->A3 + dm1, *ssup = op->A3 + dm1 + d;
  pf::band_scale_kernel<<<blocks_for(d), 256, 0, ctx->stream>>>(d, dSub, dDiag, dSuper, 1.0 / substeps, ssub, sdiag,
                                                                 ssup);
  ctx->launches++;
  if (P == 0) return PF_OK;
  double *mult = op->F, *fdiag = op->F + dm1 * P, *fsup = op->F + dm1 * P + (int64_t)d * P, *frcp = fsup + dm1 * P;
  cudaMemcpyAsync(op->d_sh, op->sh.data(), sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream);
  int row = 0, rc = PF_OK;
  const int z = factor(ctx, d, P, ssub, sdiag, ssup, op->d_sh, mult, fdiag, fsup, frcp, &row, &rc);
  if (rc) return rc;
  if (z >= 0) return zero_pivot(status, op->sh_index[z] + 1, row);  // "shift i: zero pivot at row r"
  pf::launch_band_pack_records(d, P, ssub, sdiag, ssup, mult, fdiag, fsup, frcp, op->rec, op->rec + (size_t)4 * d * P,
                               ctx->stream);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

// `substeps` fused steps v <- r(A / substeps) v on every column (band.cu), method m's weights and form
// (assemble_action, action.cpp:224-284; the shifts must be the op's)
int op_apply(pf_tridiag_op* op, const pf_method* m, const double* dV, int64_t ldv, int k, double* dOut, int64_t ldo,
             pf_status* status) {
  pf_context* ctx = op->ctx;
  const int d = op->d, P = op->P, substeps = op->substeps;
  {
    std::vector<double> sh;
    for (int i = 0; i < m->n_terms; ++i)
      if (m->shifts[i] != 0.0) sh.push_back(m->shifts[i]);
    if (sh != op->sh) return bad(status);
  }
  const bool residual = m->form == PF_FORM_RESIDUAL;
  const bool hybrid = m->has_poly != 0;
  const int64_t dm1 = std::max(d - 1, 1);
  const size_t blk = (size_t)d * k;
  double *ssub = op->A3, *sdiag = op->A3 + dm1, *ssup = op->A3 + dm1 + d;
  double *mult = op->F, *fdiag = op->F + dm1 * P, *fsup = op->F + dm1 * P + (int64_t)d * P, *frcp = fsup + dm1 * P;
  // P solutions (unfused: P x d x k) or the fused kernel's per-warp forward scratch (P x d x 32 per strip)
  const size_t kpad = (size_t)(k + 31) / 32 * 32;
  double* Y = static_cast<double*>(workspace(ctx, kWsBandY, sizeof(double) * (size_t)d * kpad * std::max(P, 1)));
  if (!Y) return PF_ERR_CUDA;
  // terms in ascending shift index: factored slot, or -1 (plain zero shift: the term is w v)
  std::vector<int> slot;
  std::vector<double> w;
  for (int i = 0, q = 0; i < m->n_terms; ++i) {
    if (m->shifts[i] != 0.0) {
      slot.push_back(q++);
      w.push_back(m->weights[i]);
    } else if (!residual) {
      slot.push_back(-1);
      w.push_back(m->weights[i]);
    }
  }
  const int nt = (int)slot.size();
  int* d_slot = static_cast<int*>(workspace(ctx, kWsSmallArrays + 42, sizeof(int) * std::max(nt, 1)));
  double* d_w = static_cast<double*>(workspace(ctx, kWsSmallArrays + 43, sizeof(double) * std::max(nt, 1)));
  if (!d_slot || !d_w) return PF_ERR_CUDA;
  if (nt) {
    cudaMemcpyAsync(d_slot, slot.data(), sizeof(int) * nt, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_w, w.data(), sizeof(double) * nt, cudaMemcpyHostToDevice, ctx->stream);
  }
  const bool add_poly = residual || hybrid;
  const double constant = residual ? m->constant[0] : (hybrid ? m->poly[0] : 0.0);
  const double d1 = hybrid ? m->poly[1] : 0.0, d2 = hybrid ? m->poly[2] : 0.0;
  static const bool unfused = std::getenv("PF_BAND_UNFUSED") != nullptr;    // A/B switches
  static const bool bulk_ok = std::getenv("PF_BAND_NO_BULK") == nullptr;
  const bool fused = P >= 1 && P <= pf::kBandMaxShifts && nt <= pf::kBandMaxTerms && !unfused;
  // iterates: the fused path ping-pongs two d x k blocks, the unfused chain also keeps A V and A^2 V
  double* XB = static_cast<double*>(workspace(ctx, kWsBandX, sizeof(double) * blk * (fused ? 2 : 4)));
  if (!XB) return PF_ERR_CUDA;
  double *X = XB, *Xn = XB + blk, *AV = fused ? nullptr : XB + 2 * blk, *A2V = fused ? nullptr : XB + 3 * blk;
  if (fused) {
    // fused substeps (band.cu band_action_step_kernel): substep s reads its V (dV for s = 0) and
    // writes the next one (dOut for the last, unless dOut overlaps dV's rows)
    pf::BandStep bs{};
    bs.n_terms = nt;
    for (int q = 0; q < nt; ++q) {
      bs.slot[q] = slot[q];
      bs.w[q] = w[q];
    }
    for (int z = 0; z < P; ++z) bs.c[z] = op->sh[z];
    bs.residual = residual;
    bs.add_poly = add_poly;
    bs.hybrid = hybrid;
    bs.constant = constant;
    bs.d1 = d1;
    bs.d2 = d2;
    bs.direct = nt == P;
    for (int q = 0; q < nt; ++q) bs.direct = bs.direct && slot[q] == q;
    double *frec = op->rec, *brec = op->rec + (size_t)4 * d * P;
    const char *v0 = reinterpret_cast<const char*>(dV), *v1 = v0 + sizeof(double) * ((d - 1) * ldv + k);
    const char *o0 = reinterpret_cast<const char*>(dOut), *o1 = o0 + sizeof(double) * ((d - 1) * ldo + k);
    const bool overlap = o0 < v1 && v0 < o1;
    const double* src = dV;
    int64_t lds = ldv;
    for (int step = 0; step < substeps; ++step) {
      const bool last = step + 1 == substeps;
      double* dst = (last && !overlap) ? dOut : Xn;
      const int64_t ldd = dst == dOut ? ldo : k;
      cudaError_t e = pf::launch_band_action_step(P, d, k, ssub, sdiag, ssup, mult, fdiag, fsup, frcp,
                                                  bulk_ok ? frec : nullptr, brec, bs, src, lds, Y, dst, ldd,
                                                  ctx->stream);
      ctx->launches++;
      if (e != cudaSuccess) return cuda_fail(e);
      src = dst;
      lds = ldd;
      std::swap(X, Xn);
    }
    if (overlap)
      cudaMemcpy2DAsync(dOut, sizeof(double) * ldo, src, sizeof(double) * k, sizeof(double) * k, d,
                        cudaMemcpyDeviceToDevice, ctx->stream);
    return cuda_fail(cudaGetLastError());
  }
  cudaMemcpy2DAsync(X, sizeof(double) * k, dV, sizeof(double) * ldv, sizeof(double) * k, d, cudaMemcpyDeviceToDevice,
                    ctx->stream);
  for (int step = 0; step < substeps; ++step) {
    if (add_poly) {
      pf::band_matvec_kernel<<<blocks_for((int64_t)blk), 256, 0, ctx->stream>>>(d, k, ssub, sdiag, ssup, X, k, AV, k);
      ctx->launches++;
    }
    if (hybrid) {
      pf::band_matvec_kernel<<<blocks_for((int64_t)blk), 256, 0, ctx->stream>>>(d, k, ssub, sdiag, ssup, AV, k, A2V,
                                                                                 k);
      ctx->launches++;
    }
    if (P > 0) {
      pf::band_solve_kernel<<<dim3((k + 127) / 128, P), 128, 0, ctx->stream>>>(
          d, k, mult, fdiag, fsup, frcp, residual ? AV : X, k, residual ? op->d_sh : nullptr, Y, k, (int64_t)blk);
      ctx->launches++;
    }
    pf::band_accumulate_kernel<<<blocks_for((int64_t)blk), 256, 0, ctx->stream>>>(
        d, k, nt, d_slot, d_w, Y, k, (int64_t)blk, X, k, add_poly ? 1 : 0, constant, hybrid ? 1 : 0, d1, d2, AV, A2V,
        Xn, k);
    ctx->launches++;
    std::swap(X, Xn);
  }
  cudaMemcpy2DAsync(dOut, sizeof(double) * ldo, X, sizeof(double) * k, sizeof(double) * k, d,
                    cudaMemcpyDeviceToDevice, ctx->stream);
  return cuda_fail(cudaGetLastError());
}

}  // namespace

extern "C" {

int pf_tridiag_matvec_batched(pf_context* ctx, int d, int k, const double* dSub, const double* dDiag,
                              const double* dSuper, const double* dV, int64_t ldv, double* dOut, int64_t ldo) {
  DeviceGuard device_guard(ctx);
  if (!ctx || d < 0 || k < 0 || ldv < k || ldo < k) return PF_ERR_BAD_ARGUMENT;
  if (d == 0 || k == 0) return PF_OK;
  pf::band_matvec_kernel<<<blocks_for((int64_t)d * k), 256, 0, ctx->stream>>>(d, k, dSub, dDiag, dSuper, dV, ldv,
                                                                              dOut, ldo);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

int pf_thomas_solve_batched(pf_context* ctx, int d, int k, const double* dSub, const double* dDiag,
                            const double* dSuper, const double* dRhs, int64_t ldr, double* dX, int64_t ldx,
                            pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (status) std::memset(status, 0, sizeof(*status));
  if (!ctx || d < 1 || k < 0 || ldr < k || ldx < k) return bad(status);
  const int64_t dm1 = std::max(d - 1, 1);
  double* F = static_cast<double*>(workspace(ctx, kWsBandF, sizeof(double) * (size_t)(2 * d + 2 * dm1)));
  if (!F) return PF_ERR_CUDA;
  double *mult = F, *fdiag = F + dm1, *fsup = F + dm1 + d, *frcp = fsup + dm1;
  int row = 0, rc = PF_OK;
  const int z = factor(ctx, d, 1, dSub, dDiag, dSuper, nullptr, mult, fdiag, fsup, frcp, &row, &rc);
  if (rc) return rc;
  if (z >= 0) return zero_pivot(status, 0, row);
  if (k == 0) return PF_OK;
  pf::band_solve_kernel<<<dim3((k + 127) / 128, 1), 128, 0, ctx->stream>>>(d, k, mult, fdiag, fsup, frcp, dRhs,
                                                                             ldr, nullptr, dX, ldx, 0);
  ctx->launches++;
  return collect_status(ctx, 0, 0, nullptr);
}

int pf_pentadiag_solve_batched(pf_context* ctx, int d, int k, const double* dSub2, const double* dSub1,
                               const double* dDiag, const double* dSuper1, const double* dSuper2,
                               const double* dRhs, int64_t ldr, double* dX, int64_t ldx, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (status) std::memset(status, 0, sizeof(*status));
  if (!ctx || d < 1 || k < 0 || ldr < k || ldx < k) return bad(status);
  double* W = static_cast<double*>(workspace(ctx, kWsBandF, sizeof(double) * (size_t)d * 7));
  int* d_fail = static_cast<int*>(workspace(ctx, kWsSmallArrays + 40, sizeof(int)));
  if (!W || !d_fail) return PF_ERR_CUDA;
  double* F = W + (size_t)d * 5;
  pf::penta_factor_kernel<<<1, 32, 0, ctx->stream>>>(d, dSub2, dSub1, dDiag, dSuper1, dSuper2, W, F, d_fail);
  ctx->launches++;
  int fail = -1;
  cudaMemcpyAsync(&fail, d_fail, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return PF_ERR_CUDA;
  if (fail >= 0) return zero_pivot(status, 0, fail);
  if (k == 0) return PF_OK;
  pf::penta_solve_kernel<<<(k + 127) / 128, 128, 0, ctx->stream>>>(d, k, W, F, dRhs, ldr, dX, ldx);
  ctx->launches++;
  return collect_status(ctx, 0, 0, nullptr);
}

int pf_tridiag_action(pf_context* ctx, const pf_method* m, int d, int k, const double* dSub, const double* dDiag,
                      const double* dSuper, const double* dV, int64_t ldv, int substeps, double* dOut, int64_t ldo,
                      int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (status) std::memset(status, 0, sizeof(*status));
  pf::SmallParams p{};
  if (!ctx || !fill_method(m, p) || d < 1 || k < 0 || substeps < 1 || ldv < k || ldo < k) return bad(status);
  pf_tridiag_op op;  // one-shot: factors in the context's workspace
  int rc = op_build(&op, ctx, m, d, dSub, dDiag, dSuper, substeps, true, status);
  if (rc || k == 0) return rc;  // k == 0: factor-only validation (ActionOperator's constructor)
  rc = op_apply(&op, m, dV, ldv, k, dOut, ldo, status);
  if (rc) return rc;
  return collect_status(ctx, 0, flags, status);
}

int pf_tridiag_op_create(pf_context* ctx, const pf_method* m, int d, const double* dSub, const double* dDiag,
                         const double* dSuper, int substeps, pf_status* status, pf_tridiag_op** out) {
  DeviceGuard device_guard(ctx);
  if (status) std::memset(status, 0, sizeof(*status));
  pf::SmallParams p{};
  if (!out || !ctx || !fill_method(m, p) || d < 1 || substeps < 1) return bad(status);
  *out = nullptr;
  auto* op = new pf_tridiag_op();
  const int rc = op_build(op, ctx, m, d, dSub, dDiag, dSuper, substeps, false, status);
  if (rc) {
    op_free(op);
    delete op;
    return rc;
  }
  *out = op;
  return PF_OK;
}

int pf_tridiag_op_apply(pf_tridiag_op* op, const pf_method* m, const double* dV, int64_t ldv, int k, double* dOut,
                        int64_t ldo, pf_status* status) {
  if (status) std::memset(status, 0, sizeof(*status));
  if (!op) return bad(status);
  DeviceGuard device_guard(op->ctx);
  pf::SmallParams p{};
  if (!fill_method(m, p) || k < 0 || ldv < k || ldo < k) return bad(status);
  if (k == 0) return PF_OK;
  const int rc = op_apply(op, m, dV, ldv, k, dOut, ldo, status);
  if (rc) return rc;
  return collect_status(op->ctx, 0, 0, status);
}

int pf_tridiag_op_destroy(pf_tridiag_op* op) {
  if (!op) return PF_OK;
  DeviceGuard device_guard(op->ctx);
  op_free(op);
  delete op;
  return PF_OK;
}

int pf_tridiag_factor_create(pf_context* ctx, int d, const double* dSub, const double* dDiag, const double* dSuper,
                             pf_status* status, pf_tridiag_factor** out) {
  DeviceGuard device_guard(ctx);
  if (status) std::memset(status, 0, sizeof(*status));
  if (!out || !ctx || d < 1) return bad(status);
  *out = nullptr;
  auto* f = new pf_tridiag_factor();
  f->ctx = ctx;
  f->d = d;
  const int64_t dm1 = std::max(d - 1, 1);
  if (cudaMalloc(&f->F, sizeof(double) * (size_t)(2 * d + 2 * dm1)) != cudaSuccess) {
    delete f;
    return PF_ERR_CUDA;
  }
  int row = 0, rc = PF_OK;
  const int z = factor(ctx, d, 1, dSub, dDiag, dSuper, nullptr, f->F, f->F + dm1, f->F + dm1 + d,
                       f->F + dm1 + d + dm1, &row, &rc);
  if (rc || z >= 0) {
    cudaFree(f->F);
    delete f;
    return rc ? rc : zero_pivot(status, 0, row);
  }
  *out = f;
  return PF_OK;
}

int pf_tridiag_factor_solve(pf_tridiag_factor* f, int k, const double* dRhs, int64_t ldr, double* dX, int64_t ldx) {
  if (!f || k < 0 || ldr < k || ldx < k) return PF_ERR_BAD_ARGUMENT;
  DeviceGuard device_guard(f->ctx);
  if (k == 0) return PF_OK;
  const int64_t dm1 = std::max(f->d - 1, 1);
  pf::band_solve_kernel<<<dim3((k + 127) / 128, 1), 128, 0, f->ctx->stream>>>(
      f->d, k, f->F, f->F + dm1, f->F + dm1 + f->d, f->F + dm1 + f->d + dm1, dRhs, ldr, nullptr, dX, ldx, 0);
  f->ctx->launches++;
  return collect_status(f->ctx, 0, 0, nullptr);
}

int pf_tridiag_factor_destroy(pf_tridiag_factor* f) {
  if (!f) return PF_OK;
  DeviceGuard device_guard(f->ctx);
  cudaFree(f->F);
  delete f;
  return PF_OK;
}

}  // extern "C"
