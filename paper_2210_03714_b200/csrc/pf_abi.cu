// C ABI (include/pf_b200.h): context, workspace, status plumbing and the host-side
// compositions (scaling and squaring, phi1 doubling, cos/sin recurrence) over the kernels.
// No exceptions cross this boundary; every error is a pf_err code + pf_status.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "pf_host.h"

namespace pf {
namespace host {

int cuda_fail(cudaError_t e) { return e == cudaSuccess ? PF_OK : PF_ERR_CUDA; }

void* workspace(pf_context* ctx, int slot, size_t bytes) {
  if ((int)ctx->ws.size() <= slot) {
    ctx->ws.resize(slot + 1, nullptr);
    ctx->ws_bytes.resize(slot + 1, 0);
  }
  if (ctx->ws_bytes[slot] < bytes) {
    if (ctx->ws[slot]) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->ws[slot]);
    }
    ctx->ws[slot] = nullptr;
    if (cudaMalloc(&ctx->ws[slot], bytes) != cudaSuccess) {
      ctx->ws_bytes[slot] = 0;
      return nullptr;
    }
    ctx->ws_bytes[slot] = bytes;
  }
  return ctx->ws[slot];
}

int ensure_status(pf_context* ctx, int batch) {
  if (ctx->status_cap < batch) {
    if (ctx->status) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->status);
    }
    ctx->status = nullptr;
    int cap = std::max(batch, 1024);
    if (cudaMalloc(&ctx->status, sizeof(pf::DevStatus) * cap) != cudaSuccess) return PF_ERR_CUDA;
    ctx->status_cap = cap;
  }
  if (ctx->sticky) return PF_OK;  // PF_FLAG_STICKY_STATUS callers reset once per pipeline
  return cuda_fail(cudaMemsetAsync(ctx->first_error, 0x7f, sizeof(int), ctx->stream));
}

// Reads the first failing batch entry (if any) back to the host.
int collect_status(pf_context* ctx, int batch, int flags, pf_status* out) {
  if (out) std::memset(out, 0, sizeof(*out));
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) return PF_ERR_CUDA;
  if (flags & PF_FLAG_ASYNC) return PF_OK;
  if (cudaMemcpyAsync(ctx->h_first_error, ctx->first_error, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) !=
      cudaSuccess)
    return PF_ERR_CUDA;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return PF_ERR_CUDA;
  const int b = *ctx->h_first_error;
  if (b < 0 || b >= batch) return PF_OK;
  pf::DevStatus st;
  if (cudaMemcpy(&st, ctx->status + b, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return PF_ERR_CUDA;
  if (out) {
    out->code = st.code;
    out->batch_index = b;
    out->shift_index = st.shift_index;
    out->column = st.column;
    out->pivot_magnitude = st.pivot_magnitude;
    out->scale = st.scale;
  }
  return st.code;
}

int bad(pf_status* st) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->code = PF_ERR_BAD_ARGUMENT;
  }
  return PF_ERR_BAD_ARGUMENT;
}

bool fill_method(const pf_method* m, pf::SmallParams& p) {
  if (!m || m->n_terms < 0 || m->n_terms > PF_MAX_TERMS || m->n_sets < 1 || m->n_sets > 2) return false;
  if (m->n_terms > 0 && (!m->shifts || !m->weights)) return false;
  if (m->form != PF_FORM_PLAIN && m->form != PF_FORM_RESIDUAL) return false;
  if (m->has_poly && !m->poly) return false;
  if (m->form == PF_FORM_RESIDUAL && !m->constant) return false;
  p.n_terms = m->n_terms;
  p.n_sets = m->n_sets;
  p.has_poly = m->has_poly ? 1 : 0;
  p.form = m->form;
  for (int i = 0; i < PF_MAX_TERMS; ++i) {
    p.shifts[i] = i < m->n_terms ? m->shifts[i] : 0.0;
    for (int s = 0; s < 2; ++s) p.weights[s][i] = (i < m->n_terms && s < m->n_sets) ? m->weights[s * m->n_terms + i] : 0.0;
  }
  for (int s = 0; s < 2; ++s) {
    for (int k = 0; k < 3; ++k) p.poly[s][k] = (m->has_poly && s < m->n_sets) ? m->poly[3 * s + k] : 0.0;
    p.constant[s] = (m->constant && s < m->n_sets) ? m->constant[s] : 0.0;
  }
  // (c, -c) shift pairs for the merged residual-form solve (small kernel; the kernel still checks
  // both systems' certificates per matrix and falls back to the per-shift path)
  static const bool no_pairs = std::getenv("PF_NO_PAIRS") != nullptr;
  p.pair_mode = 0;
  for (int i = 0; i < PF_MAX_TERMS; ++i) {
    p.pair_of[i] = 0;
    for (int s = 0; s < 2; ++s) p.pair_cm[s][i] = p.pair_cp[s][i] = 0.0;
  }
  if (m->form == PF_FORM_RESIDUAL && !no_pairs) {
    for (int i = 0; i + 1 < m->n_terms; ++i) {
      const double c = p.shifts[i];
      if (c == 0.0 || p.shifts[i + 1] != -c) continue;
      p.pair_of[i] = 1;
      for (int s = 0; s < 2; ++s) {
        p.pair_cm[s][i] = p.weights[s][i] - p.weights[s][i + 1];
        p.pair_cp[s][i] = p.weights[s][i] + p.weights[s][i + 1];
      }
      p.pair_mode = 1;
      ++i;
    }
  }
  return true;
}

// L2 persistence for a scratch region on the context's stream (PF_NO_L2_PERSIST=1 disables): the
// device-wide set-aside is raised once per device to cover `used` bytes (capped by the device limit)
bool l2_persist_window(pf_context* ctx, void* base, size_t bytes, size_t used) {
  static const bool off = std::getenv("PF_NO_L2_PERSIST") != nullptr;
  if (off) return false;
  int max_persist = 0, max_window = 0;
  if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device) != cudaSuccess ||
      max_persist <= 0 || max_window <= 0) {
    cudaGetLastError();
    return false;
  }
  static std::mutex mu;
  static std::map<int, size_t> set_aside;  // per device
  size_t limit;
  {
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set_aside[ctx->device];
    const size_t want = std::min(used, (size_t)max_persist);
    if (cur < want) {
      if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      cur = want;
    }
    limit = cur;
  }
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.base_ptr = base;
  v.accessPolicyWindow.num_bytes = std::min(bytes, (size_t)max_window);
  // the slots the SMs touch are the first `used` bytes at most (smid < SM count in practice)
  v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)limit / (double)std::max<size_t>(used, 1));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

void l2_persist_clear(pf_context* ctx) {
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

int launch_small(pf_context* ctx, pf::SmallParams& p) {
  auto* kernel = ctx->prof ? pf::small_eval_prof_kernel : pf::small_eval_kernel;
  if (pf::set_smem_attr_once(reinterpret_cast<const void*>(kernel), (int)pf::small_eval_smem_bytes()) != cudaSuccess)
    return PF_ERR_CUDA;
  int rc = ensure_status(ctx, p.batch);
  if (rc) return rc;
  p.status = ctx->status;
  p.first_error = ctx->first_error;
  p.prof = ctx->prof;
  // per-SM accumulator slots: one CTA per SM (smem-bound), so %smid indexes a private slot that
  // stays in L2 across the shifts; slots beyond the guard fall back to the output buffer
  int sms = 148;  // per call (cheap attribute query): no shared mutable state across host threads
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  p.scratch_slots = 2 * sms;
  p.scratch = static_cast<double*>(
      workspace(ctx, kWsScratch, sizeof(double) * 3 * PF_SMALL_N * PF_SMALL_N * (size_t)p.scratch_slots));
  int per_sm = 0;  // the %smid slots are private only at one resident CTA per SM
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, pf::small_eval_threads(),
                                                    pf::small_eval_smem_bytes()) != cudaSuccess ||
      per_sm != 1)
    p.scratch = nullptr;
  if (!p.scratch) p.scratch_slots = 0;
  if (p.batch == 0) return PF_OK;
  // keep the accumulator slots in L2 against the streaming input / output (without this, their dirty
  // lines are evicted and written back: 0.9 GB of DRAM writes per cfg2 launch); the window is set
  // for this launch only and the set-aside is sized to the slots the SMs use
  const bool persist = p.scratch != nullptr && l2_persist_window(ctx, p.scratch, sizeof(double) * 3 * PF_SMALL_N *
                                                                                    PF_SMALL_N * (size_t)p.scratch_slots,
                                                                 sizeof(double) * 3 * PF_SMALL_N * PF_SMALL_N * (size_t)sms);
  kernel<<<p.batch, pf::small_eval_threads(), pf::small_eval_smem_bytes(), ctx->stream>>>(p);
  ctx->launches++;
  const cudaError_t le = cudaGetLastError();
  if (persist) {
    l2_persist_clear(ctx);
    ctx->l2_persisting = true;  // lines stay persisting until the next large-path GEMM resets them
  }
  return cuda_fail(le);
}

int launch_small_reference_order(pf_context* ctx, pf::SmallParams& p) {
  int rc = ensure_status(ctx, p.batch);
  if (rc) return rc;
  p.status = ctx->status;
  p.first_error = ctx->first_error;
  p.prof = nullptr;
  p.scratch_slots = 0;
  p.scratch = static_cast<double*>(workspace(ctx, kWsRefX, sizeof(double) * (size_t)p.n * p.n * (size_t)p.batch));
  if (!p.scratch && p.batch > 0 && p.n > 0) return PF_ERR_CUDA;
  if (p.batch == 0) return PF_OK;
  cudaError_t e = pf::launch_ref_order(p, ctx->stream);
  ctx->launches++;
  return cuda_fail(e);
}

// the fused kernel, or the reference-order evaluator under PF_FLAG_REFERENCE_ORDER
int launch_small_flags(pf_context* ctx, pf::SmallParams& p, int flags) {
  return (flags & PF_FLAG_REFERENCE_ORDER) ? launch_small_reference_order(ctx, p) : launch_small(ctx, p);
}

void gemm(pf_context* ctx, int m, int n, int k, int batch, double alpha, const double* A, int64_t lda,
          int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta, double* C, int64_t ldc, int64_t sC,
          double gamma, const int* jmask, int step, const double* pass, const double* sd_ref, double* sd_d,
          double* sd_e) {
  if (ctx->l2_persisting) {  // the small kernel's slots: give the set-aside back to the GEMM tiles
    cudaCtxResetPersistingL2Cache();
    cudaGetLastError();
    ctx->l2_persisting = false;
  }
  pf::GemmParams g{};
  g.m = m;
  g.n = n;
  g.k = k;
  g.batch = batch;
  g.alpha = alpha;
  g.beta = beta;
  g.gamma = gamma;
  g.A = A;
  g.lda = lda;
  g.strideA = sA;
  g.B = B;
  g.ldb = ldb;
  g.strideB = sB;
  g.C = C;
  g.ldc = ldc;
  g.strideC = sC;
  g.jmask = jmask;
  g.step = step;
  g.pass = pass;
  g.max_sms = ctx->gemm_cap;
  g.sd_ref = sd_ref;
  g.sd_d = sd_d;
  g.sd_e = sd_e;
  const int splits = pf::gemm_split_k(m, n, k);
  // one split workspace per context: not on the LU's concurrent side / look-ahead streams
  bool concurrent = ctx->side != nullptr && ctx->stream == ctx->side;
  for (cudaStream_t a : ctx->aux) concurrent |= ctx->stream == a;
  if (splits > 1 && jmask == nullptr && sd_d == nullptr && !concurrent) {
    const int64_t elems = (int64_t)splits * batch * m * n;
    if (elems * (int64_t)sizeof(double) <= (int64_t)512 << 20) {
      g.split_ws = static_cast<double*>(workspace(ctx, kWsGemmSplit, sizeof(double) * (size_t)elems));
      g.split_ws_elems = g.split_ws ? elems : 0;
      g.splits = g.split_ws ? splits : 1;
    }
  }
  pf::launch_gemm(g, ctx->stream);
  ctx->launches++;
}

int max_j(pf_context* ctx, const int* dJ, int batch, int* out) {
  std::vector<int> h(batch);
  if (cudaMemcpyAsync(h.data(), dJ, sizeof(int) * batch, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
    return PF_ERR_CUDA;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return PF_ERR_CUDA;
  int mj = 0;
  for (int v : h) mj = std::max(mj, v);
  *out = mj;
  return PF_OK;
}

}  // namespace host
}  // namespace pf

using namespace pf::host;

extern "C" {

int pf_version(void) { return 1; }

const char* pf_error_string(int code) {
  switch (code) {
    case PF_OK: return "ok";
    case PF_ERR_DUPLICATE_SHIFT: return "DuplicateShift";
    case PF_ERR_LENGTH_MISMATCH: return "LengthMismatch";
    case PF_ERR_UNDER_DETERMINED: return "UnderDetermined";
    case PF_ERR_UNKNOWN_METHOD: return "UnknownMethod";
    case PF_ERR_INVALID_FUNCTION: return "InvalidFunction";
    case PF_ERR_NON_UNIT_CONSTANT: return "NonUnitConstant";
    case PF_ERR_SINGULAR_SHIFT: return "SingularShift";
    case PF_ERR_ZERO_PIVOT: return "ZeroPivot";
    case PF_ERR_OUT_OF_CONVERGENCE_RADIUS: return "OutOfConvergenceRadius";
    case PF_ERR_BAD_ARGUMENT: return "BadArgument";
    case PF_ERR_CUDA: return "CudaError";
    default: return "unknown";
  }
}

int pf_context_create(int device, pf_context** out) {
  if (!out) return PF_ERR_BAD_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return PF_ERR_CUDA;
  pf_context probe;
  probe.device = device;
  DeviceGuard device_guard(&probe);  // allocate on `device`, leave the caller's current device alone
  auto* ctx = new pf_context();
  ctx->device = device;
  if (cudaMalloc(&ctx->first_error, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_first_error, sizeof(int)) != cudaSuccess) {
    delete ctx;
    return PF_ERR_CUDA;
  }
  *out = ctx;
  return PF_OK;
}

int pf_context_destroy(pf_context* ctx) {
  if (!ctx) return PF_OK;
  DeviceGuard device_guard(ctx);
  group_destroy(ctx);
  cudaStreamSynchronize(ctx->stream);
  for (void* p : ctx->ws) cudaFree(p);
  cudaFree(ctx->status);
  cudaFree(ctx->first_error);
  cudaFreeHost(ctx->h_first_error);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
  }
  for (auto& g : ctx->lu_graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (ctx->gstream) {
    cudaStreamSynchronize(ctx->gstream);
    cudaStreamDestroy(ctx->gstream);
    cudaEventDestroy(ctx->ev_g0);
    cudaEventDestroy(ctx->ev_g1);
  }
  for (size_t d = 0; d < ctx->aux.size(); ++d) {
    cudaStreamSynchronize(ctx->aux[d]);
    cudaStreamDestroy(ctx->aux[d]);
    cudaEventDestroy(ctx->aux_ready[d]);
    cudaEventDestroy(ctx->aux_done[d]);
  }
  delete ctx;
  return PF_OK;
}

int pf_context_set_stream(pf_context* ctx, void* stream) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return PF_OK;
}

int64_t pf_context_launch_count(pf_context* ctx) { return ctx ? ctx->launches : 0; }

int pf_context_set_sticky_status(pf_context* ctx, int sticky) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  ctx->sticky = sticky != 0;
  return cuda_fail(cudaMemsetAsync(ctx->first_error, 0x7f, sizeof(int), ctx->stream));
}

int pf_context_pending_error(pf_context* ctx) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  if (cudaMemcpyAsync(ctx->h_first_error, ctx->first_error, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return PF_ERR_CUDA;
  return *ctx->h_first_error != 0x7f7f7f7f ? 1 : 0;
}

int pf_context_set_profile(pf_context* ctx, unsigned long long* dev_counters) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  ctx->prof = dev_counters;
  return PF_OK;
}

int pf_one_norm_batched(pf_context* ctx, int n, int batch, const double* dA, int64_t lda, int64_t strideA,
                        double* dNorm) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || n < 0 || batch < 0 || lda < n) return PF_ERR_BAD_ARGUMENT;
  if (batch == 0) return PF_OK;
  pf::launch_one_norm(n, batch, dA, lda, strideA, dNorm, ctx->stream);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

int pf_gemm_batched(pf_context* ctx, int m, int n, int k, int batch, double alpha, const double* dA, int64_t lda,
                    int64_t strideA, const double* dB, int64_t ldb, int64_t strideB, double beta, double* dC,
                    int64_t ldc, int64_t strideC, double gamma) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || m < 0 || n < 0 || k < 0 || batch < 0) return PF_ERR_BAD_ARGUMENT;
  if (batch == 0 || m == 0 || n == 0) return PF_OK;
  gemm(ctx, m, n, k, batch, alpha, dA, lda, strideA, dB, ldb, strideB, beta, dC, ldc, strideC, gamma);
  return cuda_fail(cudaGetLastError());
}

int pf_eval_dense_batched(pf_context* ctx, const pf_method* m, int n, int batch, const double* dB, int64_t ldb,
                          int64_t strideB, double* const* dOuts, int64_t ldo, int64_t strideOut, int flags,
                          pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  pf::SmallParams p{};
  if (!ctx || n < 0 || batch < 0 || !dOuts || !fill_method(m, p) || ldb < n || ldo < n) return bad(status);
  if (n > PF_SMALL_N && (flags & PF_FLAG_REFERENCE_ORDER)) return bad(status);
  if (n > PF_SMALL_N) {
    const int rc = large_eval(ctx, m, n, batch, dB, ldb, strideB, nullptr, dOuts, ldo, strideOut, flags, status);
    if (rc) return rc;
    return collect_status(ctx, 0, flags, status);
  }
  p.n = n;
  p.batch = batch;
  p.mode = pf::kModeEval;
  p.force_pivot = (flags & PF_FLAG_FORCE_PIVOT) ? 1 : 0;
  if (flags & PF_FLAG_PER_SHIFT) p.pair_mode = 0;
  p.A = dB;
  p.lda = ldb;
  p.strideA = strideB;
  p.out0 = dOuts[0];
  p.out1 = m->n_sets > 1 ? dOuts[1] : nullptr;
  p.ldo = ldo;
  p.strideOut = strideOut;
  p.pivot_rel_tol = 1e-14;
  int rc = launch_small_flags(ctx, p, flags);
  if (rc) return rc;
  return collect_status(ctx, batch, flags, status);
}

namespace {

// j_b for every matrix into dJ (device): copied from dJin, or the smallest j >= 0 with
// ldexp(||A_b||_1, -j) <= theta (one-norm kernel, dense.cpp:54-62, then the exact count).
void squaring_counts(pf_context* ctx, int n, int batch, const double* dA, int64_t lda, int64_t strideA, double theta,
                     const int* dJin, int* dJ) {
  if (dJin) {
    if (dJin != dJ) cudaMemcpyAsync(dJ, dJin, sizeof(int) * batch, cudaMemcpyDeviceToDevice, ctx->stream);
    return;
  }
  double* norms = static_cast<double*>(workspace(ctx, kWsNorm, sizeof(double) * batch));
  pf::launch_one_norm(n, batch, dA, lda, strideA, norms, ctx->stream);
  pf::launch_squarings(batch, norms, theta, dJ, ctx->stream);
  ctx->launches += 2;
}

// outs[s] = r_s(2^-j_b A_b) for every weight set; j_b written to dJ (device, required).
int eval_scaled(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA, int64_t lda,
                int64_t strideA, const int* dJin, int* dJ, double* const* outs, int64_t ldo, int64_t strideOut,
                int flags, pf_status* status) {
  if (n > PF_SMALL_N && (flags & PF_FLAG_REFERENCE_ORDER)) return bad(status);
  if (n > PF_SMALL_N) {
    squaring_counts(ctx, n, batch, dA, lda, strideA, theta, dJin, dJ);
    const int rc = large_eval(ctx, m, n, batch, dA, lda, strideA, dJ, outs, ldo, strideOut, flags, status);
    if (rc) return rc;
    return collect_status(ctx, 0, flags, status);
  }
  pf::SmallParams p{};
  fill_method(m, p);
  p.n = n;
  p.batch = batch;
  p.mode = pf::kModeScaledEval;
  p.force_pivot = (flags & PF_FLAG_FORCE_PIVOT) ? 1 : 0;
  if (flags & PF_FLAG_PER_SHIFT) p.pair_mode = 0;
  p.A = dA;
  p.lda = lda;
  p.strideA = strideA;
  p.j_in = dJin;
  p.j_out = dJ;
  p.out0 = outs[0];
  p.out1 = m->n_sets > 1 ? outs[1] : nullptr;
  p.ldo = ldo;
  p.strideOut = strideOut;
  p.theta = theta;
  p.pivot_rel_tol = 1e-14;
  int rc = launch_small_flags(ctx, p, flags);
  if (rc) return rc;
  return collect_status(ctx, batch, flags, status);
}

// copy batch of n x n (contiguous, ld n) into a strided destination
void copy_out(pf_context* ctx, int n, int batch, const double* src, double* dst, int64_t ldo, int64_t strideOut) {
  const int64_t nn = (int64_t)n * n;
  if (ldo == n && strideOut == nn) {
    if (src != dst) cudaMemcpyAsync(dst, src, sizeof(double) * nn * batch, cudaMemcpyDeviceToDevice, ctx->stream);
    return;
  }
  for (int b = 0; b < batch; ++b)
    cudaMemcpy2DAsync(dst + b * strideOut, sizeof(double) * ldo, src + b * nn, sizeof(double) * n, sizeof(double) * n,
                      n, cudaMemcpyDeviceToDevice, ctx->stream);
}

}  // namespace

int pf_eval_scaled_batched(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA,
                           int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut,
                           double* const* dOuts, int64_t ldo, int64_t strideOut, int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  pf::SmallParams p{};
  if (!ctx || n < 0 || batch < 0 || !dOuts || !fill_method(m, p) || lda < n || ldo < n ||
      (!dSquaringsIn && !(theta > 0)))
    return bad(status);
  if (batch == 0 || n == 0) return PF_OK;
  int* dJ = dSquaringsOut ? dSquaringsOut : static_cast<int*>(workspace(ctx, kWsJ, sizeof(int) * batch));
  if (!dJ) return PF_ERR_CUDA;
  return eval_scaled(ctx, m, theta > 0 ? theta : 1.0, n, batch, dA, lda, strideA, dSquaringsIn, dJ, dOuts, ldo,
                     strideOut, flags, status);
}

int pf_expm_batched(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA,
                    int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut, double* dOut,
                    int64_t ldo, int64_t strideOut, int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  pf::SmallParams p{};
  if (!ctx || n < 0 || batch < 0 || !dOut || !fill_method(m, p) || lda < n || ldo < n || !(theta > 0))
    return bad(status);
  if (batch == 0 || n == 0) return PF_OK;
  if (n > PF_SMALL_N && (flags & PF_FLAG_REFERENCE_ORDER)) return bad(status);
  if (n > PF_SMALL_N) {
    // eval (set 0) + squaring chain on the DMMA GEMM with per-matrix step counts
    pf_method m0 = *m;
    m0.n_sets = 1;
    const int64_t nn = (int64_t)n * n;
    int* dJ = dSquaringsOut ? dSquaringsOut : static_cast<int*>(workspace(ctx, kWsJ, sizeof(int) * batch));
    double* E = static_cast<double*>(workspace(ctx, kWsT1, sizeof(double) * nn * batch));
    double* T = static_cast<double*>(workspace(ctx, kWsT2, sizeof(double) * nn * batch));
    if (!dJ || !E || !T) return PF_ERR_CUDA;
    double* outs[1] = {E};
    int rc = eval_scaled(ctx, &m0, theta, n, batch, dA, lda, strideA, dSquaringsIn, dJ, outs, n, nn,
                         flags & ~PF_FLAG_ASYNC, status);
    if (rc) return rc;
    int jmax = 0;
    rc = max_j(ctx, dJ, batch, &jmax);
    if (rc) return rc;
    for (int s = 0; s < jmax; ++s) {
      gemm(ctx, n, n, n, batch, 1.0, E, n, nn, E, n, nn, 0.0, T, n, nn, 0.0, dJ, s, E);
      std::swap(E, T);
    }
    copy_out(ctx, n, batch, E, dOut, ldo, strideOut);
    return collect_status(ctx, 0, flags, status);
  }
  p.n = n;
  p.batch = batch;
  p.mode = pf::kModeExpm;
  p.force_pivot = (flags & PF_FLAG_FORCE_PIVOT) ? 1 : 0;
  if (flags & PF_FLAG_PER_SHIFT) p.pair_mode = 0;
  p.A = dA;
  p.lda = lda;
  p.strideA = strideA;
  p.j_in = dSquaringsIn;
  p.j_out = dSquaringsOut;
  p.out0 = dOut;
  p.out1 = nullptr;
  p.n_sets = 1;
  p.ldo = ldo;
  p.strideOut = strideOut;
  p.theta = theta;
  p.pivot_rel_tol = 1e-14;
  int rc = launch_small_flags(ctx, p, flags);
  if (rc) return rc;
  return collect_status(ctx, batch, flags, status);
}

int pf_solve_shifted_batched(pf_context* ctx, int n, int batch, const double* dB, int64_t ldb, int64_t strideB,
                             double c, double* dOut, int64_t ldo, int64_t strideOut, int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  // (I - cB)^{-1} = eval_dense of the one-term plain method {c; 1} (dense.cpp:165-171)
  const double w = 1.0, zero = 0.0;
  pf_method m{1, &c, 1, &w, 0, nullptr, &zero, PF_FORM_PLAIN};
  double* outs[1] = {dOut};
  int rc = pf_eval_dense_batched(ctx, &m, n, batch, dB, ldb, strideB, outs, ldo, strideOut, flags, status);
  if (status && rc) status->shift_index = 0;
  return rc;
}

int pf_expm_phi1_batched(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA,
                         int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut, double* dE,
                         double* dPhi, int64_t ldo, int64_t strideOut, int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  pf::SmallParams p{};
  if (!ctx || n < 0 || batch < 0 || !dE || !dPhi || !fill_method(m, p) || m->n_sets != 2 || lda < n || ldo < n ||
      !(theta > 0))
    return bad(status);
  if (batch == 0 || n == 0) return PF_OK;
  int* dJ = dSquaringsOut ? dSquaringsOut : static_cast<int*>(workspace(ctx, kWsJ, sizeof(int) * batch));
  const int64_t nn = (int64_t)n * n;
  double* E = static_cast<double*>(workspace(ctx, kWsT1, sizeof(double) * nn * batch));
  double* Phi = static_cast<double*>(workspace(ctx, kWsT2, sizeof(double) * nn * batch));
  double* spare = static_cast<double*>(workspace(ctx, kWsT3, sizeof(double) * nn * batch));
  double* T = static_cast<double*>(workspace(ctx, kWsT4, sizeof(double) * nn * batch));
  if (!dJ || !E || !Phi || !spare || !T) return PF_ERR_CUDA;
  double* outs[2] = {E, Phi};
  int rc = eval_scaled(ctx, m, theta, n, batch, dA, lda, strideA, dSquaringsIn, dJ, outs, n, nn,
                       flags & ~PF_FLAG_ASYNC, status);
  if (rc) return rc;
  int jmax = 0;
  rc = max_j(ctx, dJ, batch, &jmax);
  if (rc) return rc;
  // Phi <- 0.5 (E + I) Phi ; E <- E E   (per-matrix step count j_b)
  for (int s = 0; s < jmax; ++s) {
    pf::launch_scale_add_identity(n, batch, 1.0, E, n, nn, 1.0, T, n, nn, ctx->stream);
    ctx->launches++;
    gemm(ctx, n, n, n, batch, 0.5, T, n, nn, Phi, n, nn, 0.0, spare, n, nn, 0.0, dJ, s, Phi);
    std::swap(Phi, spare);
    gemm(ctx, n, n, n, batch, 1.0, E, n, nn, E, n, nn, 0.0, spare, n, nn, 0.0, dJ, s, E);
    std::swap(E, spare);
  }
  copy_out(ctx, n, batch, E, dE, ldo, strideOut);
  copy_out(ctx, n, batch, Phi, dPhi, ldo, strideOut);
  return collect_status(ctx, 0, flags, status);
}

int pf_cossin_batched(pf_context* ctx, const pf_pair_method* pm, double theta, int n, int batch, const double* dA,
                      int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut, double* dC,
                      double* dS, int64_t ldo, int64_t strideOut, int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  if (!ctx || !pm || pm->n_pairs < 0 || pm->n_pairs > PF_MAX_TERMS || n < 0 || batch < 0 || !dC || !dS || lda < n ||
      ldo < n || !(theta > 0))
    return bad(status);
  if (batch == 0 || n == 0) return PF_OK;
  const int64_t nn = (int64_t)n * n;
  int* dJ = dSquaringsOut ? dSquaringsOut : static_cast<int*>(workspace(ctx, kWsJ, sizeof(int) * batch));
  double* Bm = static_cast<double*>(workspace(ctx, kWsT1, sizeof(double) * nn * batch));
  double* B2 = static_cast<double*>(workspace(ctx, kWsT2, sizeof(double) * nn * batch));
  double* Sp = static_cast<double*>(workspace(ctx, kWsT3, sizeof(double) * nn * batch));
  double* T = static_cast<double*>(workspace(ctx, kWsT4, sizeof(double) * nn * batch));
  if (!dJ || !Bm || !B2 || !Sp || !T) return PF_ERR_CUDA;
  squaring_counts(ctx, n, batch, dA, lda, strideA, theta, dSquaringsIn, dJ);
  pf::launch_ldexp_batched(n, batch, dA, lda, strideA, dJ, Bm, n, nn, ctx->stream);
  ctx->launches++;
  gemm(ctx, n, n, n, batch, 1.0, Bm, n, nn, Bm, n, nn, 0.0, B2, n, nn, 0.0);
  // cos = a0 I + sum cw X, S' = a1 I + sum sw X with X = (I + c^2 B^2)^{-1} (-c^2 B^2): the residual
  // evaluator on B^2 with shifts -c^2 (Z_c = -X, see pf_b200.h)
  std::vector<double> shifts(pm->n_pairs), weights(2 * pm->n_pairs);
  for (int k = 0; k < pm->n_pairs; ++k) {
    shifts[k] = -pm->c2[k];
    weights[k] = pm->cw[k];
    weights[pm->n_pairs + k] = pm->sw[k];
  }
  const double constants[2] = {pm->a0, pm->a1};
  pf_method m{pm->n_pairs, shifts.data(), 2, weights.data(), 0, nullptr, constants, PF_FORM_RESIDUAL};
  double* outs[2] = {T, Sp};  // C, S'
  int rc = pf_eval_dense_batched(ctx, &m, n, batch, B2, n, nn, outs, n, nn, flags & ~PF_FLAG_ASYNC, status);
  if (rc) return rc;
  double* C = T;
  double* S = B2;  // B^2 no longer needed
  gemm(ctx, n, n, n, batch, 1.0, Bm, n, nn, Sp, n, nn, 0.0, S, n, nn, 0.0);
  int jmax = 0;
  rc = max_j(ctx, dJ, batch, &jmax);
  if (rc) return rc;
  double* C2 = Bm;  // B no longer needed
  // double angle: C <- C^2 - S^2 = (C - S)(C + S) (C and S are functions of the same matrix, so they
  // commute), S <- 2 S C: two GEMMs per step instead of three; matrices past their own j pass through
  double* D = jmax > 0 ? static_cast<double*>(workspace(ctx, kWsPairB, sizeof(double) * nn * batch)) : nullptr;
  double* Ep = jmax > 0 ? static_cast<double*>(workspace(ctx, kWsPairT, sizeof(double) * nn * batch)) : nullptr;
  if (jmax > 0 && (!D || !Ep)) return PF_ERR_CUDA;
  // D = C - S and E = C + S come from the epilogue of the GEMM that produces S (it reads C's tile
  // there), so no separate elementwise pass: the first from S = B S', then from every S <- 2 S C
  for (int s = 0; s < jmax; ++s) {
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
  copy_out(ctx, n, batch, C, dC, ldo, strideOut);
  copy_out(ctx, n, batch, S, dS, ldo, strideOut);
  return collect_status(ctx, 0, flags, status);
}

int pf_action_block(pf_context* ctx, const pf_method* m, int n, int k, const double* dA, int64_t lda,
                    const double* dV, int64_t ldv, int substeps, double* dOut, int64_t ldo, int flags,
                    pf_status* status) {
  DeviceGuard device_guard(ctx);
  pf::SmallParams p{};
  if (!ctx || !fill_method(m, p) || n < 0 || k < 0 || substeps < 1 || lda < n || ldv < k || ldo < k || !dA || !dV ||
      !dOut)
    return bad(status);
  if (n == 0 || k == 0) return PF_OK;
  const int rc = large_action(ctx, m, n, k, dA, lda, dV, ldv, substeps, dOut, ldo, flags, status);
  if (rc) return rc;
  return collect_status(ctx, 0, flags, status);
}

int pf_lu_factor_batched(pf_context* ctx, int n, int batch, double* dA, int64_t lda, int64_t strideA, int* dPiv,
                         double pivot_rel_tol, int flags, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    if (status) std::memset(status, 0, sizeof(*status));
    return PF_OK;
  }
  if (!ctx || n < 0 || batch < 0 || lda < n || !(pivot_rel_tol >= 0)) return bad(status);
  const int rc = large_lu_factor(ctx, n, batch, dA, lda, strideA, dPiv, pivot_rel_tol, flags, status);
  if (rc) return rc;
  return collect_status(ctx, 0, flags, status);
}

int pf_lu_solve_batched(pf_context* ctx, int n, int k, int batch, const double* dLU, int64_t lda, int64_t strideLU,
                        const int* dPiv, double* dRhs, int64_t ldr, int64_t strideR) {
  DeviceGuard device_guard(ctx);
  if (ctx && batch == 0) {  // nothing to evaluate (null buffers of empty tensors are fine)
    return PF_OK;
  }
  if (!ctx || n < 0 || k < 0 || batch < 0 || lda < n || ldr < k || !dPiv) return PF_ERR_BAD_ARGUMENT;
  const int rc = large_lu_solve(ctx, n, k, batch, dLU, lda, strideLU, dPiv, dRhs, ldr, strideR);
  if (rc) return rc;
  return collect_status(ctx, 0, 0, nullptr);
}

int pf_device_alloc(pf_context* ctx, size_t bytes, void** out) {
  DeviceGuard device_guard(ctx);
  if (!ctx || !out) return PF_ERR_BAD_ARGUMENT;
  *out = nullptr;
  if (bytes == 0) return PF_OK;
  return cuda_fail(cudaMalloc(out, bytes));
}

int pf_device_free(pf_context* ctx, void* p) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  if (!p) return PF_OK;
  cudaStreamSynchronize(ctx->stream);
  return cuda_fail(cudaFree(p));
}

int pf_copy_to_device(pf_context* ctx, void* dst, const void* src, size_t bytes) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  if (bytes == 0) return PF_OK;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) return PF_ERR_CUDA;
  return cuda_fail(cudaStreamSynchronize(ctx->stream));
}

int pf_copy_to_host(pf_context* ctx, void* dst, const void* src, size_t bytes) {
  DeviceGuard device_guard(ctx);
  if (!ctx) return PF_ERR_BAD_ARGUMENT;
  if (bytes == 0) return PF_OK;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess) return PF_ERR_CUDA;
  return cuda_fail(cudaStreamSynchronize(ctx->stream));
}

}  // extern "C"
