// Internal kernel parameter blocks and launchers (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "pf_b200.h"

namespace pf {

struct DevStatus;

enum SmallMode {
  kModeEval = 0,        // r(B) for every weight set, B = A (no scaling)
  kModeScaledEval = 1,  // r(2^-j A) for every weight set, j from the norm or j_in
  kModeExpm = 2,        // r(2^-j A) for set 0, then j squarings
};

struct SmallParams {
  int n, batch, mode;
  int n_terms, n_sets, has_poly, form, force_pivot;
  const double* A;
  int64_t lda, strideA;
  const int* j_in;
  int* j_out;
  double* out0;
  double* out1;
  int64_t ldo, strideOut;
  double theta, pivot_rel_tol;
  double shifts[PF_MAX_TERMS];
  double weights[2][PF_MAX_TERMS];
  double poly[2][3];
  double constant[2];
  DevStatus* status;
  int* first_error;
  unsigned long long* prof;  // optional phase profile (diagnostics), nullptr normally
  double* scratch;           // per-SM slots of 3 x 128 x 128 doubles (acc set 0, acc set 1, B^2), or nullptr
  int scratch_slots;
  // pair mode (residual form): shifts i, i+1 = (c, -c) merged into one solve of (I - c^2 B^2);
  // pair_of[i] = 1 marks the first shift of a pair, cm = w_i - w_{i+1}, cp = w_i + w_{i+1}
  int pair_mode;
  int pair_of[PF_MAX_TERMS];
  double pair_cm[2][PF_MAX_TERMS];
  double pair_cp[2][PF_MAX_TERMS];
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, current device): the
// attribute is per device, and one process may drive several (api.Engine(device=...)).
cudaError_t set_smem_attr_once(const void* fn, int bytes);

__global__ void small_eval_kernel(SmallParams p);
__global__ void small_eval_prof_kernel(SmallParams p);  // with the phase profile (p.prof)
size_t small_eval_smem_bytes();
// PF_FLAG_REFERENCE_ORDER evaluator (ref_order.cu); p.scratch = batch x n x n doubles
cudaError_t launch_ref_order(SmallParams& p, cudaStream_t stream);
int small_eval_threads();

// Batched C = alpha * A B + beta * C + gamma * I (row-major, FP64 DMMA).
struct GemmParams {
  int m, n, k, batch;
  double alpha, beta, gamma;
  const double* A;
  int64_t lda, strideA;
  const double* B;
  int64_t ldb, strideB;
  double* C;
  int64_t ldc, strideC;
  // per-matrix step predication for recurrences with matrix-dependent step counts:
  // matrix z is inactive at `step` when jmask && step >= jmask[z]; an inactive matrix gets
  // C = pass (copy) when pass != nullptr, else C is left untouched.
  const int* jmask;
  int step;
  const double* pass;
  // > 0: persistent launch on at most max_sms SMs' worth of CTAs, each looping over tiles (leaves
  // SMs free for concurrent work on other streams)
  int max_sms;
  // optional epilogue (the cos/sin double angle, pf_cossin_batched): with sd_d != nullptr, for every
  // written element v of C also sd_d = ref - v and sd_e = ref + v, ref = sd_ref (C's layout)
  const double* sd_ref;
  double* sd_d;
  double* sd_e;
  // split-K workspace for thin products (gemm_split_k): splits x batch x m x n doubles, or nullptr
  double* split_ws;
  int64_t split_ws_elems;
  int splits;  // gemm_split_k's choice (0 / 1: none)
};
void launch_gemm(const GemmParams& p, cudaStream_t stream);
// the device-scheduled LU's TMA operand maps over its systems: a = box 16 x 128 (L tile columns x
// rows), b = box 16 x 16 (U tile columns x k rows)
struct DagMaps {
  CUtensorMap a;
  CUtensorMap b;
};
// a 3-D FP64 tensor map (inner, outer, batch; 128-byte swizzle) for TMA boxes of box_inner x box_outer
bool make_tma_map(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint64_t batch, int64_t ld,
                  int64_t stride, unsigned box_inner, unsigned box_outer);

// K splits of the TMA GEMM for thin, long products (n <= 128 columns -- the action's 64 right-hand
// sides -- whose m x n output is at most 64 tiles per matrix): too few tiles to fill the SMs, so the
// k range is cut into 2-4 pieces (k / 512) summed in order by a second pass. A function of the
// product's own shape only -- not of the batch -- so the same product splits the same way however
// the systems are partitioned over devices (deterministic multi-GPU results stay bit-identical).
inline int gemm_split_k(int m, int n, int k) {
  if (n > 128 || k < 1024) return 1;
  const long long tiles = (long long)((m + 63) / 64) * ((n + 63) / 64);
  if (tiles > 64) return 1;
  const int s = k / 512;
  return s > 4 ? 4 : s;
}

// accumulate_sets_kernel (large.cu): up to four weighted sums of the same solutions in one pass
struct AccSet {
  const double* w;  // device, n_terms weights
  double constant, d1, d2;
  int add_poly;
  double* out;
  int64_t ldo, strideOut;
};
struct AccSets {
  AccSet s[4];
  int n;
};

// Partial-pivoting panel of the blocked large LU (pivot_lu.cu): rows [off, np) x columns [off, off+w)
// of each of nsys systems, pivots into piv[z * npiv + col]; the panel's row exchanges are then applied
// to every other column (moves: 2 * 64 int2 per system). SingularShift below tol[z] is recorded for
// system zorig[z] and marks failed[z] (later panels skip it).
cudaError_t launch_panel_lu(double* M, int64_t ld, int64_t strideM, int np, int off, int w, int nsys, int* piv,
                            int npiv, const double* tol, const int* zorig, int* failed, DevStatus* status,
                            int* first_error, int2* moves, int* moves_n, cudaStream_t stream,
                            cudaEvent_t panel_done = nullptr);  // recorded after the panel, before the moves

// Batched 1-norm (column sums in ascending row order, then max).
void launch_one_norm(int n, int batch, const double* A, int64_t lda, int64_t strideA, double* out,
                     cudaStream_t stream);

// Elementwise helpers used by the host-side compositions.
// Y = alpha * X  (+ beta on the diagonal), batched n x n
void launch_scale_add_identity(int n, int batch, double alpha, const double* X, int64_t ldx, int64_t strideX,
                               double diag, double* Y, int64_t ldy, int64_t strideY, cudaStream_t stream);
// Y = ldexp(X, -j_b) per matrix (j from device array)
void launch_ldexp_batched(int n, int batch, const double* X, int64_t ldx, int64_t strideX, const int* j, double* Y,
                          int64_t ldy, int64_t strideY, cudaStream_t stream);
// rows [r0, r0 + rows) of X + I (row block of the phi1 doubling's E + I)
void launch_add_identity_rows(int rows, int n, int r0, const double* X, int64_t ldx, double* Y, int64_t ldy,
                              cudaStream_t stream);
// D = C - S, E = C + S over `count` contiguous doubles (either output may be null)
void launch_sum_diff(int64_t count, const double* C, const double* S, double* D, double* E, cudaStream_t stream);
// squarings from norms: j_b = smallest j >= 0 with ldexp(norm_b, -j) <= theta
void launch_squarings(int batch, const double* norms, double theta, int* j, cudaStream_t stream);

// One fused substep of the banded (tridiagonal) action, band.cu: P factored shifted systems
// (P <= kBandMaxShifts), the ascending-index term list (slot = factored system, -1 = the plain
// form's zero shift: w v) and the polynomial part. frcp = band_rcp(fdiag) per system. Y = the
// forward sweep's scratch, P x d x 32 per 32-column strip.
constexpr int kBandMaxShifts = 12;
constexpr int kBandMaxTerms = 24;
struct BandStep {
  int n_terms;
  int slot[kBandMaxTerms];
  double w[kBandMaxTerms];
  double c[kBandMaxShifts];
  int residual, add_poly, hybrid;
  int direct;  // the terms are exactly the P factored systems in order (slot[q] == q, n_terms == P)
  double constant, d1, d2;
};
cudaError_t launch_band_action_step(int P, int d, int k, const double* ssub, const double* sdiag, const double* ssup,
                                    const double* mult, const double* fdiag, const double* fsup, const double* frcp,
                                    const double* frec, const double* brec, const BandStep& st, const double* V,
                                    int64_t ldv, double* Y, double* out, int64_t ldo, cudaStream_t s);
// frec / brec (nsys x d x 4 each): the bulk kernel's per-row coefficient records (band.cu)
void launch_band_pack_records(int d, int nsys, const double* ssub, const double* sdiag, const double* ssup,
                              const double* mult, const double* fdiag, const double* fsup, const double* frcp,
                              double* frec, double* brec, cudaStream_t s);

}  // namespace pf
