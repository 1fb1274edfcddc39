/* pf_b200.h -- C ABI of the B200 partial-fraction matrix-function engine.
 *
 * The reference (proj/core, C++20) has no C or FFI layer: its drop-in surface is the C++ API
 * in proj/core/include/parfrac/. This header is the thin C boundary that the C++ host layer
 * (paper_2210_03714_b200/cpp/, namespace parfrac) and the Python mirror call into. No torch
 * types, no exceptions: every entry point returns a pf_err code and fills pf_status so the
 * host can rethrow the identical parfrac::Error (error.hpp:8-44).
 *
 * Entry point                 replaces (reference file:line)
 * --------------------------  ------------------------------------------------------------------
 * pf_eval_dense_batched       eval_dense(method, B, opts)        proj/core/include/parfrac/dense.hpp:74-75
 *                             (dense.cpp:193-252; one call = many independent B)
 * pf_expm_batched             new: eval_dense + scaling and squaring (pattern expm_oracle
 *                             dense.cpp:460-476, theta from bounds.hpp:62)
 * pf_expm_phi1_batched        new: one solve per shift feeds exp and phi1 weight sets
 *                              + phi1 doubling
 * pf_cossin_batched           new: cos/sin pair through merged conjugate shifts + C^2-S^2 / 2SC
 * pf_action_block             new dense analogue of substep_action / ActionOperator
 *                             (action.hpp:61-82, action.cpp:224-339)
 * pf_lu_factor / pf_lu_solve  DenseLu(a, pivot_rel_tol) / DenseLu::solve_matrix (dense.hpp:46-59)
 * pf_solve_shifted            solve_shifted(b, c) (dense.hpp:62)
 * pf_one_norm_batched         DenseMatrix::one_norm (dense.hpp:32, dense.cpp:54-62)
 * pf_gemm_batched             DenseMatrix::mul (dense.hpp:26, dense.cpp:17-29)
 * pf_context_create_multi     new: the worker pool of eval_dense (EvalOptions.workers, dense.hpp:64-68;
 *   + pf_eval_multi_gpu       dense.cpp:202 parallel_for_index, worker_pool.hpp:16-44) as devices: the
 *                             shifts of ONE matrix partitioned over GPUs, one NCCL exchange, results
 *                             bit-identical for any device count in deterministic mode
 *
 * Conventions: matrices are row-major doubles (DenseMatrix layout, dense.hpp:36-37), device
 * pointers, leading dimension `ld*` in elements, batch stride `stride*` in elements. Calls are
 * ordered on the context's stream; status-returning calls synchronise that stream once at the
 * end to read the device status (pass PF_FLAG_ASYNC to skip the check).
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes: 0 = success, otherwise parfrac::Errc ordinal + 1 (error.hpp:8-19). */
enum pf_err {
  PF_OK = 0,
  PF_ERR_DUPLICATE_SHIFT = 1,
  PF_ERR_LENGTH_MISMATCH = 2,
  PF_ERR_UNDER_DETERMINED = 3,
  PF_ERR_UNKNOWN_METHOD = 4,
  PF_ERR_INVALID_FUNCTION = 5,
  PF_ERR_NON_UNIT_CONSTANT = 6,
  PF_ERR_SINGULAR_SHIFT = 7,
  PF_ERR_ZERO_PIVOT = 8,
  PF_ERR_OUT_OF_CONVERGENCE_RADIUS = 9,
  PF_ERR_BAD_ARGUMENT = 10,
  PF_ERR_CUDA = 11 /* not a reference code: device/runtime failure */
};

enum pf_form { PF_FORM_PLAIN = 0, PF_FORM_RESIDUAL = 1 };

enum pf_flags {
  PF_FLAG_NONE = 0,
  PF_FLAG_ASYNC = 1,     /* do not synchronise to read device status */
  PF_FLAG_FORCE_PIVOT = 2, /* always run the genuine partial-pivoting LU (testing) */
  PF_FLAG_PER_SHIFT = 4,   /* no (c, -c) pair merging: one solve per shift, weighted terms added in
                              ascending shift order -- dense.cpp's rounding sequence; results are then
                              bit-identical to any shift partition summed in that order */
  PF_FLAG_REFERENCE_ORDER = 8 /* n <= 128: every operation in dense.cpp's order (per shift, unblocked
                              pivoting LU with 1.0/pivot, dot-product substitution, scale-then-add,
                              poly last, squaring in i-k-j order with the zero skip, no FMA): results
                              bit-identical to the reference. pf_eval_dense_batched,
                              pf_eval_scaled_batched, pf_expm_batched; BadArgument for n > 128 */
};

/* Failure detail; enough for the C++ wrapper to rebuild the reference message
 * "shift i: singular system: pivot magnitude X at column c (scale S)" (dense.cpp:117-119,220). */
typedef struct {
  int code;
  int batch_index;
  int shift_index; /* 1-based */
  int column;
  double pivot_magnitude;
  double scale;
} pf_status;

/* One partial-fraction method, doubles exactly as the host's to_double_nearest gives them
 * (rational.cpp:66-88). `weights`, `poly`, `constant` hold one row per weight set; set 0 is the
 * primary function (e.g. exp), set 1 an optional second function on the same shifts (phi1). */
typedef struct {
  int n_terms;            /* <= PF_MAX_TERMS */
  const double* shifts;   /* c_i, n_terms */
  int n_sets;             /* 1 or 2 */
  const double* weights;  /* b_i, n_sets * n_terms */
  int has_poly;           /* hybrid methods: d0, d1, d2 per set */
  const double* poly;     /* n_sets * 3, may be NULL when !has_poly */
  const double* constant; /* a_0 = d_0 + sum b_i per set (residual form constant term) */
  int form;               /* pf_form */
} pf_method;

/* cos/sin through exp(iB): conjugate shifts +-c merged into real solves of (I + c^2 B^2). */
typedef struct {
  int n_pairs; /* <= PF_MAX_TERMS */
  const double* c2;
  const double* cw; /* b_c + b_-c */
  const double* sw; /* c (b_c - b_-c) */
  double a0, a1;
} pf_pair_method;

#define PF_MAX_TERMS 16
#define PF_SMALL_N 128 /* fused single-CTA kernels handle n <= 128 */

typedef struct pf_context pf_context;

int pf_version(void);
const char* pf_error_string(int code);

int pf_context_create(int device, pf_context** out);
int pf_context_destroy(pf_context* ctx);
/* Use an external CUDA stream (cudaStream_t as void*); NULL = the legacy default stream. */
int pf_context_set_stream(pf_context* ctx, void* stream);
/* Number of kernels this context launched so far (bench evidence). */
int64_t pf_context_launch_count(pf_context* ctx);
/* Pipelined use (several PF_FLAG_ASYNC calls in flight): sticky != 0 resets the device error flag
 * once and keeps it across launches; pf_context_pending_error synchronises the context's stream and
 * returns 1 if any launch since the reset failed (re-run synchronously to get the pf_status). */
int pf_context_set_sticky_status(pf_context* ctx, int sticky);
int pf_context_pending_error(pf_context* ctx);
/* Diagnostics: when non-NULL, the fused small-n kernel adds per-phase SM cycles (thread 0 of each
 * CTA, clock64) into dev_counters[0..9]: norm, shift-matrix load, LU, diagonal inverses, RHS load,
 * solve+accumulate, E formation, squaring, output. NULL disables (the default). */
int pf_context_set_profile(pf_context* ctx, unsigned long long* dev_counters);

/* 1-norm (max column sum, rows summed in ascending order as dense.cpp:54-62) of each matrix. */
int pf_one_norm_batched(pf_context* ctx, int n, int batch, const double* dA, int64_t lda, int64_t strideA,
                        double* dNorm);

/* r(B) for every weight set (no scaling): outs[s] + b*strideOut for set s. */
int pf_eval_dense_batched(pf_context* ctx, const pf_method* m, int n, int batch, const double* dB, int64_t ldb,
                          int64_t strideB, double* const* dOuts, int64_t ldo, int64_t strideOut, int flags,
                          pf_status* status);

/* r(2^-j_b A_b) for every weight set, no squaring (j_b from dSquaringsIn, else from theta as below);
 * the building block of the shift-partitioned multi-GPU evaluation. */
int pf_eval_scaled_batched(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA,
                           int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut,
                           double* const* dOuts, int64_t ldo, int64_t strideOut, int flags, pf_status* status);

/* exp by scaling and squaring. j_b = dSquaringsIn[b] when non-NULL, else the smallest j >= 0 with
 * ldexp(||A_b||_1, -j) <= theta. B_b = 2^-j_b A_b, E = r(B_b) (weight set 0), E <- E^2 j_b times.
 * dSquaringsOut (may be NULL) receives j_b. */
int pf_expm_batched(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA,
                    int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut, double* dOut,
                    int64_t ldo, int64_t strideOut, int flags, pf_status* status);

/* exp and phi1 together: weight set 0 = exp, set 1 = phi1 on the same shifts;
 * j doublings of Phi <- 0.5 (E + I) Phi, E <- E E. */
int pf_expm_phi1_batched(pf_context* ctx, const pf_method* m, double theta, int n, int batch, const double* dA,
                         int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut, double* dE,
                         double* dPhi, int64_t ldo, int64_t strideOut, int flags, pf_status* status);

/* cos(A), sin(A): B = 2^-j A, Z_c = (I + c^2 B^2)^{-1} c^2 B^2, C = a0 I - sum cw Z, S = B (a1 I - sum sw Z),
 * then j steps of C <- C C - S S, S <- 2 (S C). */
int pf_cossin_batched(pf_context* ctx, const pf_pair_method* pm, double theta, int n, int batch, const double* dA,
                      int64_t lda, int64_t strideA, const int* dSquaringsIn, int* dSquaringsOut, double* dC,
                      double* dS, int64_t ldo, int64_t strideOut, int flags, pf_status* status);

/* Dense block action: B = A * (1.0/substeps) (elementwise, action.cpp:330-334), factor every
 * (I - c_i B) once, then `substeps` times V <- r(B) V (weight set 0). A n x n, V and Out n x k. */
int pf_action_block(pf_context* ctx, const pf_method* m, int n, int k, const double* dA, int64_t lda,
                    const double* dV, int64_t ldv, int substeps, double* dOut, int64_t ldo, int flags,
                    pf_status* status);

/* ---- f2: banded action (proj/core/src/action.cpp). A tridiagonal matrix is three device arrays
 * sub[d-1], diag[d], super[d-1] (TridiagMatrix, action.hpp:13-24); a block of k vectors is d x k
 * row-major, and every column is processed with exactly the reference's single-vector operation
 * sequence (the results are the reference's bits). ZeroPivot (|pivot| <= 1e-300) reports the row in
 * status->column and, for the action, the 1-based shift in status->shift_index. */

/* Out = A V (TridiagMatrix::matvec, action.cpp:35-44) */
int pf_tridiag_matvec_batched(pf_context* ctx, int d, int k, const double* dSub, const double* dDiag,
                              const double* dSuper, const double* dV, int64_t ldv, double* dOut, int64_t ldo);
/* X = A^-1 R for k right-hand sides (thomas_solve / TridiagFactor, action.cpp:100-141) */
int pf_thomas_solve_batched(pf_context* ctx, int d, int k, const double* dSub, const double* dDiag,
                            const double* dSuper, const double* dRhs, int64_t ldr, double* dX, int64_t ldx,
                            pf_status* status);
/* X = P^-1 R, P pentadiagonal (pentadiag_solve: banded LU without pivoting, action.cpp:170-202) */
int pf_pentadiag_solve_batched(pf_context* ctx, int d, int k, const double* dSub2, const double* dSub1,
                               const double* dDiag, const double* dSuper1, const double* dSuper2,
                               const double* dRhs, int64_t ldr, double* dX, int64_t ldx, pf_status* status);
/* substep_action (action.cpp:327-339) on every column of V: A scaled by 1/substeps, every shifted
 * system I - c_i A factored once (ActionOperator, :300-325), then substeps x (v <- action_eval(m, A,
 * v)) with assemble_action's ascending-shift sum and polynomial part (:224-284). Weight set 0. */
int pf_tridiag_action(pf_context* ctx, const pf_method* m, int d, int k, const double* dSub, const double* dDiag,
                      const double* dSuper, const double* dV, int64_t ldv, int substeps, double* dOut, int64_t ldo,
                      int flags, pf_status* status);

/* Device-resident ActionOperator (action.hpp:73-82, action.cpp:300-325) for a tridiagonal A: the bands
 * scaled by 1/substeps and every nonzero shift's system factored ONCE at creation (ZeroPivot
 * reported then, "shift i: zero pivot at row r"); each apply runs `substeps` steps v <- r(A/N) v on
 * k columns with method m's weights and form (its nonzero shifts must be the creation method's;
 * ActionOperator::apply's opts.form may differ per apply). Same bits as pf_tridiag_action. */
typedef struct pf_tridiag_op pf_tridiag_op;
int pf_tridiag_op_create(pf_context* ctx, const pf_method* m, int d, const double* dSub, const double* dDiag,
                         const double* dSuper, int substeps, pf_status* status, pf_tridiag_op** out);
int pf_tridiag_op_apply(pf_tridiag_op* op, const pf_method* m, const double* dV, int64_t ldv, int k, double* dOut,
                        int64_t ldo, pf_status* status);
int pf_tridiag_op_destroy(pf_tridiag_op* op);
/* Device-resident TridiagFactor (action.hpp:35-44): factored once (ZeroPivot at creation), solves
 * with the reference's operation sequence (same bits as thomas_solve). */
typedef struct pf_tridiag_factor pf_tridiag_factor;
int pf_tridiag_factor_create(pf_context* ctx, int d, const double* dSub, const double* dDiag, const double* dSuper,
                             pf_status* status, pf_tridiag_factor** out);
int pf_tridiag_factor_solve(pf_tridiag_factor* f, int k, const double* dRhs, int64_t ldr, double* dX, int64_t ldx);
int pf_tridiag_factor_destroy(pf_tridiag_factor* f);

/* DenseLu: in-place PA = LU (unit lower L below the diagonal, U on and above), LAPACK-style
 * 0-based swap sequence in dPiv (n ints per matrix). SingularShift when the best pivot
 * <= pivot_rel_tol * max(max|a|, 1e-300). */
int pf_lu_factor_batched(pf_context* ctx, int n, int batch, double* dA, int64_t lda, int64_t strideA, int* dPiv,
                         double pivot_rel_tol, int flags, pf_status* status);
/* X = U^{-1} L^{-1} P RHS for k right-hand-side columns (row-major n x k), in place in dRhs. */
int pf_lu_solve_batched(pf_context* ctx, int n, int k, int batch, const double* dLU, int64_t lda, int64_t strideLU,
                        const int* dPiv, double* dRhs, int64_t ldr, int64_t strideR);

/* (I - c B)^{-1} (dense.cpp:165-171). */
int pf_solve_shifted_batched(pf_context* ctx, int n, int batch, const double* dB, int64_t ldb, int64_t strideB,
                             double c, double* dOut, int64_t ldo, int64_t strideOut, int flags, pf_status* status);

/* C = alpha * A B + beta * C (+ gamma * I), batched, FP64 DMMA. C must not alias A or B. */
int pf_gemm_batched(pf_context* ctx, int m, int n, int k, int batch, double alpha, const double* dA, int64_t lda,
                    int64_t strideA, const double* dB, int64_t ldb, int64_t strideB, double beta, double* dC,
                    int64_t ldc, int64_t strideC, double gamma);

/* ---- building blocks for callers that drive the stages themselves (multi-GPU shift partition) ---- */

/* j_b = smallest j >= 0 with ldexp(||A_b||_1, -j) <= theta, into dJ (device). */
int pf_squarings_batched(pf_context* ctx, int n, int batch, const double* dA, int64_t lda, int64_t strideA,
                         double theta, int* dJ);
/* dOut = ((t_0 + t_1) + t_2) + ... elementwise, each add rounded: the ascending-shift reduction of
 * eval_dense (dense.cpp:245-246). dTerms is a HOST array of `count` device pointers. */
int pf_ordered_sum(pf_context* ctx, int count, const double* const* dTerms, int64_t n_elems, double* dOut);
/* Row block [r0, r0 + rows) of X + I (Y = X, plus 1 where r0 + i == j): E + I of a row-split phi1
 * doubling step, rounded as pf_phi1_doubling forms it. */
int pf_add_identity_rows(pf_context* ctx, int rows, int n, int r0, const double* dX, int64_t ldx, double* dY,
                         int64_t ldy);
/* dDiff = C - S and/or dSum = C + S over `count` doubles (the cos/sin step's (C - S)(C + S)). */
int pf_sum_diff(pf_context* ctx, int64_t count, const double* dC, const double* dS, double* dDiff, double* dSum);
/* E <- E^(2^j_b) per matrix (contiguous n x n batch). */
int pf_square_chain(pf_context* ctx, int n, int batch, const int* dJ, double* dE);
/* j_b steps of Phi <- 0.5 (E + I) Phi, E <- E E. */
int pf_phi1_doubling(pf_context* ctx, int n, int batch, const int* dJ, double* dE, double* dPhi);
/* j_b steps of C <- C C - S S, S <- 2 (S C). */
int pf_cossin_doubling(pf_context* ctx, int n, int batch, const int* dJ, double* dC, double* dS);

/* ActionOperator for a dense A (action.hpp:68-82): B = A * (1/substeps), the LU factors of the
 * owned shifts are computed once and reused by every apply. `owned` (host, n_terms ints, NULL = all)
 * selects the shifts this operator handles -- one subset per rank in the multi-GPU partition. */
typedef struct pf_action_op pf_action_op;
int pf_action_create(pf_context* ctx, const pf_method* m, int n, const double* dA, int64_t lda, int substeps,
                     const int* owned, int flags, pf_status* status, pf_action_op** out);
/* One substep restricted to the owned terms: dOut = sum_owned w_i x_i (+ a_0 V + d1 BV + d2 B^2 V when
 * include_poly). With dTerms != NULL also writes every owned weighted term (ascending shift index,
 * n x k each) followed by a_0 V and d1 BV + d2 B^2 V (when include_poly): an ordered sum of all
 * ranks' terms reproduces the single-operator result bit for bit. */
int pf_action_apply(pf_action_op* op, const double* dV, int64_t ldv, int k, double* dOut, int64_t ldo,
                    int include_poly, double* dTerms, pf_status* status);
int pf_action_term_count(pf_action_op* op);
int pf_action_destroy(pf_action_op* op);

/* ---- multi-GPU evaluation of one matrix ----
 * A multi-device context: one sub-context (own stream) per entry of device_ids plus an NCCL
 * communicator over them (ncclCommInitAll; libnccl.so.2 is loaded at run time). The returned
 * context is the root (device_ids[0]) and works with every other entry point on that device.
 * Repeated ids are allowed (several shares on one GPU, for tests): the exchange then uses peer
 * copies with the same partition and reduction order. */
int pf_context_create_multi(int n_devices, const int* device_ids, pf_context** out);
int pf_context_device_count(pf_context* ctx);
int pf_context_uses_nccl(pf_context* ctx);

enum pf_recurrence {
  PF_REC_NONE = 0,     /* r(A) for every weight set (eval_dense, no scaling) */
  PF_REC_EXP = 1,      /* exp: r(2^-j A) (set 0), then j squarings on the root */
  PF_REC_EXP_PHI1 = 2  /* exp and phi1 (sets 0 and 1), then j phi1 doublings on the root */
};
/* f(A) of ONE n x n matrix (device pointers on the root device) with the nonzero shifts partitioned
 * over the context's devices: (c, -c) pairs per device when there are at least as many pairs as
 * devices, else single shifts (R8 on 8 GPUs: one shift each); zero shifts and a_0 / poly on the root.
 * Every device evaluates its share concurrently; ONE exchange brings the result to the root before
 * the recurrence: deterministic = 0 -> ncclReduce(sum) of per-device partial sums (agrees to
 * rounding for any device count); deterministic = 1 -> every weighted term is sent to the root
 * (ncclSend/ncclRecv, root only), summed in ascending shift index and completed with the
 * polynomial part exactly as eval_dense does (dense.cpp:244-250): bit-identical for any device
 * count. j_out (host, may be NULL) receives the squaring count. SingularShift reports the global
 * 1-based shift index. */
int pf_eval_multi_gpu(pf_context* ctx, const pf_method* m, double theta, int recurrence, int n, const double* dA,
                      int64_t lda, double* dOut0, double* dOut1, int64_t ldo, int deterministic, int flags,
                      int* j_out, pf_status* status);

/* Device memory helpers for hosts without their own CUDA runtime (the C++ host layer): allocation
 * on the context's device, synchronous copies ordered on the context's stream. */
int pf_device_alloc(pf_context* ctx, size_t bytes, void** out);
int pf_device_free(pf_context* ctx, void* p);
int pf_copy_to_device(pf_context* ctx, void* dst, const void* src, size_t bytes);
int pf_copy_to_host(pf_context* ctx, void* dst, const void* src, size_t bytes);

/* Measured FP64 DMMA throughput of `device` in TFLOP/s (the FP64 roofline denominator). */
double pf_probe_dmma_tflops(int device);

#ifdef __cplusplus
}
#endif
#endif /* PF_B200_H */
