/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the parfrac dense hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. The product path (paper_2210_03714_b200) never links it.
 *
 * Plain-C restatement of the reference evaluator, same loop orders, pivot rule and
 * fixed reduction order:
 *   DenseMatrix::mul / axpy / scale / add_scaled_identity / one_norm / max_abs
 *       proj/core/src/dense.cpp:17-68
 *   DenseLu (partial pivoting, strict '>' so the first max wins, full-row swaps,
 *       reciprocal multipliers, SingularShift below 1e-14*max|a|)   dense.cpp:102-133
 *   DenseLu::solve / solve_matrix                                    dense.cpp:135-163
 *   solve_shifted                                                    dense.cpp:165-171
 *   eval_dense (plain / residual, ascending accumulation, poly part) dense.cpp:176-252
 *   parallel_for_index (atomic claim, per-index slots)               worker_pool.hpp:16-44
 *   SplitMix64 / NormalSampler                                       rng.hpp:10-26, rng.cpp:7-19
 *   make_dense_matrix randn / cauchy / trid121                       cli.cpp:35-56, action.cpp:27-33
 * and the compositions SURVEY.md §8(a) a10-a13 defines on top of those primitives:
 *   scaling and squaring (pattern expm_oracle dense.cpp:460-476), exp+phi1 with
 *   phi1 doubling, cos/sin pair with C^2 - S^2 / 2SC, dense block action with
 *   factor-once substepping (assemble_action / ActionOperator / substep_action,
 *   action.cpp:224-339).
 *
 * Parity pinning: PINNED against the reference itself. oracle/Makefile compiles
 * /root/reference/proj/core/src/(*).cpp unmodified (GMP/gmpxx shims in oracle/shim/) into
 * oracle/_ref/libparfrac_ref.so; the reference's own doctest suites and acceptance checklist pass
 * on that build, and tests/test_ref_pin.py requires this restatement to equal it bit for bit
 * (LU factors and pivots, solve_shifted, mul, eval_dense for every catalog method and both forms,
 * cfg1/cfg2 expm, exp+phi1, dense block action, the banded solvers and actions, generators).
 * tests/golden/ holds reference outputs (make_golden.py) that this library must reproduce.
 */
#ifndef PF_ORACLE_H
#define PF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int code; /* 0 = ok, else Errc ordinal + 1 */
  int batch_index;
  int shift_index; /* 1-based, as in the reference's "shift i:" prefix */
  int column;
  double pivot_magnitude;
  double scale;
} pfo_status;

typedef struct {
  int n_terms;
  const double* shifts;  /* n_terms */
  int n_sets;
  const double* weights; /* n_sets * n_terms */
  int has_poly;
  const double* poly;     /* n_sets * 3: d0, d1, d2 */
  const double* constant; /* n_sets: a_0 = d_0 + sum b (used by the residual form) */
  int form;               /* 0 plain, 1 residual */
} pfo_method;

typedef struct {
  int n_pairs;
  const double* c2; /* n_pairs, c^2 of each merged +-c pair, ascending */
  const double* cw; /* cos weights b_c + b_-c */
  const double* sw; /* sin weights c (b_c - b_-c) */
  double a0, a1;
} pfo_pair_method;

/* generators (not timed) */
uint64_t pfo_splitmix_next(uint64_t* state);
void pfo_uniform_fill(uint64_t seed, int64_t count, double* out);
void pfo_randn_fill(uint64_t seed, int64_t count, double* out);

/* DenseMatrix primitives, row-major n x n */
void pfo_mul(int n, const double* a, const double* b, double* c);
void pfo_mul_rect(int n, int k, const double* a, const double* b, double* c); /* (n x n)(n x k) */
void pfo_mul_rows(int rows, int n, const double* a, const double* b, double* c); /* (rows x n)(n x n) */
void pfo_mul_mt(int n, const double* a, const double* b, double* c, int threads); /* rows split over threads */
double pfo_one_norm(int n, const double* a);
double pfo_max_abs(int n, const double* a);
int pfo_squarings(double norm1, double theta);
int pfo_substeps(double norm1, double theta);

/* DenseLu */
int pfo_lu(int n, double* lu, int* piv, double pivot_rel_tol, pfo_status* st);
void pfo_lu_solve(int n, const double* lu, const int* piv, double* x);
void pfo_lu_solve_matrix(int n, int k, const double* lu, const int* piv, const double* rhs, double* out);
int pfo_solve_shifted(int n, const double* b, double c, double* out, pfo_status* st);

/* eval_dense for every weight set of m: outs = n_sets * n * n */
int pfo_eval_dense(int n, const double* b, const pfo_method* m, int workers, double* outs, pfo_status* st);

/* a10: j = squarings(||A||_1, theta) (or j_fixed >= 0), B = 2^-j A, E = r(B), E <- E^2 j times */
int pfo_expm(int n, const double* a, const pfo_method* m, double theta, int j_fixed, int workers,
             double* out, int* j_out, pfo_status* st);
/* batched: parallel over the batch with workers = 1 inside (cli.cpp:314,228) */
int pfo_expm_batched(int n, int batch, const double* a, const pfo_method* m, double theta, int threads,
                     double* out, int* j_out, pfo_status* st);

/* a11 + a12: set 0 = exp weights, set 1 = phi1 weights on the same shifts.
 * Phi <- 0.5 (E + I) Phi, then E <- E E, j times. */
int pfo_expm_phi1(int n, const double* a, const pfo_method* m, double theta, int j_fixed, int workers,
                  double* out_e, double* out_phi, int* j_out, pfo_status* st);

/* a12: cos/sin pair. C <- C C - S S, S <- 2 (S C), j times. */
int pfo_cossin(int n, const double* a, const pfo_pair_method* pm, double theta, int j_fixed, int workers,
               double* out_c, double* out_s, int* j_out, pfo_status* st);
int pfo_cossin_batched(int n, int batch, const double* a, const pfo_pair_method* pm, double theta,
                       int threads, double* out_c, double* out_s, int* j_out, pfo_status* st);

/* a13: dense block action, V is n x k row-major. B = A * (1.0/substeps); LU of every
 * (I - c_i B) factored once; substeps x (V <- r(B) V). */
int pfo_action(int n, int k, const double* a, const double* v, const pfo_method* m, int substeps,
               int workers, double* out, pfo_status* st);

/* f2: banded action (pf_oracle_band.c, restating proj/core/src/action.cpp). Tridiagonal matrices
 * are (sub[d-1], diag[d], super[d-1]); V / out are d x k row-major (k independent columns). */
void pfo_tridiag_matvec(int d, const double* sub, const double* diag, const double* super, const double* v,
                        double* out);
double pfo_tridiag_one_norm(int d, const double* sub, const double* diag, const double* super);
int pfo_thomas_solve(int d, const double* sub, const double* diag, const double* super, const double* rhs,
                     double* x, int* row);
int pfo_tridiag_factor(int d, const double* sub, const double* diag, const double* super, double* mult,
                       double* fdiag, int* row);
void pfo_tridiag_factor_solve(int d, const double* mult, const double* fdiag, const double* super, const double* rhs,
                              double* x);
int pfo_pentadiag_solve(int d, const double* sub2, const double* sub1, const double* diag, const double* super1,
                        const double* super2, const double* rhs, double* x, int* row);
int pfo_tridiag_action(int d, int k, const double* sub, const double* diag, const double* super, const double* v,
                       const pfo_method* m, int substeps, double* out, pfo_status* st);

#ifdef __cplusplus
}
#endif
#endif
