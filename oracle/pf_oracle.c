/* TEST INFRASTRUCTURE ONLY -- see pf_oracle.h for scope and the reference citations.
 * Compiled with the reference's flags (-O3 -DNDEBUG, no -march; proj/CMakeLists.txt:3-10)
 * plus -ffp-contract=off so no FMA contraction can change a rounding. */
#include "pf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ERRC_SINGULAR_SHIFT 6
#define ERRC_BAD_ARGUMENT 9
#define CODE(e) ((e) + 1)

/* ---------------------------------------------------------------- generators (rng.hpp) */

uint64_t pfo_splitmix_next(uint64_t* state) { /* rng.hpp:14-19 */
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static double uniform01(uint64_t* s) { return (double)(pfo_splitmix_next(s) >> 11) * 0x1.0p-53; }

void pfo_uniform_fill(uint64_t seed, int64_t count, double* out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < count; ++i) out[i] = uniform01(&s);
}

void pfo_randn_fill(uint64_t seed, int64_t count, double* out) { /* rng.cpp:7-19 */
  uint64_t s = seed;
  int have_spare = 0;
  double spare = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (have_spare) {
      have_spare = 0;
      out[i] = spare;
      continue;
    }
    double u1 = 1.0 - uniform01(&s);
    double u2 = uniform01(&s);
    double r = sqrt(-2.0 * log(u1));
    double angle = 2.0 * 3.14159265358979323846 * u2;
    spare = r * sin(angle);
    have_spare = 1;
    out[i] = r * cos(angle);
  }
}

/* ---------------------------------------------------------------- worker pool */

typedef void (*pfo_task)(int i, void* ctx);
typedef struct {
  int n;
  volatile int next;
  pfo_task fn;
  void* ctx;
} pool_t;

static void* pool_body(void* p) {
  pool_t* pool = (pool_t*)p;
  for (;;) {
    int i = __sync_fetch_and_add(&pool->next, 1);
    if (i >= pool->n) return NULL;
    pool->fn(i, pool->ctx);
  }
}

/* worker_pool.hpp:16-44: each index once, per-index result slots, caller reduces in order */
static void parallel_for_index(int n, int workers, pfo_task fn, void* ctx) {
  if (n <= 0) return;
  int nthreads = workers < n ? workers : n;
  if (nthreads <= 1) {
    for (int i = 0; i < n; ++i) fn(i, ctx);
    return;
  }
  pool_t pool = {n, 0, fn, ctx};
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, pool_body, &pool);
  pool_body(&pool);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
}

/* ---------------------------------------------------------------- DenseMatrix (dense.cpp:17-68) */

/* Products in dense.cpp:17-29's i-k-j order with the a_ik == 0 skip. Every output element
 * receives its products in ascending k exactly as in the reference loop; the loops are only
 * tiled (row blocks of MB, column blocks of JB) so B streams through cache once per row block
 * instead of once per row -- the same operations, in the same per-element order, bit for bit. */
#define PFO_MB 16
#define PFO_JB 256
static void mul_block_rows(int rows, int d, int kc, const double* a, const double* o, double* out) {
  memset(out, 0, sizeof(double) * (size_t)rows * (size_t)kc);
  for (int j0 = 0; j0 < kc; j0 += PFO_JB) {
    const int j1 = j0 + PFO_JB < kc ? j0 + PFO_JB : kc;
    for (int i0 = 0; i0 < rows; i0 += PFO_MB) {
      const int i1 = i0 + PFO_MB < rows ? i0 + PFO_MB : rows;
      for (int k = 0; k < d; ++k) {
        const double* orow = &o[(size_t)k * kc];
        for (int i = i0; i < i1; ++i) {
          const double aik = a[(size_t)i * d + k];
          if (aik == 0.0) continue;
          double* orow_out = &out[(size_t)i * kc];
          for (int j = j0; j < j1; ++j) orow_out[j] += aik * orow[j];
        }
      }
    }
  }
}

void pfo_mul(int d, const double* a, const double* o, double* out) { mul_block_rows(d, d, d, a, o, out); }

/* rows of a product: out (rows x d) = a_rows (rows x d) * o (d x d), pfo_mul's i-k-j order and
 * zero skip per row (row i of pfo_mul depends on row i of a only) -- the f1 row-split doubling */
void pfo_mul_rows(int rows, int d, const double* a, const double* o, double* out) {
  mul_block_rows(rows, d, d, a, o, out);
}

void pfo_mul_rect(int d, int kc, const double* a, const double* o, double* out) {
  mul_block_rows(d, d, kc, a, o, out);
}

double pfo_one_norm(int d, const double* a) {
  double best = 0;
  for (int j = 0; j < d; ++j) {
    double col = 0;
    for (int i = 0; i < d; ++i) col += fabs(a[(size_t)i * d + j]);
    best = best > col ? best : col; /* std::max(best, col) */
  }
  return best;
}

double pfo_max_abs(int d, const double* a) {
  double best = 0;
  for (size_t i = 0; i < (size_t)d * d; ++i) {
    double v = fabs(a[i]);
    best = best > v ? best : v;
  }
  return best;
}

static void axpy(size_t cnt, double* acc, double s, const double* x) {
  for (size_t i = 0; i < cnt; ++i) acc[i] += s * x[i];
}
static void scale(size_t cnt, double* a, double s) {
  for (size_t i = 0; i < cnt; ++i) a[i] *= s;
}
static void add_scaled_identity(int d, double* a, double s) {
  for (int i = 0; i < d; ++i) a[(size_t)i * d + i] += s;
}

/* smallest j >= 0 with ldexp(norm, -j) <= theta: exact, no libm rounding */
int pfo_squarings(double norm1, double theta) {
  int j = 0;
  while (ldexp(norm1, -j) > theta && j < 2000) ++j;
  return j;
}

int pfo_substeps(double norm1, double theta) { /* action.cpp:398 */
  if (norm1 <= theta) return 1;
  return (int)ceil(norm1 / theta);
}

/* ---------------------------------------------------------------- DenseLu (dense.cpp:102-163) */

/* DenseLu (dense.cpp:102-133). The reference applies, to every element (r, j), the updates
 * a_rj -= f_r,col * u_col,j for col = 0, 1, ... in ascending order, each with the final
 * multiplier f (skipped when f == 0) and the final U row entry, and swaps whole rows at each
 * pivot. Here the same updates are applied panel by panel (width PFO_NB): within a panel
 * right-looking on the panel's columns (pivot search, full-row swaps, multipliers exactly as in the
 * reference), then the U rows of the panel and the trailing block receive the panel's updates in
 * ascending col. Per element the operation sequence is unchanged, so factors and pivots are
 * bit-identical to the unblocked loop (tests/test_ref_pin.py); the trailing matrix streams through
 * cache once per panel instead of once per column. */
#define PFO_NB 32
int pfo_lu(int d, double* lu, int* piv, double pivot_rel_tol, pfo_status* st) {
  double ma = pfo_max_abs(d, lu);
  const double sc = ma > 1e-300 ? ma : 1e-300;
  const double tol = pivot_rel_tol * sc;
  for (int c0 = 0; c0 < d; c0 += PFO_NB) {
    const int c1 = c0 + PFO_NB < d ? c0 + PFO_NB : d;
    for (int col = c0; col < c1; ++col) {
      int p = col;
      double best = fabs(lu[(size_t)col * d + col]);
      for (int r = col + 1; r < d; ++r) {
        double v = fabs(lu[(size_t)r * d + col]);
        if (v > best) {
          best = v;
          p = r;
        }
      }
      if (best <= tol) {
        if (st) {
          st->code = CODE(ERRC_SINGULAR_SHIFT);
          st->column = col;
          st->pivot_magnitude = best;
          st->scale = sc;
        }
        return CODE(ERRC_SINGULAR_SHIFT);
      }
      if (p != col)
        for (int j = 0; j < d; ++j) {
          double t = lu[(size_t)p * d + j];
          lu[(size_t)p * d + j] = lu[(size_t)col * d + j];
          lu[(size_t)col * d + j] = t;
        }
      piv[col] = p;
      const double inv_piv = 1.0 / lu[(size_t)col * d + col];
      for (int r = col + 1; r < d; ++r) {
        double f = lu[(size_t)r * d + col] * inv_piv;
        lu[(size_t)r * d + col] = f;
        if (f == 0.0) continue;
        for (int j = col + 1; j < c1; ++j) lu[(size_t)r * d + j] -= f * lu[(size_t)col * d + j];
      }
    }
    if (c1 == d) break;
    /* U rows of the panel, trailing columns: row t gets cols c0..t-1 in order (rows < t final) */
    for (int t = c0 + 1; t < c1; ++t)
      for (int s = c0; s < t; ++s) {
        const double f = lu[(size_t)t * d + s];
        if (f == 0.0) continue;
        for (int j = c1; j < d; ++j) lu[(size_t)t * d + j] -= f * lu[(size_t)s * d + j];
      }
    /* trailing block: every row gets the panel's cols c0..c1-1 in order */
    for (int j0 = c1; j0 < d; j0 += PFO_JB) {
      const int j1 = j0 + PFO_JB < d ? j0 + PFO_JB : d;
      for (int r = c1; r < d; ++r)
        for (int s = c0; s < c1; ++s) {
          const double f = lu[(size_t)r * d + s];
          if (f == 0.0) continue;
          for (int j = j0; j < j1; ++j) lu[(size_t)r * d + j] -= f * lu[(size_t)s * d + j];
        }
    }
  }
  return 0;
}

void pfo_lu_solve(int d, const double* lu, const int* piv, double* x) {
  for (int i = 0; i < d; ++i)
    if (piv[i] != i) {
      double t = x[i];
      x[i] = x[piv[i]];
      x[piv[i]] = t;
    }
  for (int i = 1; i < d; ++i) {
    double acc = x[i];
    for (int j = 0; j < i; ++j) acc -= lu[(size_t)i * d + j] * x[j];
    x[i] = acc;
  }
  for (int i = d - 1; i >= 0; --i) {
    double acc = x[i];
    for (int j = i + 1; j < d; ++j) acc -= lu[(size_t)i * d + j] * x[j];
    x[i] = acc / lu[(size_t)i * d + i];
  }
}

/* solve_matrix (dense.cpp:153-163): every RHS column runs DenseLu::solve (swaps, then the
 * dot-product forward and back substitutions with ascending j). PFO_CB columns are carried side by
 * side -- per column the same operations in the same order -- so each row of the factors is read
 * once per column block instead of once per column. */
#define PFO_CB 16
static void solve_cols(int d, int kc, const double* lu, const int* piv, const double* rhs, double* out, int cb,
                       int ce) {
  double* x = (double*)malloc(sizeof(double) * (size_t)d * PFO_CB);
  double acc[PFO_CB];
  for (int c0 = cb; c0 < ce; c0 += PFO_CB) {
    const int w = c0 + PFO_CB < ce ? PFO_CB : ce - c0;
    for (int i = 0; i < d; ++i)
      for (int c = 0; c < w; ++c) x[(size_t)i * PFO_CB + c] = rhs[(size_t)i * kc + c0 + c];
    for (int i = 0; i < d; ++i)
      if (piv[i] != i)
        for (int c = 0; c < w; ++c) {
          double t = x[(size_t)i * PFO_CB + c];
          x[(size_t)i * PFO_CB + c] = x[(size_t)piv[i] * PFO_CB + c];
          x[(size_t)piv[i] * PFO_CB + c] = t;
        }
    for (int i = 1; i < d; ++i) {
      const double* row = &lu[(size_t)i * d];
      for (int c = 0; c < w; ++c) acc[c] = x[(size_t)i * PFO_CB + c];
      for (int j = 0; j < i; ++j) {
        const double l = row[j];
        const double* xj = &x[(size_t)j * PFO_CB];
        for (int c = 0; c < w; ++c) acc[c] -= l * xj[c];
      }
      for (int c = 0; c < w; ++c) x[(size_t)i * PFO_CB + c] = acc[c];
    }
    for (int i = d - 1; i >= 0; --i) {
      const double* row = &lu[(size_t)i * d];
      for (int c = 0; c < w; ++c) acc[c] = x[(size_t)i * PFO_CB + c];
      for (int j = i + 1; j < d; ++j) {
        const double u = row[j];
        const double* xj = &x[(size_t)j * PFO_CB];
        for (int c = 0; c < w; ++c) acc[c] -= u * xj[c];
      }
      const double piv_ii = row[i];
      for (int c = 0; c < w; ++c) x[(size_t)i * PFO_CB + c] = acc[c] / piv_ii;
    }
    for (int i = 0; i < d; ++i)
      for (int c = 0; c < w; ++c) out[(size_t)i * kc + c0 + c] = x[(size_t)i * PFO_CB + c];
  }
  free(x);
}

void pfo_lu_solve_matrix(int d, int kc, const double* lu, const int* piv, const double* rhs, double* out) {
  solve_cols(d, kc, lu, piv, rhs, out, 0, kc);
}

/* Threaded variants for the big checks (cfg3/cfg4 at full size): columns of a solve and rows of a
 * product are independent, so splitting them over threads changes no element's operations. */
typedef struct {
  int d, kc, chunk;
  const double *lu, *rhs, *a, *o;
  const int* piv;
  double* out;
} mt_ctx;

static void solve_chunk(int t, void* p) {
  mt_ctx* c = (mt_ctx*)p;
  const int cb = t * c->chunk, ce = cb + c->chunk < c->kc ? cb + c->chunk : c->kc;
  solve_cols(c->d, c->kc, c->lu, c->piv, c->rhs, c->out, cb, ce);
}

static void solve_mt(int d, int kc, const double* lu, const int* piv, const double* rhs, double* out, int threads) {
  if (threads <= 1 || kc <= PFO_CB) {
    solve_cols(d, kc, lu, piv, rhs, out, 0, kc);
    return;
  }
  int chunk = (kc + threads - 1) / threads;
  chunk = (chunk + PFO_CB - 1) / PFO_CB * PFO_CB;
  mt_ctx c = {d, kc, chunk, lu, rhs, NULL, NULL, piv, out};
  parallel_for_index((kc + chunk - 1) / chunk, threads, solve_chunk, &c);
}

static void mul_chunk(int t, void* p) {
  mt_ctx* c = (mt_ctx*)p;
  const int r0 = t * c->chunk, r1 = r0 + c->chunk < c->d ? r0 + c->chunk : c->d;
  mul_block_rows(r1 - r0, c->d, c->kc, c->a + (size_t)r0 * c->d, c->o, c->out + (size_t)r0 * c->kc);
}

/* (d x d)(d x kc) split by rows over threads */
static void mul_mt(int d, int kc, const double* a, const double* o, double* out, int threads) {
  if (threads <= 1 || d < 2 * PFO_MB) {
    mul_block_rows(d, d, kc, a, o, out);
    return;
  }
  int chunk = (d + threads - 1) / threads;
  chunk = (chunk + PFO_MB - 1) / PFO_MB * PFO_MB;
  mt_ctx c = {d, kc, chunk, NULL, NULL, a, o, NULL, out};
  parallel_for_index((d + chunk - 1) / chunk, threads, mul_chunk, &c);
}

void pfo_mul_mt(int d, const double* a, const double* o, double* out, int threads) {
  mul_mt(d, d, a, o, out, threads);
}

int pfo_solve_shifted(int d, const double* b, double c, double* out, pfo_status* st) {
  size_t nn = (size_t)d * d;
  double* m = (double*)malloc(sizeof(double) * nn);
  int* piv = (int*)malloc(sizeof(int) * (size_t)(d > 0 ? d : 1));
  memcpy(m, b, sizeof(double) * nn);
  scale(nn, m, -c);
  add_scaled_identity(d, m, 1.0);
  int rc = pfo_lu(d, m, piv, 1e-14, st);
  if (!rc) {
    double* id = (double*)calloc(nn, sizeof(double));
    add_scaled_identity(d, id, 1.0);
    pfo_lu_solve_matrix(d, d, m, piv, id, out);
    free(id);
  }
  free(m);
  free(piv);
  return rc;
}

/* ---------------------------------------------------------------- eval_dense (dense.cpp:176-252) */

typedef struct {
  int d;
  const double* b;
  const pfo_method* m;
  double** x;        /* per shift: solved X_i (unweighted), NULL for zero shifts */
  pfo_status* stats; /* per shift */
  int inner;         /* threads per shift's solve (workers beyond one per shift) */
} eval_ctx;

static void eval_shift(int i, void* p) {
  eval_ctx* c = (eval_ctx*)p;
  const int d = c->d;
  const size_t nn = (size_t)d * d;
  const double sh = c->m->shifts[i];
  c->x[i] = NULL;
  if (sh == 0.0) return;
  double* mm = (double*)malloc(sizeof(double) * nn);
  int* piv = (int*)malloc(sizeof(int) * (size_t)d);
  memcpy(mm, c->b, sizeof(double) * nn);
  scale(nn, mm, -sh);
  add_scaled_identity(d, mm, 1.0);
  double* rhs = (double*)calloc(nn, sizeof(double));
  if (c->m->form == 0) {
    add_scaled_identity(d, rhs, 1.0);
  } else {
    memcpy(rhs, c->b, sizeof(double) * nn);
    scale(nn, rhs, sh);
  }
  int rc = pfo_lu(d, mm, piv, 1e-14, &c->stats[i]);
  if (rc) {
    c->stats[i].code = rc;
    c->stats[i].shift_index = i + 1;
  } else {
    double* x = (double*)malloc(sizeof(double) * nn);
    solve_mt(d, d, mm, piv, rhs, x, c->inner);
    c->x[i] = x;
  }
  free(rhs);
  free(mm);
  free(piv);
}

int pfo_eval_dense(int d, const double* b, const pfo_method* m, int workers, double* outs, pfo_status* st) {
  if (workers < 1) {
    if (st) st->code = CODE(ERRC_BAD_ARGUMENT);
    return CODE(ERRC_BAD_ARGUMENT);
  }
  const size_t nn = (size_t)d * d;
  const int n = m->n_terms;
  eval_ctx c;
  c.d = d;
  c.b = b;
  c.m = m;
  c.x = (double**)calloc((size_t)(n > 0 ? n : 1), sizeof(double*));
  c.stats = (pfo_status*)calloc((size_t)(n > 0 ? n : 1), sizeof(pfo_status));
  int nz = 0;
  for (int i = 0; i < n; ++i) nz += m->shifts[i] != 0.0;
  c.inner = nz > 0 && workers > nz ? workers / nz : 1;
  parallel_for_index(n, workers, eval_shift, &c);
  int rc = 0;
  for (int i = 0; i < n; ++i)
    if (c.stats[i].code) {
      if (st) *st = c.stats[i];
      rc = c.stats[i].code;
      break;
    }
  if (!rc) {
    double* t = (double*)malloc(sizeof(double) * nn);
    double* poly = (double*)malloc(sizeof(double) * nn);
    double* b2 = NULL;
    for (int s = 0; s < m->n_sets; ++s) {
      double* acc = outs + (size_t)s * nn;
      memset(acc, 0, sizeof(double) * nn);
      for (int i = 0; i < n; ++i) {
        const double w = m->weights[(size_t)s * n + i];
        if (c.x[i] == NULL) {
          if (m->form == 0) { /* plain zero shift: t = w I */
            memset(t, 0, sizeof(double) * nn);
            add_scaled_identity(d, t, w);
            axpy(nn, acc, 1.0, t);
          }
          continue; /* residual: zero term */
        }
        memcpy(t, c.x[i], sizeof(double) * nn);
        scale(nn, t, w);
        axpy(nn, acc, 1.0, t);
      }
      const double constant = m->form == 1 ? m->constant[s] : (m->has_poly ? m->poly[3 * s] : 0.0);
      if (m->form == 1 || m->has_poly) {
        memset(poly, 0, sizeof(double) * nn);
        add_scaled_identity(d, poly, constant);
        if (m->has_poly) {
          const double d1 = m->poly[3 * s + 1], d2 = m->poly[3 * s + 2];
          axpy(nn, poly, d1, b);
          if (d2 != 0.0) {
            if (!b2) {
              b2 = (double*)malloc(sizeof(double) * nn);
              mul_mt(d, d, b, b, b2, workers);
            }
            axpy(nn, poly, d2, b2);
          }
        }
        axpy(nn, acc, 1.0, poly);
      }
    }
    free(t);
    free(poly);
    free(b2);
  }
  for (int i = 0; i < n; ++i) free(c.x[i]);
  free(c.x);
  free(c.stats);
  return rc;
}

/* ---------------------------------------------------------------- a10: scaling and squaring */

static int pick_j(int d, const double* a, double theta, int j_fixed) {
  return j_fixed >= 0 ? j_fixed : pfo_squarings(pfo_one_norm(d, a), theta);
}

static void scaled_copy(size_t nn, const double* a, int j, double* b) {
  for (size_t i = 0; i < nn; ++i) b[i] = ldexp(a[i], -j);
}

int pfo_expm(int d, const double* a, const pfo_method* m, double theta, int j_fixed, int workers,
             double* out, int* j_out, pfo_status* st) {
  const size_t nn = (size_t)d * d;
  const int j = pick_j(d, a, theta, j_fixed);
  if (j_out) *j_out = j;
  double* b = (double*)malloc(sizeof(double) * nn);
  scaled_copy(nn, a, j, b);
  pfo_method m1 = *m;
  m1.n_sets = 1;
  int rc = pfo_eval_dense(d, b, &m1, workers, out, st);
  if (!rc) {
    double* t = (double*)malloc(sizeof(double) * nn);
    for (int s = 0; s < j; ++s) {
      mul_mt(d, d, out, out, t, workers);
      memcpy(out, t, sizeof(double) * nn);
    }
    free(t);
  }
  free(b);
  return rc;
}

typedef struct {
  int d;
  const double* a;
  const pfo_method* m;
  double theta;
  double* out;
  int* j_out;
  pfo_status* stats;
} batch_ctx;

static void expm_one(int i, void* p) {
  batch_ctx* c = (batch_ctx*)p;
  const size_t nn = (size_t)c->d * c->d;
  int j = 0;
  pfo_expm(c->d, c->a + (size_t)i * nn, c->m, c->theta, -1, 1, c->out + (size_t)i * nn, &j, &c->stats[i]);
  if (c->j_out) c->j_out[i] = j;
}

static int first_error(int batch, pfo_status* stats, pfo_status* st) {
  for (int i = 0; i < batch; ++i)
    if (stats[i].code) {
      if (st) {
        *st = stats[i];
        st->batch_index = i;
      }
      return stats[i].code;
    }
  return 0;
}

int pfo_expm_batched(int d, int batch, const double* a, const pfo_method* m, double theta, int threads,
                     double* out, int* j_out, pfo_status* st) {
  batch_ctx c = {d, a, m, theta, out, j_out, (pfo_status*)calloc((size_t)(batch > 0 ? batch : 1), sizeof(pfo_status))};
  parallel_for_index(batch, threads, expm_one, &c);
  int rc = first_error(batch, c.stats, st);
  free(c.stats);
  return rc;
}

/* ---------------------------------------------------------------- a11/a12: exp + phi1 */

int pfo_expm_phi1(int d, const double* a, const pfo_method* m, double theta, int j_fixed, int workers,
                  double* out_e, double* out_phi, int* j_out, pfo_status* st) {
  const size_t nn = (size_t)d * d;
  if (m->n_sets < 2) {
    if (st) st->code = CODE(ERRC_BAD_ARGUMENT);
    return CODE(ERRC_BAD_ARGUMENT);
  }
  const int j = pick_j(d, a, theta, j_fixed);
  if (j_out) *j_out = j;
  double* b = (double*)malloc(sizeof(double) * nn);
  double* both = (double*)malloc(sizeof(double) * nn * 2);
  scaled_copy(nn, a, j, b);
  pfo_method m2 = *m;
  m2.n_sets = 2;
  int rc = pfo_eval_dense(d, b, &m2, workers, both, st);
  if (!rc) {
    memcpy(out_e, both, sizeof(double) * nn);
    memcpy(out_phi, both + nn, sizeof(double) * nn);
    double* t = (double*)malloc(sizeof(double) * nn);
    double* u = (double*)malloc(sizeof(double) * nn);
    for (int s = 0; s < j; ++s) {
      memcpy(t, out_e, sizeof(double) * nn); /* T = E + I */
      add_scaled_identity(d, t, 1.0);
      mul_mt(d, d, t, out_phi, u, workers); /* Phi = 0.5 (T Phi) */
      scale(nn, u, 0.5);
      memcpy(out_phi, u, sizeof(double) * nn);
      mul_mt(d, d, out_e, out_e, t, workers); /* E = E E */
      memcpy(out_e, t, sizeof(double) * nn);
    }
    free(t);
    free(u);
  }
  free(b);
  free(both);
  return rc;
}

/* ---------------------------------------------------------------- a12: cos / sin pair */

typedef struct {
  int d;
  const double* b2;
  const pfo_pair_method* pm;
  double** z;
  pfo_status* stats;
} pair_ctx;

static void pair_shift(int k, void* p) {
  pair_ctx* c = (pair_ctx*)p;
  const int d = c->d;
  const size_t nn = (size_t)d * d;
  const double c2 = c->pm->c2[k];
  double* mm = (double*)malloc(sizeof(double) * nn);
  double* rhs = (double*)malloc(sizeof(double) * nn);
  int* piv = (int*)malloc(sizeof(int) * (size_t)d);
  memcpy(mm, c->b2, sizeof(double) * nn); /* M = I + c^2 B^2 */
  scale(nn, mm, c2);
  add_scaled_identity(d, mm, 1.0);
  memcpy(rhs, c->b2, sizeof(double) * nn); /* RHS = c^2 B^2 */
  scale(nn, rhs, c2);
  c->z[k] = NULL;
  int rc = pfo_lu(d, mm, piv, 1e-14, &c->stats[k]);
  if (rc) {
    c->stats[k].code = rc;
    c->stats[k].shift_index = k + 1;
  } else {
    c->z[k] = (double*)malloc(sizeof(double) * nn);
    pfo_lu_solve_matrix(d, d, mm, piv, rhs, c->z[k]);
  }
  free(mm);
  free(rhs);
  free(piv);
}

int pfo_cossin(int d, const double* a, const pfo_pair_method* pm, double theta, int j_fixed, int workers,
               double* out_c, double* out_s, int* j_out, pfo_status* st) {
  const size_t nn = (size_t)d * d;
  const int j = pick_j(d, a, theta, j_fixed);
  if (j_out) *j_out = j;
  double* b = (double*)malloc(sizeof(double) * nn);
  double* b2 = (double*)malloc(sizeof(double) * nn);
  scaled_copy(nn, a, j, b);
  mul_mt(d, d, b, b, b2, workers);
  pair_ctx c = {d, b2, pm, (double**)calloc((size_t)pm->n_pairs + 1, sizeof(double*)),
                (pfo_status*)calloc((size_t)pm->n_pairs + 1, sizeof(pfo_status))};
  parallel_for_index(pm->n_pairs, workers, pair_shift, &c);
  int rc = first_error(pm->n_pairs, c.stats, st);
  if (st && rc) st->batch_index = 0;
  if (!rc) {
    double* accc = (double*)calloc(nn, sizeof(double));
    double* accs = (double*)calloc(nn, sizeof(double));
    double* t = (double*)malloc(sizeof(double) * nn);
    for (int k = 0; k < pm->n_pairs; ++k) {
      memcpy(t, c.z[k], sizeof(double) * nn);
      scale(nn, t, pm->cw[k]);
      axpy(nn, accc, 1.0, t);
      memcpy(t, c.z[k], sizeof(double) * nn);
      scale(nn, t, pm->sw[k]);
      axpy(nn, accs, 1.0, t);
    }
    /* C = a0 I - accC ; S' = a1 I - accS ; S = B S' */
    for (size_t i = 0; i < nn; ++i) {
      out_c[i] = -accc[i];
      t[i] = -accs[i];
    }
    for (int i = 0; i < d; ++i) {
      out_c[(size_t)i * d + i] = pm->a0 - accc[(size_t)i * d + i];
      t[(size_t)i * d + i] = pm->a1 - accs[(size_t)i * d + i];
    }
    mul_mt(d, d, b, t, out_s, workers);
    double* c2m = accc; /* reuse */
    double* s2m = accs;
    for (int s = 0; s < j; ++s) {
      mul_mt(d, d, out_c, out_c, c2m, workers);
      mul_mt(d, d, out_s, out_s, s2m, workers);
      mul_mt(d, d, out_s, out_c, t, workers);
      for (size_t i = 0; i < nn; ++i) {
        out_c[i] = c2m[i] - s2m[i];
        out_s[i] = 2.0 * t[i];
      }
    }
    free(accc);
    free(accs);
    free(t);
  }
  for (int k = 0; k < pm->n_pairs; ++k) free(c.z[k]);
  free(c.z);
  free(c.stats);
  free(b);
  free(b2);
  return rc;
}

typedef struct {
  int d;
  const double* a;
  const pfo_pair_method* pm;
  double theta;
  double *oc, *os;
  int* j_out;
  pfo_status* stats;
} cs_batch_ctx;

static void cossin_one(int i, void* p) {
  cs_batch_ctx* c = (cs_batch_ctx*)p;
  const size_t nn = (size_t)c->d * c->d;
  int j = 0;
  pfo_cossin(c->d, c->a + (size_t)i * nn, c->pm, c->theta, -1, 1, c->oc + (size_t)i * nn, c->os + (size_t)i * nn, &j,
             &c->stats[i]);
  if (c->j_out) c->j_out[i] = j;
}

int pfo_cossin_batched(int d, int batch, const double* a, const pfo_pair_method* pm, double theta, int threads,
                       double* out_c, double* out_s, int* j_out, pfo_status* st) {
  cs_batch_ctx c = {d, a, pm, theta, out_c, out_s, j_out,
                    (pfo_status*)calloc((size_t)(batch > 0 ? batch : 1), sizeof(pfo_status))};
  parallel_for_index(batch, threads, cossin_one, &c);
  int rc = first_error(batch, c.stats, st);
  free(c.stats);
  return rc;
}

/* ---------------------------------------------------------------- a13: dense block action */

typedef struct {
  int d;
  const double* b;
  const pfo_method* m;
  double** lu;
  int** piv;
  pfo_status* stats;
} factor_ctx;

static void factor_shift(int i, void* p) { /* ActionOperator ctor, action.cpp:300-312 */
  factor_ctx* c = (factor_ctx*)p;
  const int d = c->d;
  const size_t nn = (size_t)d * d;
  const double sh = c->m->shifts[i];
  c->lu[i] = NULL;
  c->piv[i] = NULL;
  if (sh == 0.0) return;
  double* mm = (double*)malloc(sizeof(double) * nn);
  memcpy(mm, c->b, sizeof(double) * nn);
  scale(nn, mm, -sh);
  add_scaled_identity(d, mm, 1.0);
  int* piv = (int*)malloc(sizeof(int) * (size_t)d);
  int rc = pfo_lu(d, mm, piv, 1e-14, &c->stats[i]);
  if (rc) {
    c->stats[i].code = rc;
    c->stats[i].shift_index = i + 1;
    free(mm);
    free(piv);
    return;
  }
  c->lu[i] = mm;
  c->piv[i] = piv;
}

typedef struct {
  int d, k;
  const pfo_method* m;
  double** lu;
  int** piv;
  const double* x;  /* current V */
  const double* bv; /* B V */
  double** terms;
  int inner;        /* threads per shift's solve */
} solve_ctx;

static void solve_shift(int i, void* p) { /* assemble_action per-shift body, action.cpp:240-263 */
  solve_ctx* c = (solve_ctx*)p;
  const size_t cnt = (size_t)c->d * c->k;
  const double sh = c->m->shifts[i], w = c->m->weights[i];
  double* term = c->terms[i];
  if (c->m->form == 0) {
    if (sh == 0.0)
      memcpy(term, c->x, sizeof(double) * cnt);
    else
      solve_mt(c->d, c->k, c->lu[i], c->piv[i], c->x, term, c->inner);
    scale(cnt, term, w);
  } else {
    if (sh == 0.0) {
      memset(term, 0, sizeof(double) * cnt);
      return;
    }
    double* rhs = (double*)malloc(sizeof(double) * cnt);
    for (size_t j = 0; j < cnt; ++j) rhs[j] = sh * c->bv[j];
    solve_mt(c->d, c->k, c->lu[i], c->piv[i], rhs, term, c->inner);
    scale(cnt, term, w);
    free(rhs);
  }
}

int pfo_action(int d, int k, const double* a, const double* v, const pfo_method* m, int substeps, int workers,
               double* out, pfo_status* st) {
  if (substeps < 1 || workers < 1) {
    if (st) st->code = CODE(ERRC_BAD_ARGUMENT);
    return CODE(ERRC_BAD_ARGUMENT);
  }
  const size_t nn = (size_t)d * d, cnt = (size_t)d * k;
  const int n = m->n_terms;
  double* b = (double*)malloc(sizeof(double) * nn);
  const double inv = 1.0 / substeps; /* action.cpp:330-334 */
  for (size_t i = 0; i < nn; ++i) b[i] = a[i] * inv;
  factor_ctx fc = {d, b, m, (double**)calloc((size_t)n + 1, sizeof(double*)), (int**)calloc((size_t)n + 1, sizeof(int*)),
                   (pfo_status*)calloc((size_t)n + 1, sizeof(pfo_status))};
  parallel_for_index(n, workers, factor_shift, &fc);
  int rc = first_error(n, fc.stats, st);
  if (st && rc) st->batch_index = 0;
  if (!rc) {
    double* x = (double*)malloc(sizeof(double) * cnt);
    double* bv = (double*)malloc(sizeof(double) * cnt);
    double* b2v = (double*)malloc(sizeof(double) * cnt);
    double** terms = (double**)calloc((size_t)n + 1, sizeof(double*));
    for (int i = 0; i < n; ++i) terms[i] = (double*)malloc(sizeof(double) * cnt);
    memcpy(x, v, sizeof(double) * cnt);
    for (int step = 0; step < substeps; ++step) {
      if (m->form == 1 || m->has_poly) mul_mt(d, k, b, x, bv, workers);
      int nz = 0;
      for (int i = 0; i < n; ++i) nz += m->shifts[i] != 0.0;
      solve_ctx sc = {d, k, m, fc.lu, fc.piv, x, bv, terms, nz > 0 && workers > nz ? workers / nz : 1};
      parallel_for_index(n, workers, solve_shift, &sc);
      memset(out, 0, sizeof(double) * cnt);
      for (int i = 0; i < n; ++i) axpy(cnt, out, 1.0, terms[i]);
      const double constant = m->form == 1 ? m->constant[0] : (m->has_poly ? m->poly[0] : 0.0);
      if (m->form == 1 || m->has_poly) {
        for (size_t j = 0; j < cnt; ++j) out[j] += constant * x[j];
        if (m->has_poly) {
          const double d1 = m->poly[1], d2 = m->poly[2];
          mul_mt(d, k, b, bv, b2v, workers);
          for (size_t j = 0; j < cnt; ++j) out[j] += d1 * bv[j] + d2 * b2v[j];
        }
      }
      memcpy(x, out, sizeof(double) * cnt);
    }
    for (int i = 0; i < n; ++i) free(terms[i]);
    free(terms);
    free(x);
    free(bv);
    free(b2v);
  }
  for (int i = 0; i < n; ++i) {
    free(fc.lu[i]);
    free(fc.piv[i]);
  }
  free(fc.lu);
  free(fc.piv);
  free(fc.stats);
  free(b);
  return rc;
}
