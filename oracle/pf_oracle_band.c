/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the banded (tridiagonal / pentadiagonal) action,
 * SURVEY.md §8(f) row f2. Plain-C restatement of proj/core/src/action.cpp, same operation order:
 *   TridiagMatrix::matvec                          action.cpp:35-44
 *   TridiagMatrix::one_norm                        action.cpp:55-64
 *   thomas_solve (ZeroPivot below 1e-300)          action.cpp:100-118
 *   TridiagFactor / TridiagFactor::solve           action.cpp:120-141
 *   pentadiag_solve (banded LU, skip f == 0)       action.cpp:170-202
 *   shifted_system  (1 - c a_ii, -c a_i,i+-1)      action.cpp:206-215
 *   assemble_action / action_eval / ActionOperator / substep_action
 *                                                  action.cpp:224-339
 * Vectors are applied one column at a time; a "block" here is k independent columns of a d x k
 * row-major array (the GPU API's layout), each processed exactly as the reference processes one
 * vector. Only tests/ and bench-side baselines may load this code.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "pf_oracle.h"

#define PIVOT_FLOOR 1e-300
#define ERR_ZERO_PIVOT 8 /* Errc::ZeroPivot + 1 */
#define ERR_BAD_ARGUMENT 10

void pfo_tridiag_matvec(int d, const double* sub, const double* diag, const double* super, const double* v,
                        double* out) {
  for (int i = 0; i < d; ++i) {
    double acc = diag[i] * v[i];
    if (i > 0) acc += sub[i - 1] * v[i - 1];
    if (i + 1 < d) acc += super[i] * v[i + 1];
    out[i] = acc;
  }
}

double pfo_tridiag_one_norm(int d, const double* sub, const double* diag, const double* super) {
  double best = 0;
  for (int j = 0; j < d; ++j) {
    double col = fabs(diag[j]);
    if (j > 0) col += fabs(super[j - 1]);
    if (j + 1 < d) col += fabs(sub[j]);
    if (col > best) best = col;
  }
  return best;
}

/* returns 0 or ZeroPivot + 1 with *row = failing row */
int pfo_thomas_solve(int d, const double* sub, const double* diag, const double* super, const double* rhs,
                     double* x, int* row) {
  double* dia = (double*)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
  memcpy(dia, diag, sizeof(double) * (size_t)d);
  memcpy(x, rhs, sizeof(double) * (size_t)d);
  for (int i = 1; i < d; ++i) {
    if (fabs(dia[i - 1]) <= PIVOT_FLOOR) {
      *row = i - 1;
      free(dia);
      return ERR_ZERO_PIVOT;
    }
    const double w = sub[i - 1] / dia[i - 1];
    dia[i] -= w * super[i - 1];
    x[i] -= w * x[i - 1];
  }
  if (fabs(dia[d - 1]) <= PIVOT_FLOOR) {
    *row = d - 1;
    free(dia);
    return ERR_ZERO_PIVOT;
  }
  x[d - 1] /= dia[d - 1];
  for (int i = d - 2; i >= 0; --i) x[i] = (x[i] - super[i] * x[i + 1]) / dia[i];
  free(dia);
  return 0;
}

int pfo_tridiag_factor(int d, const double* sub, const double* diag, const double* super, double* mult,
                       double* fdiag, int* row) {
  memcpy(fdiag, diag, sizeof(double) * (size_t)d);
  for (int i = 1; i < d; ++i) {
    if (fabs(fdiag[i - 1]) <= PIVOT_FLOOR) {
      *row = i - 1;
      return ERR_ZERO_PIVOT;
    }
    const double w = sub[i - 1] / fdiag[i - 1];
    mult[i - 1] = w;
    fdiag[i] -= w * super[i - 1];
  }
  if (d > 0 && fabs(fdiag[d - 1]) <= PIVOT_FLOOR) {
    *row = d - 1;
    return ERR_ZERO_PIVOT;
  }
  return 0;
}

void pfo_tridiag_factor_solve(int d, const double* mult, const double* fdiag, const double* super, const double* rhs,
                              double* x) {
  memcpy(x, rhs, sizeof(double) * (size_t)d);
  for (int i = 1; i < d; ++i) x[i] -= mult[i - 1] * x[i - 1];
  x[d - 1] /= fdiag[d - 1];
  for (int i = d - 2; i >= 0; --i) x[i] = (x[i] - super[i] * x[i + 1]) / fdiag[i];
}

int pfo_pentadiag_solve(int d, const double* sub2, const double* sub1, const double* diag, const double* super1,
                        const double* super2, const double* rhs, double* x, int* row) {
  double* w = (double*)calloc((size_t)(d > 0 ? d : 1) * 5, sizeof(double));
#define W(i, c) w[(size_t)(i) * 5 + (size_t)((c) + 2)]
  for (int i = 0; i < d; ++i) {
    W(i, 0) = diag[i];
    if (i > 1) W(i, -2) = sub2[i - 2];
    if (i > 0) W(i, -1) = sub1[i - 1];
    if (i + 1 < d) W(i, 1) = super1[i];
    if (i + 2 < d) W(i, 2) = super2[i];
  }
  memcpy(x, rhs, sizeof(double) * (size_t)d);
  for (int i = 0; i < d; ++i) {
    const double piv = W(i, 0);
    if (fabs(piv) <= PIVOT_FLOOR) {
      *row = i;
      free(w);
      return ERR_ZERO_PIVOT;
    }
    for (int off = 1; off <= 2; ++off) {
      const int r = i + off;
      if (r >= d) break;
      const double f = W(r, -off) / piv;
      if (f == 0.0) continue;
      W(r, -off) = 0.0;
      for (int c = 1; c <= 2; ++c)
        if (i + c < d) W(r, c - off) -= f * W(i, c);
      x[r] -= f * x[i];
    }
  }
  for (int i = d - 1; i >= 0; --i) {
    double acc = x[i];
    for (int c = 1; c <= 2; ++c)
      if (i + c < d) acc -= W(i, c) * x[i + c];
    x[i] = acc / W(i, 0);
  }
#undef W
  free(w);
  return 0;
}

/* substep_action on every column of V (d x k row-major): A scaled by 1/N, then N x
 * (v <- action_eval(m, A/N, v)); the shifted systems factored once (ActionOperator's factors
 * perform the same operations as thomas_solve). Returns 0 or Errc + 1 (st->shift_index, column = row). */
int pfo_tridiag_action(int d, int k, const double* sub, const double* diag, const double* super, const double* v,
                       const pfo_method* m, int substeps, double* out, pfo_status* st) {
  if (st) memset(st, 0, sizeof(*st));
  if (substeps < 1 || d < 1 || k < 0) {
    if (st) st->code = ERR_BAD_ARGUMENT;
    return ERR_BAD_ARGUMENT;
  }
  const double inv = 1.0 / substeps;
  const size_t dm1 = (size_t)(d > 1 ? d - 1 : 1);
  double* ss = (double*)malloc(sizeof(double) * dm1);
  double* sd = (double*)malloc(sizeof(double) * (size_t)d);
  double* sp = (double*)malloc(sizeof(double) * dm1);
  for (int i = 0; i + 1 < d; ++i) {
    ss[i] = sub[i] * inv;
    sp[i] = super[i] * inv;
  }
  for (int i = 0; i < d; ++i) sd[i] = diag[i] * inv;
  int nz = 0;
  for (int i = 0; i < m->n_terms; ++i) nz += m->shifts[i] != 0.0;
  double* mult = (double*)malloc(sizeof(double) * dm1 * (size_t)(nz > 0 ? nz : 1));
  double* fdiag = (double*)malloc(sizeof(double) * (size_t)d * (size_t)(nz > 0 ? nz : 1));
  double* msub = (double*)malloc(sizeof(double) * dm1);
  double* mdiag = (double*)malloc(sizeof(double) * (size_t)d);
  double* msup = (double*)malloc(sizeof(double) * dm1);
  int rc = 0, slot = 0;
  for (int i = 0; i < m->n_terms && !rc; ++i) {
    const double c = m->shifts[i];
    if (c == 0.0) continue;
    /* shifted_system: diag 1 - c a_ii, off-diagonals -c a */
    for (int q = 0; q < d; ++q) mdiag[q] = 1.0 - c * sd[q];
    for (int q = 0; q + 1 < d; ++q) {
      msub[q] = -c * ss[q];
      msup[q] = -c * sp[q];
    }
    int row = 0;
    rc = pfo_tridiag_factor(d, msub, mdiag, msup, mult + (size_t)slot * dm1, fdiag + (size_t)slot * (size_t)d, &row);
    if (rc && st) {
      st->code = rc;
      st->shift_index = i + 1;
      st->column = row;
    }
    ++slot;
  }
  if (!rc) {
    /* per-slot super-diagonals */
    double* supers = (double*)malloc(sizeof(double) * dm1 * (size_t)(nz > 0 ? nz : 1));
    slot = 0;
    for (int i = 0; i < m->n_terms; ++i) {
      const double c = m->shifts[i];
      if (c == 0.0) continue;
      for (int q = 0; q + 1 < d; ++q) supers[(size_t)slot * dm1 + (size_t)q] = -c * sp[q];
      ++slot;
    }
    double* col = (double*)malloc(sizeof(double) * (size_t)d);
    double* nxt = (double*)malloc(sizeof(double) * (size_t)d);
    double* av = (double*)malloc(sizeof(double) * (size_t)d);
    double* a2v = (double*)malloc(sizeof(double) * (size_t)d);
    double* rhs = (double*)malloc(sizeof(double) * (size_t)d);
    double* x = (double*)malloc(sizeof(double) * (size_t)d);
    for (int cidx = 0; cidx < k; ++cidx) {
      for (int q = 0; q < d; ++q) col[q] = v[(size_t)q * (size_t)k + (size_t)cidx];
      for (int s = 0; s < substeps; ++s) {
        /* assemble_action: terms in ascending shift order, then the polynomial part */
        const int residual = m->form == 1, hybrid = m->has_poly != 0;
        if (residual || hybrid) pfo_tridiag_matvec(d, ss, sd, sp, col, av);
        for (int q = 0; q < d; ++q) nxt[q] = 0.0;
        int sl = 0;
        for (int i = 0; i < m->n_terms; ++i) {
          const double c = m->shifts[i], w = m->weights[i];
          if (!residual && c == 0.0) {
            for (int q = 0; q < d; ++q) nxt[q] += col[q] * w;
            continue;
          }
          if (c == 0.0) continue; /* residual zero shift: zero term (0 + 0 leaves acc unchanged) */
          const double* src = col;
          if (residual) {
            for (int q = 0; q < d; ++q) rhs[q] = c * av[q];
            src = rhs;
          }
          pfo_tridiag_factor_solve(d, mult + (size_t)sl * dm1, fdiag + (size_t)sl * (size_t)d,
                                   supers + (size_t)sl * dm1, src, x);
          for (int q = 0; q < d; ++q) nxt[q] += x[q] * w;
          ++sl;
        }
        if (residual || hybrid) {
          const double constant = residual ? m->constant[0] : m->poly[0];
          for (int q = 0; q < d; ++q) nxt[q] += constant * col[q];
          if (hybrid) {
            const double d1 = m->poly[1], d2 = m->poly[2];
            pfo_tridiag_matvec(d, ss, sd, sp, av, a2v);
            for (int q = 0; q < d; ++q) nxt[q] += d1 * av[q] + d2 * a2v[q];
          }
        }
        memcpy(col, nxt, sizeof(double) * (size_t)d);
      }
      for (int q = 0; q < d; ++q) out[(size_t)q * (size_t)k + (size_t)cidx] = col[q];
    }
    free(col);
    free(nxt);
    free(av);
    free(a2v);
    free(rhs);
    free(x);
    free(supers);
  }
  free(ss);
  free(sd);
  free(sp);
  free(mult);
  free(fdiag);
  free(msub);
  free(mdiag);
  free(msup);
  return rc;
}
