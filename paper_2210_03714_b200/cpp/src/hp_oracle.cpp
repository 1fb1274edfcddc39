// High-precision oracles of the experiment drivers, in IEEE binary128
// (__float128, 113-bit significand, ~34 decimal digits) in place of the reference's GMP BigFloat
// (GMP's C++ layer is absent here). Same algorithms as the reference:
//   taylor_degree_for          dense.cpp:417-425
//   taylor_sum_ps              dense.cpp:428-458  (Paterson-Stockmeyer blocks)
//   expm_oracle                dense.cpp:460-476  (halve to ||.||_1 <= 1/4, Taylor, square back)
//   phi1_oracle                dense.cpp:478-487  (direct Taylor of phi1)
//   error_vs_oracle (dense)    dense.cpp:489-499  (diff rounded toward zero like mpf get_d, then
//                                                  two_norm_est)
//   two_norm_est               dense.cpp:70-96, action.cpp:67-94 (power iteration on M^T M)
//   action_oracle              action.cpp:440-490 (Taylor substeps at scaled norm <= 1/2)
//   error_vs_oracle (action)   action.cpp:492-502 (2-norm of the diff vector)
// The requested digits only set the Taylor degree (as in the reference); the working precision is
// binary128's, far below the 1e-16 errors these drivers measure.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace {

using q128 = __float128;

int taylor_degree_for(double x, int target_digits) {
  if (x <= 0) return 1;
  double log_term = std::log10(x);
  for (int m = 1; m < 20000; ++m) {
    log_term += std::log10(x) - std::log10(double(m + 1));
    if (x / (m + 2) < 0.5 && log_term + std::log10(2.0) < -double(target_digits)) return m;
  }
  return -1;
}

q128 qabs(q128 x) { return x < 0 ? -x : x; }

// round toward zero (mpf_get_d semantics)
double to_double_rz(q128 x) {
  double r = (double)x;
  if (qabs((q128)r) > qabs(x)) r = std::nextafter(r, 0.0);
  return r;
}

struct QMat {
  int d;
  std::vector<q128> a;
  explicit QMat(int n) : d(n), a(size_t(n) * n, 0) {}
  q128& at(int i, int j) { return a[size_t(i) * d + j]; }
  q128 at(int i, int j) const { return a[size_t(i) * d + j]; }
  static QMat identity(int n) {
    QMat m(n);
    for (int i = 0; i < n; ++i) m.at(i, i) = 1;
    return m;
  }
  QMat mul(const QMat& b) const {  // i-k-j, like DenseMatrix::mul
    QMat c(d);
    for (int i = 0; i < d; ++i)
      for (int k = 0; k < d; ++k) {
        const q128 aik = at(i, k);
        if (aik == 0) continue;
        q128* crow = &c.a[size_t(i) * d];
        const q128* brow = &b.a[size_t(k) * d];
        for (int j = 0; j < d; ++j) crow[j] += aik * brow[j];
      }
    return c;
  }
  void axpy(q128 s, const QMat& x) {
    for (size_t i = 0; i < a.size(); ++i) a[i] += s * x.a[i];
  }
  double one_norm_d() const {
    q128 best = 0;
    for (int j = 0; j < d; ++j) {
      q128 s = 0;
      for (int i = 0; i < d; ++i) s += qabs(at(i, j));
      if (s > best) best = s;
    }
    return (double)best;
  }
};

// sum_{k=0..m} coeff_k X^k, Paterson-Stockmeyer: p = ceil(sqrt(m + 1)) powers, q = m / p blocks
QMat taylor_sum_ps(const QMat& x, const std::vector<q128>& coeffs) {
  const int m = int(coeffs.size()) - 1, d = x.d;
  const int p = std::max(1, int(std::ceil(std::sqrt(double(m + 1)))));
  const int q = m / p;
  std::vector<QMat> powers;
  powers.push_back(QMat::identity(d));
  for (int r = 1; r <= p; ++r) powers.push_back(powers.back().mul(x));
  QMat acc(d);
  for (int j = q; j >= 0; --j) {
    QMat block(d);
    for (int r = 0; r < p; ++r) {
      const int k = j * p + r;
      if (k > m) break;
      if (coeffs[size_t(k)] == 0) continue;
      block.axpy(coeffs[size_t(k)], powers[size_t(r)]);
    }
    if (j == q) {
      acc = std::move(block);
    } else {
      acc = acc.mul(powers[size_t(p)]);
      acc.axpy(1, block);
    }
  }
  return acc;
}

std::vector<q128> exp_coeffs(int m, int shift) {  // 1 / (k + shift)!, shift 0: exp, 1: phi1
  std::vector<q128> c(size_t(m) + 1);
  q128 f = 1;
  for (int k = 1; k <= shift; ++k) f *= k;
  for (int k = 0; k <= m; ++k) {
    if (k > 0) f *= (k + shift);
    c[size_t(k)] = 1 / f;
  }
  return c;
}

QMat from_doubles(int d, const double* b) {
  QMat h(d);
  for (size_t i = 0; i < h.a.size(); ++i) h.a[i] = b[i];
  return h;
}

double two_norm_est_dense(int d, const double* m, int iterations) {
  if (d == 0) return 0;
  std::vector<double> v(static_cast<size_t>(d)), w(static_cast<size_t>(d)), u(static_cast<size_t>(d));
  for (int i = 0; i < d; ++i) v[size_t(i)] = 1.0 + double(i) / double(d);
  auto normalize = [](std::vector<double>& x) {
    double n = 0;
    for (double e : x) n += e * e;
    n = std::sqrt(n);
    if (n > 0)
      for (double& e : x) e /= n;
    return n;
  };
  normalize(v);
  double sigma = 0;
  for (int it = 0; it < iterations; ++it) {
    for (int i = 0; i < d; ++i) {  // DenseMatrix::matvec: row dot products, ascending j
      double acc = 0;
      for (int j = 0; j < d; ++j) acc += m[size_t(i) * d + j] * v[size_t(j)];
      w[size_t(i)] = acc;
    }
    std::fill(u.begin(), u.end(), 0.0);
    for (int i = 0; i < d; ++i) {
      const double wi = w[size_t(i)];
      if (wi == 0.0) continue;
      for (int j = 0; j < d; ++j) u[size_t(j)] += m[size_t(i) * d + j] * wi;
    }
    const double un = normalize(u);
    v.swap(u);
    sigma = std::sqrt(un);
    if (un == 0) break;
  }
  return sigma;
}

}  // namespace

extern "C" {

// kind 0: exp(b), 1: phi1(b). diff[t] = RZ(oracle - approx[t]) for t < n_approx (d x d row-major
// each). Returns 0, or 10 (BadArgument: digits < 30, d < 1, no Taylor degree).
int pf_hp_dense_diff(int kind, int d, const double* b, int digits, int n_approx, const double* approx, double* diff) {
  if (d < 1 || digits < 30 || (kind != 0 && kind != 1)) return 10;
  QMat h = from_doubles(d, b);
  QMat e(d);
  if (kind == 0) {
    double nrm = h.one_norm_d();
    long squarings = 0;
    while (nrm > 0.25) {
      nrm /= 2;
      ++squarings;
    }
    q128 s = 1;
    for (long i = 0; i < squarings; ++i) s /= 2;
    for (auto& x : h.a) x *= s;
    const int m = taylor_degree_for(0.25, digits + 10);
    if (m < 0) return 10;
    e = taylor_sum_ps(h, exp_coeffs(m, 0));
    for (long i = 0; i < squarings; ++i) e = e.mul(e);
  } else {
    // phi1_oracle takes max(||b||_1, 1) from the double matrix (DenseMatrix::one_norm)
    double nrm = 0;
    for (int j = 0; j < d; ++j) {
      double s = 0;
      for (int i = 0; i < d; ++i) s += std::fabs(b[size_t(i) * d + j]);
      nrm = std::max(nrm, s);
    }
    nrm = std::max(nrm, 1.0);
    const int m = taylor_degree_for(nrm, digits + 10);
    if (m < 0) return 10;
    e = taylor_sum_ps(h, exp_coeffs(m, 1));
  }
  const size_t nn = size_t(d) * d;
  for (int t = 0; t < n_approx; ++t)
    for (size_t i = 0; i < nn; ++i) diff[size_t(t) * nn + i] = to_double_rz(e.a[i] - (q128)approx[size_t(t) * nn + i]);
  return 0;
}

// exp(A) v for tridiagonal A (sub / super d - 1, diag d), by the reference's Taylor substeps.
// err[t] = || RZ(oracle - approx[t]) ||_2 (approx: n_approx vectors of length d).
int pf_hp_action_error(int d, const double* sub, const double* diag, const double* super, const double* v, int digits,
                       int n_approx, const double* approx, double* err) {
  if (d < 1 || digits < 30) return 10;
  double nrm = 0;  // TridiagMatrix::one_norm (action.cpp:55-64)
  for (int j = 0; j < d; ++j) {
    double col = std::fabs(diag[j]);
    if (j > 0) col += std::fabs(super[j - 1]);
    if (j + 1 < d) col += std::fabs(sub[j]);
    nrm = std::max(nrm, col);
  }
  const int substeps = std::max(1, int(std::ceil(nrm / 0.5)));
  int degree = 1;
  {
    double log_term = std::log10(0.5);
    for (int m = 1; m < 20000; ++m) {
      log_term += std::log10(0.5) - std::log10(double(m + 1));
      if (log_term + std::log10(2.0) < -double(digits + 10)) {
        degree = m;
        break;
      }
    }
  }
  std::vector<q128> x(static_cast<size_t>(d)), acc(x), w(x), t(x);
  for (int i = 0; i < d; ++i) x[size_t(i)] = v[i];
  for (int step = 0; step < substeps; ++step) {
    acc = x;
    w = x;
    for (int k = 1; k <= degree; ++k) {
      for (int i = 0; i < d; ++i) {
        q128 a = (q128)diag[i] * w[size_t(i)];
        if (i > 0) a += (q128)sub[i - 1] * w[size_t(i - 1)];
        if (i + 1 < d) a += (q128)super[i] * w[size_t(i + 1)];
        t[size_t(i)] = a;
      }
      const q128 scale = (q128)substeps * k;
      for (int i = 0; i < d; ++i) {
        w[size_t(i)] = t[size_t(i)] / scale;
        acc[size_t(i)] += w[size_t(i)];
      }
    }
    x = acc;
  }
  for (int s = 0; s < n_approx; ++s) {
    double a2 = 0;
    for (int i = 0; i < d; ++i) {
      const double e = to_double_rz(x[size_t(i)] - (q128)approx[size_t(s) * d + i]);
      a2 += e * e;
    }
    err[s] = std::sqrt(a2);
  }
  return 0;
}

double pf_two_norm_est_dense(int d, const double* m, int iterations) { return two_norm_est_dense(d, m, iterations); }

double pf_two_norm_est_tridiag(int d, const double* sub, const double* diag, const double* super, int iterations) {
  if (d <= 0) return 0;
  std::vector<double> v(static_cast<size_t>(d)), w(static_cast<size_t>(d)), u(static_cast<size_t>(d));
  for (int i = 0; i < d; ++i) v[size_t(i)] = 1.0 + double(i) / double(d);
  auto normalize = [](std::vector<double>& x) {
    double n = 0;
    for (double e : x) n += e * e;
    n = std::sqrt(n);
    if (n > 0)
      for (double& e : x) e /= n;
    return n;
  };
  normalize(v);
  double sigma = 0;
  for (int it = 0; it < iterations; ++it) {
    for (int i = 0; i < d; ++i) {  // TridiagMatrix::matvec
      double acc = diag[i] * v[size_t(i)];
      if (i > 0) acc += sub[i - 1] * v[size_t(i - 1)];
      if (i + 1 < d) acc += super[i] * v[size_t(i + 1)];
      w[size_t(i)] = acc;
    }
    std::fill(u.begin(), u.end(), 0.0);
    for (int i = 0; i < d; ++i) {
      const double wi = w[size_t(i)];
      u[size_t(i)] += diag[i] * wi;
      if (i > 0) u[size_t(i - 1)] += sub[i - 1] * wi;
      if (i + 1 < d) u[size_t(i + 1)] += super[i] * wi;
    }
    const double un = normalize(u);
    v.swap(u);
    sigma = std::sqrt(un);
    if (un == 0) break;
  }
  return sigma;
}

}  // extern "C"
