// f2: the banded action on the GPU -- tridiagonal shifted solves and the
// pentadiagonal banded LU of proj/core/src/action.cpp, applied to a block of k vectors (V is
// d x k row-major: one thread per column reads 32 consecutive columns per warp, so every band row
// access is a coalesced 256-byte segment). Each column runs exactly the reference's per-vector
// operation sequence (every product and difference separately rounded, IEEE division), so the
// results are the reference's bits.
//
//   band_factor_kernel      TridiagFactor (action.cpp:120-133) of M = I - c A (shifted_system,
//                           action.cpp:206-215) or of A itself; one thread per system -- the
//                           multiplier recurrence is sequential. ZeroPivot below 1e-300.
//   band_solve_kernel       TridiagFactor::solve (action.cpp:135-141) with the residual RHS c (A v)
//                           formed on the fly (assemble_action, action.cpp:250-254); thread per
//                           (system, column)
//   band_matvec_kernel      TridiagMatrix::matvec (action.cpp:35-44)
//   band_accumulate_kernel  assemble_action's ascending-shift sum and polynomial part (:262-283)
//   penta_factor_kernel /   pentadiag_solve (action.cpp:170-202) split into the band elimination
//   penta_solve_kernel      (matrix only, one thread) and the per-column substitution
#include "pf_common.cuh"

#ifndef PF_BAND_KR
#define PF_BAND_KR 6
#endif

namespace pf {

namespace {
constexpr double kFloor = 1e-300;
}

// sub / diag / super scaled by s (substep_action's A * (1/N), action.cpp:330-334)
__global__ void band_scale_kernel(int d, const double* sub, const double* diag, const double* super, double s,
                                  double* osub, double* odiag, double* osuper) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    odiag[i] = __dmul_rn(diag[i], s);
    if (i + 1 < d) {
      osub[i] = __dmul_rn(sub[i], s);
      osuper[i] = __dmul_rn(super[i], s);
    }
  }
}

// System z: shifted (c = shifts[z]): diag 1 - c a, sub / super -c a; else A itself (shifts null).
// mult[z] (d - 1), fdiag[z] (d), fsup[z] (d - 1, the system's super-diagonal). fail[z] = the
// ZeroPivot row or -1.
__global__ void band_factor_kernel(int d, int nsys, const double* sub, const double* diag, const double* super,
                                   const double* shifts, double* mult, double* fdiag, double* fsup, int* fail) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z >= nsys) return;
  const double c = shifts ? shifts[z] : 0.0;
  const bool shifted = shifts != nullptr;
  double* mu = mult + (int64_t)z * (d > 1 ? d - 1 : 1);
  double* fd = fdiag + (int64_t)z * d;
  double* fs = fsup + (int64_t)z * (d > 1 ? d - 1 : 1);
  double prev = shifted ? __dsub_rn(1.0, __dmul_rn(c, diag[0])) : diag[0];
  fd[0] = prev;
  int bad = -1;
  for (int i = 1; i < d; ++i) {
    const double l = shifted ? __dmul_rn(-c, sub[i - 1]) : sub[i - 1];
    const double u = shifted ? __dmul_rn(-c, super[i - 1]) : super[i - 1];
    const double dg = shifted ? __dsub_rn(1.0, __dmul_rn(c, diag[i])) : diag[i];
    fs[i - 1] = u;
    if (fabs(prev) <= kFloor) {
      bad = i - 1;
      break;
    }
    const double w = __ddiv_rn(l, prev);
    mu[i - 1] = w;
    prev = __dsub_rn(dg, __dmul_rn(w, u));
    fd[i] = prev;
  }
  if (bad < 0 && fabs(prev) <= kFloor) bad = d - 1;
  fail[z] = bad;
}

// X[z] (d x k, ldx) = M_z^-1 R, R = c_z * src (residual; rounded product) or src; z = blockIdx.y.
// The recurrence is sequential in the row, so memory-level parallelism comes from batching: every
// sweep issues the loads of kR rows (RHS / band coefficients / the forward result) before the
// dependent arithmetic on them (kR = 6 measured best of 4, 6, 8, 16, 32: profiles/r01_band_action.jsonl).
constexpr int kR = PF_BAND_KR;

__global__ void __launch_bounds__(128) band_solve_kernel(int d, int k, const double* __restrict__ mult,
                                                         const double* __restrict__ fdiag,
                                                         const double* __restrict__ fsup,
                                                         const double* __restrict__ src, int64_t lds,
                                                         const double* __restrict__ rhs_scale, double* __restrict__ X,
                                                         int64_t ldx, int64_t strideX) {
  const int z = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= k) return;
  const int64_t dm1 = d > 1 ? d - 1 : 1;
  const double* __restrict__ mu = mult + (int64_t)z * dm1;
  const double* __restrict__ fd = fdiag + (int64_t)z * d;
  const double* __restrict__ fs = fsup + (int64_t)z * dm1;
  double* __restrict__ x = X + (int64_t)z * strideX + col;
  const double* __restrict__ s = src + col;
  const bool scaled = rhs_scale != nullptr;
  const double cz = scaled ? rhs_scale[z] : 1.0;
  // forward: x_i = r_i - mult_{i-1} x_{i-1}
  double prev = scaled ? __dmul_rn(cz, s[0]) : s[0];
  x[0] = prev;
  for (int i0 = 1; i0 < d; i0 += kR) {
    double r[kR], m[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int i = i0 + u;
      r[u] = i < d ? __ldg(s + (int64_t)i * lds) : 0.0;  // shared by the P shift CTAs (L2)
      m[u] = i < d ? __ldg(mu + i - 1) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int i = i0 + u;
      if (i < d) {
        const double ri = scaled ? __dmul_rn(cz, r[u]) : r[u];
        prev = __dsub_rn(ri, __dmul_rn(m[u], prev));
        x[(int64_t)i * ldx] = prev;
      }
    }
  }
  // backward: x_{d-1} /= fdiag_{d-1}; x_i = (x_i - super_i x_{i+1}) / fdiag_i
  double nxt = __ddiv_rn(prev, fd[d - 1]);
  x[(int64_t)(d - 1) * ldx] = nxt;
  for (int i0 = d - 2; i0 >= 0; i0 -= kR) {
    double y[kR], f[kR], g[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int i = i0 - u;
      y[u] = i >= 0 ? x[(int64_t)i * ldx] : 0.0;
      f[u] = i >= 0 ? __ldg(fs + i) : 0.0;
      g[u] = i >= 0 ? __ldg(fd + i) : 1.0;
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int i = i0 - u;
      if (i >= 0) {
        nxt = __ddiv_rn(__dsub_rn(y[u], __dmul_rn(f[u], nxt)), g[u]);
        x[(int64_t)i * ldx] = nxt;
      }
    }
  }
}

// Out = A V (TridiagMatrix::matvec order: diag v_i, + sub v_{i-1}, + super v_{i+1})
__global__ void band_matvec_kernel(int d, int k, const double* sub, const double* diag, const double* super,
                                   const double* V, int64_t ldv, double* Out, int64_t ldo) {
  const int64_t total = (int64_t)d * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / k), c = (int)(idx % k);
    double acc = __dmul_rn(diag[i], V[(int64_t)i * ldv + c]);
    if (i > 0) acc = __dadd_rn(acc, __dmul_rn(sub[i - 1], V[(int64_t)(i - 1) * ldv + c]));
    if (i + 1 < d) acc = __dadd_rn(acc, __dmul_rn(super[i], V[(int64_t)(i + 1) * ldv + c]));
    Out[(int64_t)i * ldo + c] = acc;
  }
}

// out = sum_t (w_t x_t) in ascending t (x_t = X[slot_t], or V for a plain zero shift), acc starting
// at 0; then + constant v, + (d1 av + d2 a2v) when add_poly (hybrid: has_poly)
__global__ void band_accumulate_kernel(int d, int k, int n_terms, const int* slot, const double* w, const double* X,
                                       int64_t ldx, int64_t strideX, const double* V, int64_t ldv, int add_poly,
                                       double constant, int hybrid, double d1, double d2, const double* AV,
                                       const double* A2V, double* out, int64_t ldo) {
  const int64_t total = (int64_t)d * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / k), c = (int)(idx % k);
    const double v = V[(int64_t)i * ldv + c];
    double acc = 0.0;
    for (int t = 0; t < n_terms; ++t) {
      const double xv = slot[t] >= 0 ? X[(int64_t)slot[t] * strideX + (int64_t)i * ldx + c] : v;
      acc = __dadd_rn(acc, __dmul_rn(xv, w[t]));
    }
    if (add_poly) {
      acc = __dadd_rn(acc, __dmul_rn(constant, v));
      if (hybrid) {
        const double av = AV[(int64_t)i * k + c], a2v = A2V[(int64_t)i * k + c];
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(d1, av), __dmul_rn(d2, a2v)));
      }
    }
    out[(int64_t)i * ldo + c] = acc;
  }
}

// pentadiag_solve's band elimination (matrix only): F[i * 2 + off - 1] = the multiplier of row
// i + off (0 when the reference skips it, f == 0), U[i * 3 + c] = the eliminated band W(i, c),
// c = 0..2. fail = ZeroPivot row or -1. One thread.
__global__ void penta_factor_kernel(int d, const double* sub2, const double* sub1, const double* diag,
                                    const double* super1, const double* super2, double* W, double* F, int* fail) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  // W(i, c) for c in [-2, 2] at W[i * 5 + c + 2]
  for (int i = 0; i < d; ++i) {
    for (int c = 0; c < 5; ++c) W[(int64_t)i * 5 + c] = 0.0;
    W[(int64_t)i * 5 + 2] = diag[i];
    if (i > 1) W[(int64_t)i * 5 + 0] = sub2[i - 2];
    if (i > 0) W[(int64_t)i * 5 + 1] = sub1[i - 1];
    if (i + 1 < d) W[(int64_t)i * 5 + 3] = super1[i];
    if (i + 2 < d) W[(int64_t)i * 5 + 4] = super2[i];
  }
  int bad = -1;
  for (int i = 0; i < d && bad < 0; ++i) {
    const double piv = W[(int64_t)i * 5 + 2];
    if (fabs(piv) <= kFloor) {
      bad = i;
      break;
    }
    for (int off = 1; off <= 2; ++off) {
      F[(int64_t)i * 2 + off - 1] = 0.0;
      const int r = i + off;
      if (r >= d) break;
      const double f = __ddiv_rn(W[(int64_t)r * 5 + 2 - off], piv);
      F[(int64_t)i * 2 + off - 1] = f;
      if (f == 0.0) continue;
      W[(int64_t)r * 5 + 2 - off] = 0.0;
      for (int c = 1; c <= 2; ++c)
        if (i + c < d) {
          double& t = W[(int64_t)r * 5 + 2 + c - off];
          t = __dsub_rn(t, __dmul_rn(f, W[(int64_t)i * 5 + 2 + c]));
        }
    }
  }
  *fail = bad;
}

__global__ void penta_solve_kernel(int d, int k, const double* W, const double* F, const double* rhs, int64_t ldr,
                                   double* X, int64_t ldx) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= k) return;
  double* x = X + col;
  for (int i = 0; i < d; ++i) x[(int64_t)i * ldx] = rhs[(int64_t)i * ldr + col];
  for (int i = 0; i < d; ++i) {
    const double xi = x[(int64_t)i * ldx];
    for (int off = 1; off <= 2; ++off) {
      const int r = i + off;
      if (r >= d) break;
      const double f = F[(int64_t)i * 2 + off - 1];
      if (f == 0.0) continue;
      x[(int64_t)r * ldx] = __dsub_rn(x[(int64_t)r * ldx], __dmul_rn(f, xi));
    }
  }
  for (int i = d - 1; i >= 0; --i) {
    double acc = x[(int64_t)i * ldx];
    for (int c = 1; c <= 2; ++c)
      if (i + c < d) acc = __dsub_rn(acc, __dmul_rn(W[(int64_t)i * 5 + 2 + c], x[(int64_t)(i + c) * ldx]));
    x[(int64_t)i * ldx] = __ddiv_rn(acc, W[(int64_t)i * 5 + 2]);
  }
}

}  // namespace pf
