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
//   band_action_bulk_kernel / band_action_step_kernel
//                           one whole substep (action_eval on every column) fused: forward sweep,
//                           back-substitution and the ordered sum in one launch (the three kernels
//                           above remain the path for methods with more than 12 factored shifts)
//   band_pack_records_kernel per-row coefficient records for the bulk kernel's copies
//   penta_factor_kernel /   pentadiag_solve (action.cpp:170-202) split into the band elimination
//   penta_solve_kernel      (matrix only, one thread) and the per-column substitution
#include <algorithm>

#include "pf_common.cuh"
#include "pf_kernels.h"
#include "band_div.cuh"

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
// mult[z] (d - 1), fdiag[z] (d), fsup[z] (d - 1, the system's super-diagonal), frcp[z] (d,
// band_rcp of the pivots; optional). fail[z] = the ZeroPivot row or -1.
__global__ void band_factor_kernel(int d, int nsys, const double* __restrict__ sub, const double* __restrict__ diag,
                                   const double* __restrict__ super, const double* shifts, double* __restrict__ mult,
                                   double* __restrict__ fdiag, double* __restrict__ fsup, double* __restrict__ frcp,
                                   int* fail) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z >= nsys) return;
  const double c = shifts ? shifts[z] : 0.0;
  const bool shifted = shifts != nullptr;
  double* __restrict__ mu = mult + (int64_t)z * (d > 1 ? d - 1 : 1);
  double* __restrict__ fd = fdiag + (int64_t)z * d;
  double* __restrict__ fs = fsup + (int64_t)z * (d > 1 ? d - 1 : 1);
  double* __restrict__ fr = frcp ? frcp + (int64_t)z * d : nullptr;
  double prev = shifted ? __dsub_rn(1.0, __dmul_rn(c, diag[0])) : diag[0];
  fd[0] = prev;
  if (fr) fr[0] = band_rcp(prev);
  int bad = -1;
  // the recurrence is sequential: the coefficient loads of the next 8 rows are issued while the
  // current 8 are eliminated, so global latency stays off the chain (same operations, same bits)
  constexpr int kF = 8;
  double la[kF], ua[kF], da[kF], lb[kF], ub[kF], db[kF];
  auto fetch = [&](double (&ls)[kF], double (&us)[kF], double (&ds)[kF], int i0) {
#pragma unroll
    for (int u = 0; u < kF; ++u) {
      const int i = i0 + u;
      ls[u] = i < d ? __ldg(sub + i - 1) : 0.0;
      us[u] = i < d ? __ldg(super + i - 1) : 0.0;
      ds[u] = i < d ? __ldg(diag + i) : 1.0;
    }
  };
  auto eliminate = [&](const double (&ls)[kF], const double (&us)[kF], const double (&ds)[kF], int i0) {
#pragma unroll
    for (int u = 0; u < kF; ++u) {
      const int i = i0 + u;
      if (i >= d || bad >= 0) break;
      const double l = shifted ? __dmul_rn(-c, ls[u]) : ls[u];
      const double uu = shifted ? __dmul_rn(-c, us[u]) : us[u];
      const double dg = shifted ? __dsub_rn(1.0, __dmul_rn(c, ds[u])) : ds[u];
      fs[i - 1] = uu;
      if (fabs(prev) <= kFloor) {
        bad = i - 1;
        break;
      }
      const double w = __ddiv_rn(l, prev);
      mu[i - 1] = w;
      prev = __dsub_rn(dg, __dmul_rn(w, uu));
      fd[i] = prev;
      if (fr) fr[i] = band_rcp(prev);
    }
  };
  if (d > 1) fetch(la, ua, da, 1);
  for (int i0 = 1; i0 < d && bad < 0; i0 += 2 * kF) {  // two batches per trip: static buffers
    if (i0 + kF < d) fetch(lb, ub, db, i0 + kF);
    eliminate(la, ua, da, i0);
    if (i0 + kF >= d || bad >= 0) break;
    if (i0 + 2 * kF < d) fetch(la, ua, da, i0 + 2 * kF);
    eliminate(lb, ub, db, i0 + kF);
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
                                                         const double* __restrict__ frcp,
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
  const double* __restrict__ fr = frcp + (int64_t)z * d;  // band_rcp of the pivots (div_rcp)
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
  double nxt = div_rcp(prev, fd[d - 1], fr[d - 1]);
  x[(int64_t)(d - 1) * ldx] = nxt;
  for (int i0 = d - 2; i0 >= 0; i0 -= kR) {
    double y[kR], f[kR], g[kR], gr[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int i = i0 - u;
      y[u] = i >= 0 ? x[(int64_t)i * ldx] : 0.0;
      f[u] = i >= 0 ? __ldg(fs + i) : 0.0;
      g[u] = i >= 0 ? __ldg(fd + i) : 1.0;
      gr[u] = i >= 0 ? __ldg(fr + i) : 1.0;
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int i = i0 - u;
      if (i >= 0) {
        nxt = div_rcp(__dsub_rn(y[u], __dmul_rn(f[u], nxt)), g[u], gr[u]);
        x[(int64_t)i * ldx] = nxt;
      }
    }
  }
}

// One substep of the banded action, fused (action_eval, action.cpp:224-283, on every column):
// CTA = one 32-column strip, warp t = factored shift t. Forward: each warp forms its RHS row by
// row (residual: c_t * (A v)_i from a 3-row sliding window of V, the matvec in
// TridiagMatrix::matvec order; plain: v_i), eliminates, and parks the forward result in Y[t].
// Backward: each warp back-substitutes R rows at a time into shared memory; after one barrier
// the whole CTA sums the R x 32 outputs over the terms in ascending shift index (acc from 0,
// every product / sum separately rounded), adds the polynomial part and writes out. HBM passes
// per substep: V twice, Y[t] twice per shift, out once (2P + 3) -- the unfused chain
// (matvec, P solves writing / re-reading / rewriting X_t, a P-way accumulate) moves ~5P + 5.
//
// The recurrences are latency chains, so the streams feeding them run ahead through a per-warp
// cp.async queue of S stages: a stage holds R rows of the warp's 32 columns (each lane copies its
// own column, 8 bytes) plus the R rows of band coefficients those rows need (one scalar per lane,
// lanes < 4R). S - 1 stages are in flight while the warp works on the oldest. Interior stages
// take a bounds-free path (pointer increments, immediate offsets); the first and last stage of
// each sweep take the checked one. The division by the pivot uses the pivot's reciprocal
// (band_div.cuh: bit-identical to IEEE division, checked by tools/probe_div.cu).
namespace {
__device__ __forceinline__ void cp8(unsigned sa, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
}  // namespace

template <int G, int S, int R>
constexpr size_t band_step_smem() {
  return sizeof(double) * ((size_t)G * S * (R * 32 + 4 * R) + (size_t)S * R * 32);
}

template <int G, int S, int R>
__global__ void __launch_bounds__(G * 32) band_action_step_kernel(
    int d, int k, const double* __restrict__ ssub, const double* __restrict__ sdiag, const double* __restrict__ ssup,
    const double* __restrict__ mult, const double* __restrict__ fdiag, const double* __restrict__ fsup,
    const double* __restrict__ frcp, BandStep st, const double* __restrict__ V, int64_t ldv, double* __restrict__ Y,
    double* __restrict__ out, int64_t ldo) {
  constexpr int QS = R * 32 + 4 * R;  // one queue stage: R data rows, then 4 coefficient rows of R
  extern __shared__ double smem[];
  const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* q = smem + (size_t)t * S * QS;
  double* vq = smem + (size_t)G * S * QS;  // [S][R][32] V rows for the backward sums
  const unsigned q_sa = smem_u32(q), vq_sa = smem_u32(vq);
  const int col0 = blockIdx.x * 32;
  const int colc = min(col0 + lane, k - 1);  // dead lanes mirror the last column (Y is padded; out skips them)
  const int64_t dm1 = d > 1 ? d - 1 : 1;
  const double* __restrict__ mu = mult + t * dm1;
  const double* __restrict__ fd = fdiag + (int64_t)t * d;
  const double* __restrict__ fs = fsup + t * dm1;
  const double* __restrict__ fr = frcp + (int64_t)t * d;
  // Y is the kernel's own scratch, blocked per warp (row i of the warp's 32 columns at i * 32):
  // each warp streams one contiguous region instead of 256-byte pieces 8 k bytes apart
  double* __restrict__ y = Y + ((int64_t)blockIdx.x * G + t) * d * 32 + lane;
  const double* __restrict__ v = V + colc;
  const double c = st.c[t];
  const bool residual = st.residual != 0;
  const int nbf = (d + R - 1) / R;

  // ---- forward. Stage b, slot u: row j = bR + u of V, and the coefficients of row i = j - 1
  // (mult_{i-1}, diag_i, sub_{i-1}, super_i), the row completed when v_j arrives. Lane
  // l < 4R copies coefficient kind l / R of slot l % R.
  const int ckind = lane / R, cu = lane % R;
  const int ncoef_f = (residual ? 4 : 1) * R;
  const double* cbase_f = ckind == 0 ? mu + cu - 2 : ckind == 1 ? sdiag + cu - 1 : ckind == 2 ? ssub + cu - 2 : ssup + cu - 1;
  auto issue_fwd = [&](int b) {
    if (b < nbf) {
      const unsigned sa = q_sa + (unsigned)((b % S) * QS * 8);
      const int j0 = b * R;
      if (b >= 1 && j0 + R <= d) {
        const double* p = v + (int64_t)j0 * ldv;
#pragma unroll
        for (int u = 0; u < R; ++u, p += ldv) cp8(sa + (u * 32 + lane) * 8, p);
        if (lane < ncoef_f) cp8(sa + (R * 32 + lane) * 8, cbase_f + j0);
      } else {
#pragma unroll
        for (int u = 0; u < R; ++u)
          if (j0 + u < d) cp8(sa + (u * 32 + lane) * 8, v + (int64_t)(j0 + u) * ldv);
        const int i = j0 + cu - 1;
        if (lane < ncoef_f && i >= 0 && i < d - 1 && (i >= 1 || ckind == 1 || ckind == 3))
          cp8(sa + (R * 32 + lane) * 8, cbase_f + j0);
      }
    }
    cp_commit();  // empty groups keep the wait count uniform
  };
  double prev = 0.0, vim1 = 0.0, vi = 0.0;
  // row i of the forward sweep from (v_{i-1}, v_i, v_{i+1}) and its coefficients
  auto row_fwd = [&](int i, double m, double ad, double as, double ap, double vip1) {
    double r = vi;
    if (residual) {
      double acc = __dmul_rn(ad, vi);
      if (i > 0) acc = __dadd_rn(acc, __dmul_rn(as, vim1));
      if (i + 1 < d) acc = __dadd_rn(acc, __dmul_rn(ap, vip1));
      r = __dmul_rn(c, acc);
    }
    prev = i == 0 ? r : __dsub_rn(r, __dmul_rn(m, prev));
  };
#pragma unroll
  for (int b = 0; b < S - 1; ++b) issue_fwd(b);
  for (int b = 0; b < nbf; ++b) {
    issue_fwd(b + S - 1);
    cp_wait<S - 1>();
    __syncwarp();
    const double* sq = q + (b % S) * QS;
    const int j0 = b * R;
    double* yb = y + (int64_t)(j0 - 1) * 32;
    if (b >= 1 && j0 + R <= d) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const double vj = sq[u * 32 + lane];
        const double* cf = sq + R * 32 + u;
        const double m = cf[0];
        if (residual) {
          const double acc = __dadd_rn(__dadd_rn(__dmul_rn(cf[R], vi), __dmul_rn(cf[2 * R], vim1)),
                                       __dmul_rn(cf[3 * R], vj));
          prev = __dsub_rn(__dmul_rn(c, acc), __dmul_rn(m, prev));
        } else {
          prev = __dsub_rn(vi, __dmul_rn(m, prev));
        }
        __stcg(yb + u * 32, prev);
        vim1 = vi;
        vi = vj;
      }
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int j = j0 + u;
        if (j < d) {
          const double vj = sq[u * 32 + lane];
          if (j > 0) {
            const double* cf = sq + R * 32 + u;
            row_fwd(j - 1, cf[0], residual ? cf[R] : 0.0, residual ? cf[2 * R] : 0.0, residual ? cf[3 * R] : 0.0, vj);
            __stcg(yb + u * 32, prev);
          }
          vim1 = vi;
          vi = vj;
        }
      }
    }
    __syncwarp();  // the slot is refilled by a later issue
  }
  // row d - 1 (kept in the register; Y holds rows 0 .. d - 2)
  row_fwd(d - 1, d > 1 ? mu[d - 2] : 0.0, residual ? sdiag[d - 1] : 0.0, (residual && d > 1) ? ssub[d - 2] : 0.0, 0.0,
          0.0);
  __threadfence_block();  // this thread's Y stores precede its own cp.async reads of them

  // ---- backward. Stage b, slot u: row i = d - 1 - bR - u: Y_i (i < d - 1), super_i, fdiag_i,
  // 1 / fdiag_i in the warp's queue; V_i (all 32 columns, row u copied by warp u % G) in the
  // CTA's ring vq. The back-substituted x_i overwrites Y_i in the slot, where the whole CTA sums
  // it after the barrier; a stage is therefore refilled only after the next barrier.
  const int nbb = nbf;
  const double* cbase_b = (ckind == 0 ? fs : ckind == 1 ? fd : fr) + (d - 1 - cu);
  auto issue_bwd = [&](int b) {
    if (b < nbb) {
      const int slot = b % S;
      const unsigned sa = q_sa + (unsigned)(slot * QS * 8);
      const int i0 = d - 1 - b * R;
      if (b >= 1 && i0 - (R - 1) >= 0) {
        const double* py = y + (int64_t)i0 * 32;
#pragma unroll
        for (int u = 0; u < R; ++u) cp8(sa + (u * 32 + lane) * 8, py - u * 32);
#pragma unroll
        for (int u = 0; u < R; ++u)
          if (u % G == t) cp8(vq_sa + ((slot * R + u) * 32 + lane) * 8, v + (int64_t)(i0 - u) * ldv);
        if (lane < 3 * R) cp8(sa + (R * 32 + lane) * 8, cbase_b - b * R);
      } else {
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const int i = i0 - u;
          if (i >= 0 && i < d - 1) cp8(sa + (u * 32 + lane) * 8, y + (int64_t)i * 32);
          if (u % G == t && i >= 0) cp8(vq_sa + ((slot * R + u) * 32 + lane) * 8, v + (int64_t)i * ldv);
        }
        const int i = i0 - cu;
        if (lane < 3 * R && i >= 0 && (ckind != 0 || i < d - 1)) cp8(sa + (R * 32 + lane) * 8, cbase_b - b * R);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int b = 0; b < S - 1; ++b) issue_bwd(b);
  const bool direct = st.direct != 0;
  double nxt = 0.0;
  for (int b = 0; b < nbb; ++b) {
    cp_wait<S - 2>();  // stages <= b landed (this thread's copies)
    __syncwarp();
    const int slot = b % S;
    double* sq = q + slot * QS;
    const int i0 = d - 1 - b * R;
    if (b >= 1 && i0 - (R - 1) >= 0) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const double* cf = sq + R * 32 + u;
        nxt = div_rcp(__dsub_rn(sq[u * 32 + lane], __dmul_rn(cf[0], nxt)), cf[R], cf[2 * R]);
        sq[u * 32 + lane] = nxt;
      }
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int i = i0 - u;
        if (i >= 0) {
          const double* cf = sq + R * 32 + u;
          nxt = i == d - 1 ? div_rcp(prev, cf[R], cf[2 * R])
                           : div_rcp(__dsub_rn(sq[u * 32 + lane], __dmul_rn(cf[0], nxt)), cf[R], cf[2 * R]);
          sq[u * 32 + lane] = nxt;
        }
      }
    }
    __syncthreads();  // every warp's x rows and the V rows of stage b visible; stage b - 1 drained
    issue_bwd(b + S - 1);
    const double* vs = vq + slot * R * 32;
    for (int o = threadIdx.x; o < R * 32; o += G * 32) {
      const int u = o >> 5, ln = o & 31, i = i0 - u, cc = col0 + ln;
      if (i < 0 || cc >= k) continue;
      const double vv = vs[u * 32 + ln];
      const double* xs = smem + (size_t)slot * QS + u * 32 + ln;  // warp g's x at xs[g * S * QS]
      double acc = 0.0;
      if (direct) {
#pragma unroll
        for (int g = 0; g < G; ++g) acc = __dadd_rn(acc, __dmul_rn(xs[(size_t)g * S * QS], st.w[g]));
      } else {
        for (int qq = 0; qq < st.n_terms; ++qq) {
          const double xv = st.slot[qq] >= 0 ? xs[(size_t)st.slot[qq] * S * QS] : vv;
          acc = __dadd_rn(acc, __dmul_rn(xv, st.w[qq]));
        }
      }
      if (st.add_poly) {
        acc = __dadd_rn(acc, __dmul_rn(st.constant, vv));
        if (st.hybrid) {
          // (A v)_{i-1..i+1} and (A^2 v)_i in TridiagMatrix::matvec order, from V rows i-2..i+2
          auto av_at = [&](int r) {
            double a = __dmul_rn(sdiag[r], V[(int64_t)r * ldv + cc]);
            if (r > 0) a = __dadd_rn(a, __dmul_rn(ssub[r - 1], V[(int64_t)(r - 1) * ldv + cc]));
            if (r + 1 < d) a = __dadd_rn(a, __dmul_rn(ssup[r], V[(int64_t)(r + 1) * ldv + cc]));
            return a;
          };
          const double av = av_at(i);
          double a2v = __dmul_rn(sdiag[i], av);
          if (i > 0) a2v = __dadd_rn(a2v, __dmul_rn(ssub[i - 1], av_at(i - 1)));
          if (i + 1 < d) a2v = __dadd_rn(a2v, __dmul_rn(ssup[i], av_at(i + 1)));
          acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(st.d1, av), __dmul_rn(st.d2, a2v)));
        }
      }
      __stcs(out + (int64_t)i * ldo + cc, acc);
    }
  }
  cp_wait<0>();  // drain (empty) groups before exit
}

// Per-row coefficient records for band_action_bulk_kernel (32 bytes each, so a stage's rows are
// one contiguous bulk copy). Forward record j of system z holds what row i = j - 1 needs when
// v_j arrives: {mult_{i-1}, diag_i, sub_{i-1}, super_i} of the scaled A (0 where undefined).
// Backward record i: {super_i of M_z (0 at i = d - 1), fdiag_i, band_rcp(fdiag_i), 0}.
__global__ void band_pack_records_kernel(int d, int nsys, const double* __restrict__ ssub,
                                         const double* __restrict__ sdiag, const double* __restrict__ ssup,
                                         const double* __restrict__ mult, const double* __restrict__ fdiag,
                                         const double* __restrict__ fsup, const double* __restrict__ frcp,
                                         double4* __restrict__ frec, double4* __restrict__ brec) {
  const int64_t dm1 = d > 1 ? d - 1 : 1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)nsys * d;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int z = (int)(idx / d), j = (int)(idx % d), i = j - 1;
    double4 f;
    f.x = i >= 1 ? mult[z * dm1 + i - 1] : 0.0;
    f.y = i >= 0 ? sdiag[i] : 0.0;
    f.z = i >= 1 ? ssub[i - 1] : 0.0;
    f.w = (i >= 0 && i + 1 < d) ? ssup[i] : 0.0;
    frec[idx] = f;
    double4 b;
    b.x = j + 1 < d ? fsup[z * dm1 + j] : 0.0;
    b.y = fdiag[(int64_t)z * d + j];
    b.z = frcp[(int64_t)z * d + j];
    b.w = 0.0;
    brec[idx] = b;
  }
}

void launch_band_pack_records(int d, int nsys, const double* ssub, const double* sdiag, const double* ssup,
                              const double* mult, const double* fdiag, const double* fsup, const double* frcp,
                              double* frec, double* brec, cudaStream_t s) {
  const int64_t n = (int64_t)nsys * d;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4736));
  band_pack_records_kernel<<<blocks, 256, 0, s>>>(d, nsys, ssub, sdiag, ssup, mult, fdiag, fsup, frcp,
                                                  reinterpret_cast<double4*>(frec), reinterpret_cast<double4*>(brec));
}

// The same fused substep with the queue filled by the bulk-copy engine (cp.async.bulk, completion
// on a per-warp mbarrier per stage): a stage is one copy of the warp's R Y rows (contiguous in the
// blocked layout), one copy of the R coefficient records, and R row copies of V (one per lane,
// 8 * (columns in the strip) bytes each) -- a handful of instructions per stage instead of one
// per row per lane. Needs 16-byte aligned V rows (V aligned, ldv and k even); otherwise the
// host takes band_action_step_kernel.
namespace {
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
}  // namespace

// H shifts per warp (G / H warps per CTA): the warp's shifts share one V stream, one sliding-window
// matvec and one copy schedule, and their H recurrences are independent chains the scheduler can
// interleave. The queue slot of a warp holds [H][R][32] data rows (the forward uses the first R x 32
// for V, the backward one block per shift for Y / x) and [H][R] 4-double records.
template <int G, int H, int S, int R>
constexpr size_t band_bulk_smem() {
  return sizeof(double) * ((size_t)(G / H) * S * (H * R * 32 + H * R * 4) + (size_t)S * R * 32) +
         sizeof(uint64_t) * (G / H) * S;
}

template <int G, int H, int S, int R>
__global__ void __launch_bounds__(G / H * 32) band_action_bulk_kernel(
    int d, int k, const double* __restrict__ ssub, const double* __restrict__ sdiag, const double* __restrict__ ssup,
    const double* __restrict__ mult, const double4* __restrict__ frec, const double4* __restrict__ brec, BandStep st,
    const double* __restrict__ V, int64_t ldv, double* __restrict__ Y, double* __restrict__ out, int64_t ldo) {
  constexpr int NW = G / H;                     // warps per CTA
  constexpr int QS = H * R * 32 + H * R * 4;    // one stage of one warp
  constexpr int REC = H * R * 32;               // records start
  extern __shared__ __align__(128) double smem[];
  // warp index through a shuffle: provably warp-uniform, so the bulk-copy operands derived from it
  // live in uniform registers (no per-lane waterfall around UBLKCP)
  const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  double* q = smem + (size_t)w * S * QS;
  double* vq = smem + (size_t)NW * S * QS;  // [S][R][32] V rows for the backward sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(vq + S * R * 32);
  const unsigned q_sa = smem_u32(q), vq_sa = smem_u32(vq), bar_sa = smem_u32(bars + w * S);
  const int col0 = blockIdx.x * 32, ncols = min(32, k - col0);
  const unsigned row_bytes = 8u * (unsigned)ncols;
  const int64_t dm1 = d > 1 ? d - 1 : 1;
  const int t0 = w * H;  // the warp's first shift
  // shift t's blocked Y region: ((strip * G) + t) * d * 32
  double* __restrict__ yw = Y + ((int64_t)blockIdx.x * G + t0) * d * 32;
  const double* __restrict__ vstrip = V + col0;
  const double4* __restrict__ fr4 = frec + (int64_t)t0 * d;
  const double4* __restrict__ br4 = brec + (int64_t)t0 * d;
  double c[H];
#pragma unroll
  for (int h = 0; h < H; ++h) c[h] = st.c[t0 + h];
  const bool residual = st.residual != 0;
  const int nbf = (d + R - 1) / R;
  if (lane < S) mbar_init(bar_sa + 8 * lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();

  // stage n (forward b = n, backward b = n - nbf) lives in slot n % S, phase parity (n / S) & 1
  auto issue_fwd = [&](int b) {
    if (b >= nbf) return;
    const int slot = b % S;
    const unsigned sa = q_sa + (unsigned)(slot * QS * 8), bar = bar_sa + 8 * slot;
    const int j0 = b * R, nr = min(R, d - j0);
    if (lane == 0) {
      mbar_expect(bar, (unsigned)nr * (row_bytes + 32u * H));
      const double* src = vstrip + (int64_t)j0 * ldv;
      for (int u = 0; u < nr; ++u, src += ldv) bulk_g2s(sa + u * 256, src, row_bytes, bar);
#pragma unroll
      for (int h = 0; h < H; ++h) bulk_g2s(sa + (REC + h * R * 4) * 8, fr4 + (int64_t)h * d + j0, (unsigned)nr * 32u, bar);
    }
  };
  auto issue_bwd = [&](int b) {
    if (b >= nbf) return;
    const int n = nbf + b, slot = n % S;
    const unsigned sa = q_sa + (unsigned)(slot * QS * 8), bar = bar_sa + 8 * slot;
    const int i0 = d - 1 - b * R, base = i0 - (R - 1);  // slot position p holds row base + p
    const int lo = max(base, 0), hi_y = min(i0, d - 2);
    const int ny = max(hi_y - lo + 1, 0), nrec = i0 - lo + 1;
    const bool vrows = b % NW == w;
    if (lane == 0) {
      mbar_expect(bar, H * ((unsigned)ny * 256u + (unsigned)nrec * 32u) + (vrows ? (unsigned)nrec * row_bytes : 0u));
#pragma unroll
      for (int h = 0; h < H; ++h) {
        if (ny > 0)
          bulk_g2s(sa + (h * R * 32 + (lo - base) * 32) * 8, yw + ((int64_t)h * d + lo) * 32, (unsigned)ny * 256u, bar);
        bulk_g2s(sa + (REC + h * R * 4 + (lo - base) * 4) * 8, br4 + (int64_t)h * d + lo, (unsigned)nrec * 32u, bar);
      }
      if (vrows) {
        const double* src = vstrip + (int64_t)lo * ldv;
        for (int p = lo - base; p < R; ++p, src += ldv)
          bulk_g2s(vq_sa + (unsigned)((slot * R + p) * 256), src, row_bytes, bar);
      }
    }
  };

  // ---- forward (slot position u = row j0 + u; record u = the coefficients of row j0 + u - 1)
#pragma unroll
  for (int b = 0; b < S - 1; ++b) issue_fwd(b);
  double prev[H], vim1 = 0.0, vi = 0.0;
#pragma unroll
  for (int h = 0; h < H; ++h) prev[h] = 0.0;
  double* yl = yw + lane;
  for (int b = 0; b < nbf; ++b) {
    issue_fwd(b + S - 1);
    const int slot = b % S;
    mbar_wait(bar_sa + 8 * slot, (unsigned)(b / S) & 1u);
    const double* sq = q + slot * QS;
    const double4* rec = reinterpret_cast<const double4*>(sq + REC);  // rec[h * R + u]
    const int j0 = b * R;
    double* yb = yl + (int64_t)(j0 - 1) * 32;
    if (b >= 1 && j0 + R <= d) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const double vj = sq[u * 32 + lane];
        const double4 c0 = rec[u];
        const double acc =
            residual ? __dadd_rn(__dadd_rn(__dmul_rn(c0.y, vi), __dmul_rn(c0.z, vim1)), __dmul_rn(c0.w, vj)) : 0.0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const double m = h == 0 ? c0.x : rec[h * R + u].x;
          prev[h] = residual ? __dsub_rn(__dmul_rn(c[h], acc), __dmul_rn(m, prev[h])) : __dsub_rn(vi, __dmul_rn(m, prev[h]));
          __stcg(yb + (int64_t)h * d * 32 + u * 32, prev[h]);
        }
        vim1 = vi;
        vi = vj;
      }
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int j = j0 + u;
        if (j < d) {
          const double vj = sq[u * 32 + lane];
          if (j > 0) {
            const int i = j - 1;
            const double4 c0 = rec[u];
            double acc = 0.0;
            if (residual) {
              acc = __dmul_rn(c0.y, vi);
              if (i > 0) acc = __dadd_rn(acc, __dmul_rn(c0.z, vim1));
              acc = __dadd_rn(acc, __dmul_rn(c0.w, vj));  // i + 1 = j < d
            }
#pragma unroll
            for (int h = 0; h < H; ++h) {
              const double r = residual ? __dmul_rn(c[h], acc) : vi;
              prev[h] = i == 0 ? r : __dsub_rn(r, __dmul_rn(rec[h * R + u].x, prev[h]));
              __stcg(yb + (int64_t)h * d * 32 + u * 32, prev[h]);
            }
          }
          vim1 = vi;
          vi = vj;
        }
      }
    }
    __syncwarp();  // every lane is done with the slot before a later issue refills it
  }
  {  // row d - 1 (kept in the register; Y holds rows 0 .. d - 2)
    const int i = d - 1;
    double acc = 0.0;
    if (residual) {
      acc = __dmul_rn(sdiag[i], vi);
      if (i > 0) acc = __dadd_rn(acc, __dmul_rn(ssub[i - 1], vim1));
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double r = residual ? __dmul_rn(c[h], acc) : vi;
      prev[h] = i == 0 ? r : __dsub_rn(r, __dmul_rn(mult[(t0 + h) * dm1 + i - 1], prev[h]));
    }
  }
  fence_proxy_async_global();  // the Y stores above are read back by the bulk copies below
  __syncwarp();

  // ---- backward (slot position p = row base + p, base = i0 - R + 1; the x rows overwrite Y rows
  // in place and are summed by the whole CTA after the barrier)
#pragma unroll
  for (int b = 0; b < S - 1; ++b) issue_bwd(b);
  const bool direct = st.direct != 0;
  double nxt[H];
#pragma unroll
  for (int h = 0; h < H; ++h) nxt[h] = 0.0;
  for (int b = 0; b < nbf; ++b) {
    const int n = nbf + b, slot = n % S;
    mbar_wait(bar_sa + 8 * slot, (unsigned)(n / S) & 1u);
    double* sq = q + slot * QS;
    const double4* rec = reinterpret_cast<const double4*>(sq + REC);
    const int i0 = d - 1 - b * R;
    if (b >= 1 && i0 - (R - 1) >= 0) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int p = R - 1 - u;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const double4 cf = rec[h * R + p];
          double* x = sq + h * R * 32 + p * 32 + lane;
          nxt[h] = div_rcp(__dsub_rn(*x, __dmul_rn(cf.x, nxt[h])), cf.y, cf.z);
          *x = nxt[h];
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int i = i0 - u, p = R - 1 - u;
        if (i >= 0) {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const double4 cf = rec[h * R + p];
            double* x = sq + h * R * 32 + p * 32 + lane;
            nxt[h] = i == d - 1 ? div_rcp(prev[h], cf.y, cf.z)
                                : div_rcp(__dsub_rn(*x, __dmul_rn(cf.x, nxt[h])), cf.y, cf.z);
            *x = nxt[h];
          }
        }
      }
    }
    fence_proxy_async_smem();  // the x rows (generic stores) precede the bulk refill of this slot
    __syncthreads();           // every warp's x rows and stage b's V rows visible; stage b - 1 drained
    issue_bwd(b + S - 1);
    const double* vs = vq + slot * R * 32;
    for (int o = threadIdx.x; o < R * 32; o += NW * 32) {
      const int u = o >> 5, ln = o & 31, i = i0 - u, p = R - 1 - u, cc = col0 + ln;
      if (i < 0 || cc >= k) continue;
      const double vv = vs[p * 32 + ln];
      // shift g's x: warp g / H, block g % H of its slot
      const double* xs = smem + (size_t)slot * QS + p * 32 + ln;
      double acc = 0.0;
      if (direct) {
#pragma unroll
        for (int g = 0; g < G; ++g)
          acc = __dadd_rn(acc, __dmul_rn(xs[(size_t)(g / H) * S * QS + (g % H) * R * 32], st.w[g]));
      } else {
        for (int qq = 0; qq < st.n_terms; ++qq) {
          const int g = st.slot[qq];
          const double xv = g >= 0 ? xs[(size_t)(g / H) * S * QS + (g % H) * R * 32] : vv;
          acc = __dadd_rn(acc, __dmul_rn(xv, st.w[qq]));
        }
      }
      if (st.add_poly) {
        acc = __dadd_rn(acc, __dmul_rn(st.constant, vv));
        if (st.hybrid) {
          auto av_at = [&](int r) {
            double a = __dmul_rn(sdiag[r], V[(int64_t)r * ldv + cc]);
            if (r > 0) a = __dadd_rn(a, __dmul_rn(ssub[r - 1], V[(int64_t)(r - 1) * ldv + cc]));
            if (r + 1 < d) a = __dadd_rn(a, __dmul_rn(ssup[r], V[(int64_t)(r + 1) * ldv + cc]));
            return a;
          };
          const double av = av_at(i);
          double a2v = __dmul_rn(sdiag[i], av);
          if (i > 0) a2v = __dadd_rn(a2v, __dmul_rn(ssub[i - 1], av_at(i - 1)));
          if (i + 1 < d) a2v = __dadd_rn(a2v, __dmul_rn(ssup[i], av_at(i + 1)));
          acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(st.d1, av), __dmul_rn(st.d2, a2v)));
        }
      }
      __stcs(out + (int64_t)i * ldo + cc, acc);
    }
  }
}


#ifndef PF_BAND_STAGES
#define PF_BAND_STAGES 5
#endif
#ifndef PF_BAND_ROWS
#define PF_BAND_ROWS 4
#endif
#ifndef PF_BAND_H
// shifts per warp in the bulk kernel (even shift counts). H = 2 cuts instructions 30 % but halves
// the resident warps; the kernel is latency-bound by its k / 32 x P independent chains, and
// d 8192 k 16384 R8 measured 24.0 ms (H = 2) vs 21.7 ms (H = 1) -- profiles/r01_ncu_band_h2.txt
#define PF_BAND_H 1
#endif

cudaError_t launch_band_action_step(int P, int d, int k, const double* ssub, const double* sdiag, const double* ssup,
                                    const double* mult, const double* fdiag, const double* fsup, const double* frcp,
                                    const double* frec, const double* brec, const BandStep& st, const double* V,
                                    int64_t ldv, double* Y, double* out, int64_t ldo, cudaStream_t s) {
  constexpr int S = PF_BAND_STAGES, R = PF_BAND_ROWS;
  const dim3 grid((k + 31) / 32);
  // bulk copies need 16-byte aligned rows; they win once the grid is at least two CTAs per SM
  // (k 16384: 4.7 vs 5.5 ms a substep), the per-lane queue wins on small grids where each warp's
  // latency chain is the whole story (k 256 / 4096)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool bulk = frec && brec && (reinterpret_cast<uintptr_t>(V) & 15) == 0 && ldv % 2 == 0 && k % 2 == 0 &&
                    (int64_t)grid.x >= 2 * (int64_t)sms;
  switch (P) {
#define PF_BAND_CASE(G)                                                                                           \
  case G:                                                                                                         \
    if (bulk) {                                                                                                   \
      constexpr int H = (G % 2 == 0 && PF_BAND_H == 2) ? 2 : 1;                                                   \
      auto fn = band_action_bulk_kernel<G, H, S, R>;                                                              \
      constexpr size_t smem = band_bulk_smem<G, H, S, R>();                                                       \
      set_smem_attr_once(reinterpret_cast<const void*>(fn), (int)smem);                                           \
      fn<<<grid, G / H * 32, smem, s>>>(d, k, ssub, sdiag, ssup, mult, reinterpret_cast<const double4*>(frec),    \
                                        reinterpret_cast<const double4*>(brec), st, V, ldv, Y, out, ldo);         \
    } else {                                                                                                      \
      auto fn = band_action_step_kernel<G, S, R>;                                                                 \
      constexpr size_t smem = band_step_smem<G, S, R>();                                                          \
      set_smem_attr_once(reinterpret_cast<const void*>(fn), (int)smem);                                           \
      fn<<<grid, G * 32, smem, s>>>(d, k, ssub, sdiag, ssup, mult, fdiag, fsup, frcp, st, V, ldv, Y, out, ldo);   \
    }                                                                                                             \
    break;
    PF_BAND_CASE(1)
    PF_BAND_CASE(2)
    PF_BAND_CASE(3)
    PF_BAND_CASE(4)
    PF_BAND_CASE(5)
    PF_BAND_CASE(6)
    PF_BAND_CASE(7)
    PF_BAND_CASE(8)
    PF_BAND_CASE(9)
    PF_BAND_CASE(10)
    PF_BAND_CASE(11)
    PF_BAND_CASE(12)
#undef PF_BAND_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
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

// Forward elimination with a register window (x[i], x[i+1] partially updated, x[i+2] arriving from
// the RHS): each element receives the same updates in the same order as pentadiag_solve's in-place
// loop (off 2 from row r - 2, then off 1 from row r - 1; f == 0 skipped), without the RHS copy pass
// or read-modify-writes through memory; loads issued R rows ahead. Back substitution keeps
// x[i+1], x[i+2] in registers.
__global__ void __launch_bounds__(128) penta_solve_kernel(int d, int k, const double* __restrict__ W,
                                                          const double* __restrict__ F,
                                                          const double* __restrict__ rhs, int64_t ldr,
                                                          double* __restrict__ X, int64_t ldx) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= k) return;
  constexpr int R = 8;
  double* __restrict__ x = X + col;
  const double* __restrict__ b = rhs + col;
  double x0 = d > 0 ? b[0] : 0.0, x1 = d > 1 ? b[ldr] : 0.0;
  for (int i0 = 0; i0 < d; i0 += R) {
    double nb[R], f0[R], f1[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = i0 + u;
      nb[u] = i + 2 < d ? b[(int64_t)(i + 2) * ldr] : 0.0;
      f0[u] = i < d ? __ldg(F + (int64_t)i * 2) : 0.0;
      f1[u] = i < d ? __ldg(F + (int64_t)i * 2 + 1) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = i0 + u;
      if (i < d) {
        const double xi = x0;
        double x2 = nb[u];
        if (i + 1 < d && f0[u] != 0.0) x1 = __dsub_rn(x1, __dmul_rn(f0[u], xi));
        if (i + 2 < d && f1[u] != 0.0) x2 = __dsub_rn(x2, __dmul_rn(f1[u], xi));
        x[(int64_t)i * ldx] = xi;
        x0 = x1;
        x1 = x2;
      }
    }
  }
  double n1 = 0.0, n2 = 0.0;  // x[i+1], x[i+2] (final)
  for (int i0 = d - 1; i0 >= 0; i0 -= R) {
    double xv[R], w2[R], w3[R], w4[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = i0 - u;
      xv[u] = i >= 0 ? x[(int64_t)i * ldx] : 0.0;
      w2[u] = i >= 0 ? __ldg(W + (int64_t)i * 5 + 2) : 1.0;
      w3[u] = i >= 0 ? __ldg(W + (int64_t)i * 5 + 3) : 0.0;
      w4[u] = i >= 0 ? __ldg(W + (int64_t)i * 5 + 4) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = i0 - u;
      if (i >= 0) {
        double acc = xv[u];
        if (i + 1 < d) acc = __dsub_rn(acc, __dmul_rn(w3[u], n1));
        if (i + 2 < d) acc = __dsub_rn(acc, __dmul_rn(w4[u], n2));
        const double xi = __ddiv_rn(acc, w2[u]);
        x[(int64_t)i * ldx] = xi;
        n2 = n1;
        n1 = xi;
      }
    }
  }
}

}  // namespace pf
