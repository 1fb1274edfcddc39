// LU variants measured against small_eval.cu's lu_block by tools/bench_lu.cu (not used by the
// library). Staging for the variants lives in LuExtra, placed after Smem in dynamic shared memory.
#pragma once

namespace pf {
namespace {

struct LuExtra {
  double tinv[2][NB * (NB + 4)];  // U_kk^-1, L_kk^-1 of the current diagonal block
  double rowbuf[2][NB];           // pivot-row broadcast (double buffered)
};
constexpr int TS = NB + 4;  // row stride of tinv: conflict-free DMMA fragment loads

// 1/x: MUFU.RCP64H seed r0 (relative error e0 < 2^-20) and one cubic step r0 (1 + e + e^2),
// e = 1 - x r0: error e0^3 plus rounding, three dependent FMAs instead of fast_rcp's four.
__device__ __forceinline__ double rcp_cubic(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Same factorization, pivot row broadcast through shared memory: a 64-bit SHFL costs ~9 issue
// cycles per warp against ~2.3 per double for a broadcast LDS.128 (tools/probe_latency.cu). The
// pivot value alone still goes by SHFL so its reciprocal starts before the row lands.
__device__ __forceinline__ void factor_diag_block_sm(Smem& sm, LuExtra& ex, int k0) {
  const int lane = lane_id();
  const bool row = lane < NB;
  double d[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) d[c] = row ? sm.S[(k0 + lane) * LS + k0 + c] : 0.0;
#pragma unroll
  for (int m = 0; m < NB; ++m) {
    const double piv = __shfl_sync(FULL, d[m], m);
    double* rb = ex.rowbuf[m & 1];
    const int c0 = (m + 1) & ~1;
    if (lane == m) {
#pragma unroll
      for (int c = c0; c < NB; c += 2) *reinterpret_cast<double2*>(&rb[c]) = make_double2(d[c], d[c + 1]);
    }
    const double inv = rcp_cubic(piv);
    __syncwarp();
    double u[NB];
#pragma unroll
    for (int c = c0; c < NB; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(&rb[c]);
      u[c] = v.x;
      u[c + 1] = v.y;
    }
    if (lane > m && row) {
      const double dm = d[m];
      const double f = dm * inv;
      d[m] = f;
#pragma unroll
      for (int c = m + 1; c < NB; ++c) d[c] = fma(-f, u[c], d[c]);
    }
  }
  if (row) {
#pragma unroll
    for (int c = 0; c < NB; c += 2)
      *reinterpret_cast<double2*>(&sm.S[(k0 + lane) * LS + k0 + c]) = make_double2(d[c], d[c + 1]);
  }
}

// The lead warp's chain step: the 16x16 diagonal block D at (k0, k0) (lane i < 16 holds row i) is
// factored D = L U without exchanges and only its triangular inverses leave the warp: U^-1 into
// tinv[0], L^-1 into tinv[1] (S is not written; the solve's D^-1 is formed from tinv later).
//  - factor: the next pivot's update is formed as fma(-(d_m u), 1/p, d) so the chain per pivot is
//    shuffle + reciprocal (rcp_cubic) + one FMA;
//  - inverses: both by row sweeps in one pass: lanes 16-31 the rows of L^-1 (forward over m),
//    lanes 0-15 the rows of U'^-1, U' = diag(1/p) U unit upper (backward over m, run as a forward
//    sweep in reversed indices), one shuffle + FMA per step; U^-1 = U'^-1 diag(1/p).
__device__ __forceinline__ void factor_invert_block(Smem& sm, LuExtra& ex, int k0) {
  const int lane = lane_id();
  const bool row = lane < NB;
  double d[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) d[c] = row ? sm.S[(k0 + lane) * LS + k0 + c] : 0.0;
  double myinv = 0.0;
#pragma unroll
  for (int m = 0; m < NB; ++m) {
    const double piv = __shfl_sync(FULL, d[m], m);
    double u[NB];
#pragma unroll
    for (int c = m + 1; c < NB; ++c) u[c] = __shfl_sync(FULL, d[c], m);
    const double inv = rcp_cubic(piv);
    if (lane == m) myinv = inv;
    if (lane > m && row) {
      const double dm = d[m];
      if (m + 1 < NB) {
        const double pm = dm * u[m + 1];
        d[m + 1] = fma(-pm, inv, d[m + 1]);  // the next pivot first
      }
      const double f = dm * inv;
      d[m] = f;
#pragma unroll
      for (int c = m + 2; c < NB; ++c) d[c] = fma(-f, u[c], d[c]);
    }
  }
  // lane row index r (reversed for the U half) and the sweep coefficients coef[s]
  const bool up = row;
  const int r = up ? NB - 1 - lane : lane - NB;
  double coef[NB], w[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double lrow = __shfl_sync(FULL, d[c], lane & (NB - 1));  // L[lane - 16][c] for the lower half
    coef[c] = up ? d[NB - 1 - c] * myinv : lrow;
    w[c] = (c == r) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int s = 0; s < NB - 1; ++s) {
    const int src = up ? NB - 1 - s : NB + s;
    double rw[NB];
#pragma unroll
    for (int c = 0; c <= s; ++c) rw[c] = __shfl_sync(FULL, w[c], src);
    if (r > s) {
#pragma unroll
      for (int c = 0; c <= s; ++c) w[c] = fma(-coef[s], rw[c], w[c]);
    }
  }
  // U half: column 15 - c of U^-1 row `lane` = w[c] / p_{15-c}
  double* dst = up ? &ex.tinv[0][lane * TS + NB - 1] : &ex.tinv[1][(lane - NB) * TS];
  const int ds = up ? -1 : 1;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double sc = __shfl_sync(FULL, myinv, NB - 1 - c);
    dst[c * ds] = up ? w[c] * sc : w[c];
  }
}

// Lt21 block (rows R0 .. R0+15) = (A21 U_kk^-1) L_kk^-1 by one warp: two K = 16 DMMA products, the
// intermediate moved from C to A fragments by quad shuffles.
__device__ __forceinline__ void panel_block(Smem& sm, LuExtra& ex, int k0, int R0) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  double p[2][2][2] = {};
#pragma unroll
  for (int kk = 0; kk < NB; kk += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = sm.S[(R0 + 8 * mi + g) * LS + k0 + kk + t];
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) bf[nj] = ex.tinv[0][(kk + t) * TS + 8 * nj + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) dmma(p[mi][nj], af[mi], bf[nj]);
  }
  double q[2][2][2] = {};
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    // A element (8mi + g, 4ks + t) sits in C tile nj = ks >> 1, lane (g, (4 (ks & 1) + t) >> 1), e = t & 1
    const int src = g * 4 + ((4 * (ks & 1) + t) >> 1);
    double af[2], bf[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double v0 = __shfl_sync(FULL, p[mi][ks >> 1][0], src);
      const double v1 = __shfl_sync(FULL, p[mi][ks >> 1][1], src);
      af[mi] = (t & 1) ? v1 : v0;
    }
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) bf[nj] = ex.tinv[1][(4 * ks + t) * TS + 8 * nj + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) dmma(q[mi][nj], af[mi], bf[nj]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
      *reinterpret_cast<double2*>(&sm.S[(R0 + 8 * mi + g) * LS + k0 + 8 * nj + 2 * t]) =
          make_double2(q[mi][nj][0], q[mi][nj][1]);
}

// D_k^-1 = U_kk^-1 L_kk^-1 into the diagonal block by one warp.
__device__ __forceinline__ void diag_inverse_product(Smem& sm, LuExtra& ex, int k0) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  double acc[2][2][2] = {};
#pragma unroll
  for (int kk = 0; kk < NB; kk += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = ex.tinv[0][(8 * mi + g) * TS + kk + t];
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) bf[nj] = ex.tinv[1][(kk + t) * TS + 8 * nj + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
      *reinterpret_cast<double2*>(&sm.S[(k0 + 8 * mi + g) * LS + k0 + 8 * nj + 2 * t]) =
          make_double2(acc[mi][nj][0], acc[mi][nj][1]);
}

}  // namespace
}  // namespace pf
