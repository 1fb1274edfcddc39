// The DMMA GEMM tile (one BM x BN output tile of C = alpha A B + beta C + gamma I), shared by the
// batched GEMM kernel (gemm.cu) and the device-scheduled LU (large.cu). Operands are staged with
// cp.async.cg (L2 only) and C is re-read with ld.global.cg: the tile is coherent with data other
// SMs wrote during the same kernel (the persistent LU's tasks).
#pragma once
#include "pf_common.cuh"
#include "pf_kernels.h"

namespace pf {
namespace {

#ifndef PF_GEMM_STAGES
#define PF_GEMM_STAGES 3
#endif
#ifndef PF_GEMM_BK
#define PF_GEMM_BK 32
#endif
#ifndef PF_GEMM_WN
#define PF_GEMM_WN 64
#endif
constexpr int STAGES = PF_GEMM_STAGES;

template <int BM, int BN, int BK>
struct GemmSmem {
  static constexpr int LA = BK + 4;  // A tile row stride (doubles): 32-byte skew
  static constexpr int LB = BN + 4;
  double a[STAGES][BM * LA];
  double b[STAGES][BK * LB];
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BM, int BN, int BK, int NT, bool V16>
__device__ __forceinline__ void load_stage(GemmSmem<BM, BN, BK>& sm, int stage, const GemmParams& p, const double* A,
                                           const double* B, int m0, int n0, int k0) {
  constexpr int LA = GemmSmem<BM, BN, BK>::LA;
  constexpr int LB = GemmSmem<BM, BN, BK>::LB;
  if constexpr (V16) {
#pragma unroll
    for (int it = 0; it < (BM * BK / 2) / NT; ++it) {
      const int idx = threadIdx.x + it * NT;
      const int r = idx / (BK / 2), c = 2 * (idx % (BK / 2));
      const int gr = m0 + r, gc = k0 + c;
      const int bytes = gr < p.m ? (gc + 1 < p.k ? 16 : (gc < p.k ? 8 : 0)) : 0;
      cp_async16(&sm.a[stage][r * LA + c], bytes ? A + (int64_t)gr * p.lda + gc : A, bytes);
    }
#pragma unroll
    for (int it = 0; it < (BK * BN / 2) / NT; ++it) {
      const int idx = threadIdx.x + it * NT;
      const int r = idx / (BN / 2), c = 2 * (idx % (BN / 2));
      const int gr = k0 + r, gc = n0 + c;
      const int bytes = gr < p.k ? (gc + 1 < p.n ? 16 : (gc < p.n ? 8 : 0)) : 0;
      cp_async16(&sm.b[stage][r * LB + c], bytes ? B + (int64_t)gr * p.ldb + gc : B, bytes);
    }
  } else {
#pragma unroll
    for (int it = 0; it < (BM * BK) / NT; ++it) {
      const int idx = threadIdx.x + it * NT;
      const int r = idx / BK, c = idx % BK;
      const int gr = m0 + r, gc = k0 + c;
      const bool ok = gr < p.m && gc < p.k;
      cp_async8(&sm.a[stage][r * LA + c], ok ? A + (int64_t)gr * p.lda + gc : A, ok);
    }
#pragma unroll
    for (int it = 0; it < (BK * BN) / NT; ++it) {
      const int idx = threadIdx.x + it * NT;
      const int r = idx / BN, c = idx % BN;
      const int gr = k0 + r, gc = n0 + c;
      const bool ok = gr < p.k && gc < p.n;
      cp_async8(&sm.b[stage][r * LB + c], ok ? B + (int64_t)gr * p.ldb + gc : B, ok);
    }
  }
}

}  // namespace

// warps (BM / WM) (M) x (BN / WN) (N), each a WM x WN tile of (WM / 8) x (WN / 8) DMMA tiles.
// One BM x BN output tile (tile index `tile` of matrix bz).
template <int BM, int BN, int BK, int WM, int WN, bool V16>
__device__ __forceinline__ void gemm_tile(const GemmParams& p, GemmSmem<BM, BN, BK>& sm, int bz, int tile,
                                          int tiles_n) {
  constexpr int LA = GemmSmem<BM, BN, BK>::LA;
  constexpr int LB = GemmSmem<BM, BN, BK>::LB;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int MI = WM / 8;      // DMMA tiles down
  constexpr int NJ = WN / 8;      // DMMA tiles across
  constexpr int WCOLS = BN / WN;  // warps across
  const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
  const double* A = p.A + (int64_t)bz * p.strideA;
  const double* B = p.B + (int64_t)bz * p.strideB;
  double* C = p.C + (int64_t)bz * p.strideC;
  if (p.jmask != nullptr && p.step >= p.jmask[bz]) {
    if (p.pass != nullptr) {
      const double* src = p.pass + (int64_t)bz * p.strideC;
      for (int idx = threadIdx.x; idx < BM * BN; idx += NT) {
        const int r = m0 + idx / BN, c = n0 + idx % BN;
        if (r < p.m && c < p.n) C[(int64_t)r * p.ldc + c] = src[(int64_t)r * p.ldc + c];
      }
    }
    return;
  }
  const int lane = lane_id(), warp = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wm = WM * (warp / WCOLS), wn = WN * (warp % WCOLS);

  double acc[MI][NJ][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  const int nk = (p.k + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage<BM, BN, BK, NT, V16>(sm, s, p, A, B, m0, n0, s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) load_stage<BM, BN, BK, NT, V16>(sm, nxt % STAGES, p, A, B, m0, n0, nxt * BK);
    cp_async_commit();
    const double* as = sm.a[kt % STAGES];
    const double* bs = sm.b[kt % STAGES];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NJ];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = as[(wm + 8 * mi + g) * LA + kk + t];
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) bf[nj] = bs[(kk + t) * LB + wn + 8 * nj + g];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
    }
  }
  cp_async_wait<0>();

  // epilogue: alpha * acc (+ beta * C) (+ gamma on the diagonal)
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = m0 + wm + 8 * mi + g, c = n0 + wn + 8 * nj + 2 * t + e;
        if (r < p.m && c < p.n) {
          double v = p.alpha == 1.0 ? acc[mi][nj][e] : __dmul_rn(p.alpha, acc[mi][nj][e]);
          double* dst = C + (int64_t)r * p.ldc + c;
          if (p.beta != 0.0) {
            const double cv = __ldcg(dst);
            v = __dadd_rn(p.beta == 1.0 ? cv : __dmul_rn(p.beta, cv), v);
          }
          if (p.gamma != 0.0 && r == c) v = __dadd_rn(v, p.gamma);
          *dst = v;
          if (p.sd_d != nullptr) {
            const int64_t o = (int64_t)bz * p.strideC + (int64_t)r * p.ldc + c;
            const double cv = __ldcg(p.sd_ref + o);
            p.sd_d[o] = cv - v;
            p.sd_e[o] = cv + v;
          }
        }
      }
}

}  // namespace pf
