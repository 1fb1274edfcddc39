// K5: batched FP64 GEMM on DMMA.8x8x4, C = alpha * A B + beta * C + gamma * I (row-major).
//
// Replaces DenseMatrix::mul (proj/core/src/dense.cpp:17-29) for the squaring chain, B^2, the
// phi1 / cos-sin recurrences and B V. CTA tile 128 x 128 x 16, 8 warps (4 x 2) of 32 x 64,
// 3-stage cp.async pipeline; 8-byte async copies with zero fill make any shape / leading
// dimension legal (FP64 rows are only 8-byte aligned in general).
#include "pf_common.cuh"
#include "pf_kernels.h"

namespace pf {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 3, NT = 256;
constexpr int LA = BK + 4;  // A tile row stride (doubles)
constexpr int LB = BN + 4;  // B tile row stride

struct GemmSmem {
  double a[STAGES][BM * LA];
  double b[STAGES][BK * LB];
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void load_stage(GemmSmem& sm, int stage, const GemmParams& p, const double* A,
                                           const double* B, int m0, int n0, int k0) {
  // A tile: BM x BK = 2048 doubles, 8 per thread
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

}  // namespace

__global__ void __launch_bounds__(NT, 1) gemm_kernel(GemmParams p, int tiles_n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GemmSmem& sm = *reinterpret_cast<GemmSmem*>(smem_raw);
  const int bz = blockIdx.y;
  const int m0 = (blockIdx.x / tiles_n) * BM, n0 = (blockIdx.x % tiles_n) * BN;
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
  const int wm = 32 * (warp >> 1), wn = 64 * (warp & 1);

  double acc[4][8][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  const int nk = (p.k + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(sm, s, p, A, B, m0, n0, s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) load_stage(sm, nxt % STAGES, p, A, B, m0, n0, nxt * BK);
    cp_async_commit();
    const double* as = sm.a[kt % STAGES];
    const double* bs = sm.b[kt % STAGES];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[8];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = as[(wm + 8 * mi + g) * LA + kk + t];
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) bf[nj] = bs[(kk + t) * LB + wn + 8 * nj + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 8; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
    }
  }
  cp_async_wait<0>();

  // epilogue: alpha * acc (+ beta * C) (+ gamma on the diagonal)
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 8; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = m0 + wm + 8 * mi + g, c = n0 + wn + 8 * nj + 2 * t + e;
        if (r < p.m && c < p.n) {
          double v = p.alpha == 1.0 ? acc[mi][nj][e] : __dmul_rn(p.alpha, acc[mi][nj][e]);
          double* dst = C + (int64_t)r * p.ldc + c;
          if (p.beta != 0.0) v = __dadd_rn(p.beta == 1.0 ? *dst : __dmul_rn(p.beta, *dst), v);
          if (p.gamma != 0.0 && r == c) v = __dadd_rn(v, p.gamma);
          *dst = v;
        }
      }
}

void launch_gemm(const GemmParams& p, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GemmSmem));
    configured = true;
  }
  const int tiles_m = (p.m + BM - 1) / BM, tiles_n = (p.n + BN - 1) / BN;
  dim3 grid(tiles_m * tiles_n, p.batch);
  gemm_kernel<<<grid, NT, sizeof(GemmSmem), stream>>>(p, tiles_n);
}

}  // namespace pf
