// K5: batched FP64 GEMM on DMMA.8x8x4, C = alpha * A B + beta * C + gamma * I (row-major).
//
// Replaces DenseMatrix::mul (proj/core/src/dense.cpp:17-29) for the squaring chain, B^2, the
// phi1 / cos-sin recurrences, B V, and every off-diagonal update of the large-n LU / triangular
// solves. CTA tile BM x BN x BK: 64 x 64 x 16 (4 warps of 32 x 32, four CTAs = 16 DMMA warps per SM)
// for every shape -- measured faster than 128 x 128 x 32 (8 warps of 32 x 64, one CTA per SM) and
// 128 x 64 x 16 at every size (see launch_gemm); 3-stage cp.async pipeline, 16-byte
// copies when the operands allow it (8-byte copies with zero fill otherwise: any shape / leading
// dimension is legal).
#include <algorithm>
#include <cstdlib>

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
          if (p.beta != 0.0) v = __dadd_rn(p.beta == 1.0 ? *dst : __dmul_rn(p.beta, *dst), v);
          if (p.gamma != 0.0 && r == c) v = __dadd_rn(v, p.gamma);
          *dst = v;
        }
      }
}

template <int BM, int BN, int BK, int WM, int WN, int MINB, bool V16>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB) gemm_kernel(GemmParams p, int tiles_n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GemmSmem<BM, BN, BK>& sm = *reinterpret_cast<GemmSmem<BM, BN, BK>*>(smem_raw);
  if (p.max_sms <= 0) {
    gemm_tile<BM, BN, BK, WM, WN, V16>(p, sm, blockIdx.y, blockIdx.x, tiles_n);
    return;
  }
  // persistent: tiles of all matrices, strided by the grid
  const int tiles = ((p.m + BM - 1) / BM) * tiles_n;
  const int64_t total = (int64_t)tiles * p.batch;
  for (int64_t L = blockIdx.x; L < total; L += gridDim.x) {
    gemm_tile<BM, BN, BK, WM, WN, V16>(p, sm, (int)(L / tiles), (int)(L % tiles), tiles_n);
    __syncthreads();  // the next tile's prologue refills the stage buffers
  }
}

namespace {
template <int BM, int BN, int BK, int WM, int WN, int MINB, bool V16>
void launch_tile(const GemmParams& p, cudaStream_t stream) {
  const int smem = (int)sizeof(GemmSmem<BM, BN, BK>);
  set_smem_attr_once(reinterpret_cast<const void*>(gemm_kernel<BM, BN, BK, WM, WN, MINB, V16>), smem);
  const int tiles_m = (p.m + BM - 1) / BM, tiles_n = (p.n + BN - 1) / BN;
  dim3 grid(tiles_m * tiles_n, p.batch);
  if (p.max_sms > 0) {
    const int64_t total = (int64_t)tiles_m * tiles_n * p.batch;
    grid = dim3((unsigned)std::min<int64_t>(total, (int64_t)p.max_sms * MINB), 1);
  }
  gemm_kernel<BM, BN, BK, WM, WN, MINB, V16><<<grid, (BM / WM) * (BN / WN) * 32, smem, stream>>>(p, tiles_n);
}

template <int BM, int BN, int BK, int WM, int WN, int MINB>
void launch_v(const GemmParams& p, bool v16, cudaStream_t stream) {
  if (v16)
    launch_tile<BM, BN, BK, WM, WN, MINB, true>(p, stream);
  else
    launch_tile<BM, BN, BK, WM, WN, MINB, false>(p, stream);
}
}  // namespace

void launch_gemm_chunk(const GemmParams& p, cudaStream_t stream);

// grid.y carries the batch (at most 65535 per launch): larger batches run as several launches on
// consecutive slices of the matrices and of the per-matrix step masks.
void launch_gemm(const GemmParams& p, cudaStream_t stream) {
  constexpr int kMaxGridY = 65535;
  if (p.max_sms > 0 || p.batch <= kMaxGridY) {
    launch_gemm_chunk(p, stream);
    return;
  }
  for (int b0 = 0; b0 < p.batch; b0 += kMaxGridY) {
    GemmParams q = p;
    q.batch = std::min(kMaxGridY, p.batch - b0);
    q.A = p.A + (int64_t)b0 * p.strideA;
    q.B = p.B + (int64_t)b0 * p.strideB;
    q.C = p.C + (int64_t)b0 * p.strideC;
    if (p.jmask) q.jmask = p.jmask + b0;
    if (p.pass) q.pass = p.pass + (int64_t)b0 * p.strideC;
    launch_gemm_chunk(q, stream);
  }
}

void launch_gemm_chunk(const GemmParams& p, cudaStream_t stream) {
  // 16-byte copies need even leading dimensions / batch strides and 16-byte aligned bases
  const bool v16 = ((p.lda | p.ldb | p.strideA | p.strideB) & 1) == 0 &&
                   ((reinterpret_cast<uintptr_t>(p.A) | reinterpret_cast<uintptr_t>(p.B)) & 15) == 0;
  // 64 x 64 x 16 tiles, 4 warps of 32 x 32, four CTAs (16 DMMA warps) per SM for every shape: the
  // occupancy beats the larger tiles' operand reuse everywhere measured (tools/large_timing.py,
  // profiles/r01_gemm_sweep.txt): 2048^3 30.8 vs 27.2 TF/s, 8192^3 32.7 vs 32.1, cfg5 83.9 vs
  // 98.2 ms, 8 x 4096^2 LU 18.1 vs 19.8 ms. PF_GEMM_FORCE=1 / 3 selects the 128 x 64 / 128 x 128
  // tiles for A/B runs. (Every variant accumulates each element in the same k order.)
  static const int force = std::getenv("PF_GEMM_FORCE") ? std::atoi(std::getenv("PF_GEMM_FORCE")) : 0;
  if (force == 1) {
    launch_v<128, 64, 16, 32, 32, 2>(p, v16, stream);
  } else if (force == 3) {
    launch_v<128, 128, PF_GEMM_BK, 32, PF_GEMM_WN, 1>(p, v16, stream);
  } else {
    launch_v<64, 64, 16, 32, 32, 4>(p, v16, stream);
  }
}

}  // namespace pf
