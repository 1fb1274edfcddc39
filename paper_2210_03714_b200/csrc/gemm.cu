// K5: batched FP64 GEMM on DMMA.8x8x4, C = alpha * A B + beta * C + gamma * I (row-major).
//
// Replaces DenseMatrix::mul (proj/core/src/dense.cpp:17-29) for the squaring chain, B^2, the
// phi1 / cos-sin recurrences, B V, and every off-diagonal update of the large-n LU / triangular
// solves. launch_gemm_chunk takes the TMA-staged kernel of gemm_tma.cu wherever the operands allow
// it (16-byte aligned bases, even leading dimensions / batch strides); this file's cp.async kernel
// covers the rest and the persistent (SM-capped) mode: CTA tile 64 x 64 x 16 (4 warps of 32 x 32,
// four CTAs = 16 DMMA warps per SM), 3-stage cp.async pipeline, 16-byte copies when the operands
// allow it (8-byte copies with zero fill otherwise: any shape / leading dimension is legal).
#include <algorithm>
#include <cstdlib>

#include "pf_common.cuh"
#include "pf_kernels.h"

#include "gemm_tile.cuh"

namespace pf {

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
    if (p.sd_d) {
      q.sd_ref = p.sd_ref + (int64_t)b0 * p.strideC;
      q.sd_d = p.sd_d + (int64_t)b0 * p.strideC;
      q.sd_e = p.sd_e + (int64_t)b0 * p.strideC;
    }
    launch_gemm_chunk(q, stream);
  }
}

bool launch_gemm_tma(const GemmParams& p, cudaStream_t stream);  // gemm_tma.cu

void launch_gemm_chunk(const GemmParams& p, cudaStream_t stream) {
  if (launch_gemm_tma(p, stream)) return;  // TMA staging wherever the operands allow it
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
