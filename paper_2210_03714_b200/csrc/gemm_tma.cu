// K5 with TMA operand staging: the batched FP64 DMMA GEMM of gemm.cu (64 x 64 x 16 CTA tile, 4 warps
// of 32 x 32, four CTAs per SM), with the A / B tiles moved by the tensor-memory accelerator
// (cp.async.bulk.tensor, 128-byte swizzle) instead of per-thread cp.async copies.
//
// Why: with the operands in shared memory the k-loop alone runs at the DMMA peak
// (tools/probe_gemm_inner.cu: 37.0 TF/s), while the cp.async kernel reaches 32.0 TF/s at 4096^3 --
// and the same 31.2 when every copy hits L2 (tools/probe_gemm_pipe.cu, lda = ldb = 0). The loss is
// the copy instructions, their address arithmetic and the per-stage group waits, not the memory
// system. Here one thread issues five bulk copies per stage; completion is an mbarrier transaction
// count, and stage reuse is an "empty" mbarrier with one arrival per warp (no CTA-wide barrier).
//
// Bank conflicts. TMA writes dense, swizzled boxes: A box = 64 rows x 16 k (128-byte rows), B = four
// boxes of 16 k-rows x 16 columns. The 16-byte chunk c of row r sits at chunk c ^ (r & 7). Each
// DMMA of a 16-wide k tile takes the k set {s', s'+1, s'+4, s'+5} (s' = 2 (s & 1) + 8 (s >> 1),
// s = 0..3; lane t supplies k = s' + (t & 1) + 4 (t >> 1)) instead of 4 consecutive k: then both the
// A and the B fragment loads of a warp touch every bank exactly twice (two wavefronts, the minimum
// for 256 bytes) -- in the full-warp view. 8-byte loads are served per half-warp, and there each
// set still costs 2 wavefronts (ncu: 269M bank conflicts at 4096^3). The conflict-free sets
// {0, 3, 13, 14} ^ {0, 1, 4, 5} (distinct (bit 3, bit 0) and (bit 2, bit 1) of k over the lanes t)
// bring that to 1.2M but run slower, measured back to back: 34.3 / 35.2 / 27.7 TF/s vs 34.7 / 35.5 /
// 29.1 at 4096^3 / 8192^3 / 16384 x 64 x 16384 -- shared-memory bandwidth is not the limiter here.
// Every element still accumulates its k products in one fixed order.
//
// Stages (tools/large_timing.py gemm, PF_TMA_STAGES / PF_TMA_MINB builds): 2 stages x 4 CTAs per SM
// 34.7 / 35.5 / 32.5 TF/s at 4096^3 / 8192^3 / 2048^3; 3 x 4: 34.5 / 35.2 / 32.5; 4 x 3: 34.0 / 35.0 /
// 31.7; 5 x 2: 33.5 / 33.7 / 28.6; 2 x 5 (102 registers, spills): 32.8 / 33.1. Four resident CTAs
// (16 DMMA warps per SM) hide the copy latency; deeper rings only cost occupancy -- also for the
// LU recursion's short-k products on grids under one wave (a 4-stage ring there: 8 x 2048^2 LU
// 3.57 vs 3.47 ms).
//
// Edges: the tensor maps cover the true m, n, k (out-of-range box elements are zero-filled), so any
// shape is legal; the host takes this path when the bases are 16-byte aligned and the leading
// dimensions / batch strides are multiples of 2 doubles (otherwise gemm.cu's cp.async kernel).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "pf_common.cuh"
#include "pf_kernels.h"
#include "tma_util.cuh"

namespace pf {
namespace {

#ifndef PF_TMA_STAGES
#define PF_TMA_STAGES 2
#endif
#ifndef PF_TMA_MINB
#define PF_TMA_MINB 4
#endif
constexpr int TBM = 64, TBN = 64, TBK = 16, TSTAGES = PF_TMA_STAGES;
constexpr int A_BYTES = TBM * TBK * 8;  // 8 KB
constexpr int B_BYTES = TBK * TBN * 8;  // 8 KB (four 2 KB boxes)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;

struct TmaMaps {
  CUtensorMap a;  // dims {k, m, batch}, box {16, 64, 1}
  CUtensorMap b;  // dims {n, k, batch}, box {16, 16, 1}
};

__global__ void __launch_bounds__(128, PF_TMA_MINB) gemm_tma_kernel(const __grid_constant__ TmaMaps maps, GemmParams p,
                                                          int tiles_n) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // 1024-byte alignment for the 128-byte swizzle pattern
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + TSTAGES * STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  const int bz = blockIdx.y, tile = blockIdx.x;
  const int m0 = (tile / tiles_n) * TBM, n0 = (tile % tiles_n) * TBN;
  double* C = p.C + (int64_t)bz * p.strideC;
  if (p.jmask != nullptr && p.step >= p.jmask[bz]) {
    if (p.pass != nullptr) {
      const double* src = p.pass + (int64_t)bz * p.strideC;
      for (int idx = threadIdx.x; idx < TBM * TBN; idx += blockDim.x) {
        const int r = m0 + idx / TBN, c = n0 + idx % TBN;
        if (r < p.m && c < p.n) C[(int64_t)r * p.ldc + c] = src[(int64_t)r * p.ldc + c];
      }
    }
    return;
  }
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wm = 32 * (warp >> 1), wn = 32 * (warp & 1);
  const unsigned base = su32(tsm), fullb = su32(full), emptyb = su32(empty);
  // split-K: this CTA's k tiles [kb, ke) (gridDim.z splits)
  const int nk_all = (p.k + TBK - 1) / TBK;
  const int per = (nk_all + gridDim.z - 1) / gridDim.z;
  const int kb = blockIdx.z * per, ke = min(nk_all, kb + per);
  const int nk = max(ke - kb, 0);
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mb_init(fullb + 8 * s, 1);
      mb_init(emptyb + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.b)) : "memory");
  }
  __syncthreads();
  auto issue = [&](int kt) {
    const int s = kt % TSTAGES;
    const unsigned sa = base + s * STAGE_BYTES, sb = sa + A_BYTES, bar = fullb + 8 * s;
    mb_expect(bar, STAGE_BYTES);
    tma3(sa, &maps.a, (kb + kt) * TBK, m0, bz, bar);
#pragma unroll
    for (int q = 0; q < 4; ++q) tma3(sb + q * 2048, &maps.b, n0 + 16 * q, (kb + kt) * TBK, bz, bar);
  };
  if (tid == 0)
    for (int kt = 0; kt < TSTAGES - 1 && kt < nk; ++kt) issue(kt);

  // per-lane fragment offsets (bytes within a stage) for the four k sets of a 16-wide tile
  unsigned offA[4], offB[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int kt_ = 2 * (s & 1) + 8 * (s >> 1) + (t & 1) + 4 * (t >> 1);  // this lane's k
    offA[s] = (unsigned)((wm + g) * 128 + ((((kt_ >> 1) ^ g) & 7) << 4) + ((kt_ & 1) << 3));
    offB[s] = (unsigned)(A_BYTES + (wn / 16) * 2048 + kt_ * 128 + ((((g >> 1) ^ (kt_ & 7)) & 7) << 4) + ((g & 1) << 3));
  }
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TSTAGES;
    const unsigned use = (unsigned)(kt / TSTAGES) & 1u;
    if (tid == 0) {
      const int nxt = kt + TSTAGES - 1;
      if (nxt < nk) {
        // the stage nxt refills was consumed at iteration nxt - TSTAGES (= kt - 1): all 4 warps arrived
        if (nxt >= TSTAGES) mb_wait(emptyb + 8 * (nxt % TSTAGES), (unsigned)((nxt / TSTAGES) - 1) & 1u);
        issue(nxt);
      }
    }
    mb_wait(fullb + 8 * s, use);
    const unsigned char* sp = tsm + s * STAGE_BYTES;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = *reinterpret_cast<const double*>(sp + offA[ks] + mi * 1024);
#pragma unroll
      for (int nj = 0; nj < 4; ++nj)
        bf[nj] = *reinterpret_cast<const double*>(sp + ((offB[ks] + (nj >> 1) * 2048) ^ ((nj & 1) << 6)));
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
    }
    __syncwarp();
    if (lane == 0) mb_arrive(emptyb + 8 * s);
  }

  if (gridDim.z > 1) {  // split-K: the raw partial product; splitk_reduce_kernel finishes
    double* w = p.split_ws + ((int64_t)blockIdx.z * p.batch + bz) * p.m * p.n;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int nj = 0; nj < 4; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = m0 + wm + 8 * mi + g, c = n0 + wn + 8 * nj + 2 * t + e;
          if (r < p.m && c < p.n) w[(int64_t)r * p.n + c] = acc[mi][nj][e];
        }
    return;
  }
  // epilogue: alpha * acc (+ beta * C) (+ gamma on the diagonal), as gemm_tile
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj)
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    cudaGetLastError();
  });
  return fn;
}

bool encode(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint64_t batch, int64_t ld,
            int64_t stride, unsigned box_inner, unsigned box_outer) {
  const auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {inner, outer, batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)(batch > 1 ? stride : ld * (int64_t)outer) * 8};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C = alpha (sum of the split partials, ascending split) (+ beta C) (+ gamma I): gemm_tile's epilogue
__global__ void splitk_reduce_kernel(GemmParams p, int splits) {
  const int bz = blockIdx.y;
  const int64_t mn = (int64_t)p.m * p.n;
  // rows over blockIdx.x / threadIdx.y, columns over threadIdx.x (no 64-bit index division)
  for (int r = blockIdx.x * blockDim.y + threadIdx.y; r < p.m; r += gridDim.x * blockDim.y)
    for (int c = threadIdx.x; c < p.n; c += blockDim.x) {
    const int64_t idx = (int64_t)r * p.n + c;
    double a = p.split_ws[(int64_t)bz * mn + idx];
    for (int z = 1; z < splits; ++z) a = __dadd_rn(a, p.split_ws[((int64_t)z * p.batch + bz) * mn + idx]);
    double v = p.alpha == 1.0 ? a : __dmul_rn(p.alpha, a);
    double* dst = p.C + (int64_t)bz * p.strideC + (int64_t)r * p.ldc + c;
    if (p.beta != 0.0) {
      const double cv = *dst;
      v = __dadd_rn(p.beta == 1.0 ? cv : __dmul_rn(p.beta, cv), v);
    }
    if (p.gamma != 0.0 && r == c) v = __dadd_rn(v, p.gamma);
    *dst = v;
    }
}

}  // namespace

bool make_tma_map(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint64_t batch, int64_t ld,
                  int64_t stride, unsigned box_inner, unsigned box_outer) {
  return encode(map, base, inner, outer, batch, ld, stride, box_inner, box_outer);
}

size_t gemm_tma_smem_bytes() { return TSTAGES * STAGE_BYTES + 2 * TSTAGES * 8 + 1024; }

// true: launched on the TMA path; false: not applicable (the caller runs the cp.async kernel)
bool launch_gemm_tma(const GemmParams& p, cudaStream_t stream) {
  static const bool off = std::getenv("PF_GEMM_TMA") != nullptr && std::atoi(std::getenv("PF_GEMM_TMA")) == 0;
  if (off || p.max_sms > 0 || p.m <= 0 || p.n <= 0 || p.k <= 0) return false;
  const auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!al(p.A) || !al(p.B) || ((p.lda | p.ldb) & 1) || p.lda < p.k || p.ldb < p.n) return false;
  if (p.batch > 1 && (((p.strideA | p.strideB) & 1) || p.strideA <= 0 || p.strideB <= 0)) return false;
  if (p.batch > 65535) return false;
  TmaMaps maps;
  if (!encode(&maps.a, p.A, (uint64_t)p.k, (uint64_t)p.m, (uint64_t)p.batch, p.lda, p.strideA, 16, 64) ||
      !encode(&maps.b, p.B, (uint64_t)p.n, (uint64_t)p.k, (uint64_t)p.batch, p.ldb, p.strideB, 16, 16))
    return false;
  const int smem = (int)gemm_tma_smem_bytes();
  if (set_smem_attr_once(reinterpret_cast<const void*>(gemm_tma_kernel), smem) != cudaSuccess) return false;
  const int tiles_m = (p.m + TBM - 1) / TBM, tiles_n = (p.n + TBN - 1) / TBN;
  int splits = p.splits > 1 ? p.splits : 1;
  if (splits > 1 && (p.jmask != nullptr || p.sd_d != nullptr || p.split_ws == nullptr ||
                     p.split_ws_elems < (int64_t)splits * p.batch * p.m * p.n))
    splits = 1;
  gemm_tma_kernel<<<dim3(tiles_m * tiles_n, p.batch, splits), 128, smem, stream>>>(maps, p, tiles_n);
  if (splits > 1) {
    const int tx = p.n >= 64 ? 64 : 32, ty = 256 / tx;
    const unsigned blocks = (unsigned)std::max(1, std::min((p.m + ty - 1) / ty, 2368 / std::max(1, p.batch) + 1));
    splitk_reduce_kernel<<<dim3(blocks, p.batch), dim3(tx, ty), 0, stream>>>(p, splits);
  }
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace pf
