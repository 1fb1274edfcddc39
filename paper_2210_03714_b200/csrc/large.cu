// K3 / K4 / K6 building blocks for n > 128 (large dense and batched mid-size systems).
//
// Every system z of a batch lives in a workspace of order np (n rounded up to a multiple of 64,
// identity padding), row-major, stride np^2. The host recursion (pf_large.cu) factors
// M_z = P_z L_z U_z and solves L U X = P R with DMMA GEMMs for all off-diagonal work and the
// kernels below for the diagonal blocks:
//   lu_base64_kernel    no-exchange LU of a 64 x 64 diagonal block (certified systems), plus the
//                       explicit inverses of its L and U factors (used by every block solve)
//   lu_base128_kernel   the same for a 128 x 128 diagonal block in one launch: a blocked 16-wide
//                       right-looking LU in shared memory with a look-ahead lead warp, then both
//                       64 halves' inverses (lu128_block)
//   trsm128_kernel      a 128-row / -column triangular solve chunk with the 64-block inverses
//   apply_inv64_kernel  B <- Linv B, B <- Uinv B (left) or B <- B Uinv (right), in place, DMMA
//   lu_dag_kernel       the device-scheduled tile-DAG LU (one persistent launch; see there)
//   lu_pivot_kernel     genuine partial pivoting, unblocked, in the reference's operation order
//                       (dense.cpp:105-132) -- the A/B fallback (PF_PIVOT_UNBLOCKED); the blocked
//                       pivoting LU is pivot_lu.cu + the recursion
//   form / certificate / accumulate / norm elementwise kernels (HBM-bound)
#include <climits>

#include "gemm_tile.cuh"
#include "tma_util.cuh"
#include "pf_common.cuh"
#include "pf_kernels.h"

namespace pf {
namespace {

constexpr int B64 = 64;
constexpr int L64 = B64 + 4;  // smem row stride

__device__ __forceinline__ double ldexp_j(double x, int j) { return j == 0 ? x : ldexp(x, -j); }

}  // namespace

// ---------------------------------------------------------------------------------------------
// LU of the 64 x 64 diagonal block at (off, off) of every system, no row exchanges, in place;
// inverses of L (unit lower) and U written to inv + z * inv_stride + (off / 64) * 2 * 64 * 64.
//  factor: right-looking, thread (r, q) keeps row r's columns q, q + 4, ... in registers; the
//          multiplier comes from the row's quad by shuffle and the pivot row from smem, one barrier
//          per pivot (the previous smem-only version with two barriers and an IEEE division per
//          step, plus 128-thread substitution inverses, took 86 us per call);
//  inverses: the eight 16 x 16 diagonal blocks of L and U by eight warps at once (16-step
//          substitution chains), then the off-diagonal blocks by block substitution on DMMA in
//          three dependency levels: X_ij = -X_ii (sum_k L_ik X_kj), Y_ij = -Y_ii (sum_k U_ik Y_kj).
namespace {
constexpr int TSW = 20;  // per-warp 16 x 16 scratch row stride

// acc += A (16 x K) B (K x 16), A / B row-major in smem (K a multiple of 4)
__device__ __forceinline__ void mm16(const double* A, int lda, const double* B, int ldb, int K, double (&acc)[2][2][2]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  for (int k = 0; k < K; k += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = A[(8 * mi + g) * lda + k + t];
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) bf[nj] = B[(k + t) * ldb + 8 * nj + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
  }
}

__device__ __forceinline__ void store16(double* D, int ldd, const double (&acc)[2][2][2], double scale) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) D[(8 * mi + g) * ldd + 8 * nj + 2 * t + e] = scale * acc[mi][nj][e];
}

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
}  // namespace

namespace {
// rows x 64 doubles from global (row stride ldg, 16-byte aligned rows) into smem (row stride lds) with
// 16-byte cp.async.cg (L2, coherent with other SMs' writes): every copy in flight at once instead
// of one latency-bound round trip per loop iteration. The caller commits and waits.
__device__ __forceinline__ void async_tile64(double* dst, int lds, const double* src, int64_t ldg, int rows) {
  for (int idx = threadIdx.x; idx < rows * 32; idx += blockDim.x) {
    const int r = idx >> 5, c2 = idx & 31;
    cp_async16(dst + r * lds + 2 * c2, src + (int64_t)r * ldg + 2 * c2, 16);
  }
}
__device__ __forceinline__ bool aligned16(const void* p, int64_t ld) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && ((ld & 1) == 0);
}
}  // namespace

size_t lu_base64_smem_bytes() { return sizeof(double) * (3 * B64 * L64 + 8 * 16 * TSW); }

// The 64 x 64 block s (smem, stride L64; xl / xu zeroed): LU in place (factor) and the inverses of
// its L (unit lower) and U into xl / xu. 256 threads.
__device__ void lu64_smem(double* s, double* xl, double* xu, double* scratch, int factor, int ls = L64) {
  const int lane = lane_id(), warp = warp_id();
  if (factor) {
    const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = s[r * ls + q + 4 * k];
#pragma unroll
    for (int m = 0; m < B64 - 1; ++m) {
      const double ip = rcp_nr(s[m * ls + m]);
      const double xm = __shfl_sync(0xffffffffu, v[m >> 2], (lane & ~3) | (m & 3));
      if (r > m) {
        const double f = xm * ip;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (q + 4 * k > m) v[k] = fma(-f, s[m * ls + q + 4 * k], v[k]);
        if (q == (m & 3)) v[m >> 2] = f;
      }
      if (r == m + 1) {
#pragma unroll
        for (int k = 0; k < 16; ++k) s[r * ls + q + 4 * k] = v[k];
      }
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) s[r * ls + q + 4 * k] = v[k];
    __syncthreads();
  }
  // diagonal 16 x 16 blocks: warps 0-3 L_bb^-1, warps 4-7 U_bb^-1 (lane l < 16: column l)
  {
    const int bb = warp & 3, o = 16 * bb, l = lane & 15;
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (i == l) ? 1.0 : 0.0;
    if (warp < 4) {
#pragma unroll
      for (int m = 0; m < 15; ++m)
#pragma unroll
        for (int i = m + 1; i < 16; ++i) x[i] = fma(-s[(o + i) * ls + o + m], x[m], x[i]);
      if (lane < 16)
#pragma unroll
        for (int i = 0; i < 16; ++i) xl[(o + i) * L64 + o + l] = x[i];
    } else {
#pragma unroll
      for (int m = 15; m >= 0; --m) {
        x[m] = x[m] * rcp_nr(s[(o + m) * ls + o + m]);
#pragma unroll
        for (int i = 0; i < m; ++i) x[i] = fma(-s[(o + i) * ls + o + m], x[m], x[i]);
      }
      if (lane < 16)
#pragma unroll
        for (int i = 0; i < 16; ++i) xu[(o + i) * L64 + o + l] = x[i];
    }
  }
  __syncthreads();
  // off-diagonal blocks, level d = 1, 2, 3: tasks (L, j) j < 4 - d and (U, i) i < 4 - d
  double* ws = scratch + warp * 16 * TSW;
  for (int d = 1; d < 4; ++d) {
    const int ntask = 4 - d;
    if (warp < 2 * ntask) {
      const bool lower = warp < ntask;
      const int b0 = lower ? warp : warp - ntask;
      double acc[2][2][2] = {};
      if (lower) {  // X_ij, i = b0 + d, j = b0: P = L[i, j..i-1] X[j..i-1, j]
        const int i = b0 + d, j = b0;
        mm16(s + 16 * i * ls + 16 * j, ls, xl + 16 * j * L64 + 16 * j, L64, 16 * d, acc);
        store16(ws, TSW, acc, 1.0);
        __syncwarp();
        double acc2[2][2][2] = {};
        mm16(xl + 16 * i * L64 + 16 * i, L64, ws, TSW, 16, acc2);
        store16(xl + 16 * i * L64 + 16 * j, L64, acc2, -1.0);
      } else {  // Y_ij, i = b0, j = b0 + d: P = U[i, i+1..j] Y[i+1..j, j]
        const int i = b0, j = b0 + d;
        mm16(s + 16 * i * ls + 16 * (i + 1), ls, xu + 16 * (i + 1) * L64 + 16 * j, L64, 16 * d, acc);
        store16(ws, TSW, acc, 1.0);
        __syncwarp();
        double acc2[2][2][2] = {};
        mm16(xu + 16 * i * L64 + 16 * i, L64, ws, TSW, 16, acc2);
        store16(xu + 16 * i * L64 + 16 * j, L64, acc2, -1.0);
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) lu_base64_kernel(double* M, int64_t ld, int64_t strideM, int off,
                                                        double* inv, int64_t inv_stride, int factor, const int* zlist) {
  extern __shared__ __align__(16) double lu_smem[];
  double* s = lu_smem;             // the block, LU in place
  double* xl = s + B64 * L64;      // L^-1
  double* xu = xl + B64 * L64;     // U^-1
  double* scratch = xu + B64 * L64;
  const int z = zlist ? zlist[blockIdx.x] : blockIdx.x;
  double* a = M + (int64_t)z * strideM + (int64_t)off * ld + off;
  const bool fast = aligned16(a, ld);
  if (fast) {
    async_tile64(s, L64, a, ld, B64);
    cp_async_commit();
  }
  for (int idx = threadIdx.x; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    if (!fast) s[r * L64 + c] = a[(int64_t)r * ld + c];
    xl[r * L64 + c] = 0.0;
    xu[r * L64 + c] = 0.0;
  }
  if (fast) cp_async_wait<0>();
  __syncthreads();
  lu64_smem(s, xl, xu, scratch, factor);
  double* out = inv + (int64_t)z * inv_stride + (int64_t)(off / B64) * 2 * B64 * B64;
  for (int idx = threadIdx.x; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    if (factor) a[(int64_t)r * ld + c] = s[r * L64 + c];
    out[idx] = xl[r * L64 + c];
    out[B64 * B64 + idx] = xu[r * L64 + c];
  }
}

// 128 x 128 diagonal block at (off, off), no exchanges, in one launch (one CTA per system): the
// four steps the host recursion would otherwise launch separately -- LU(A11) with its inverses,
// U12 = L11^-1 A12 and L21 = A21 U11^-1 (DMMA), A22 -= L21 U12 (DMMA), LU(A22) with its inverses.
// Same outputs as two 64 leaves and the level between them: the factors in place, the L / U
// inverses of both 64 blocks in `inv`.
namespace {
constexpr int L128 = 128 + 4;  // 128-tile smem row stride (32-byte skew)
constexpr int NB16 = 16;

// pointwise LU of the 16 x 16 block at (k0, k0) of S (stride L128), in place, by one warp: lane
// i < 16 holds row i; the pivot and the pivot row's tail come by shuffle
__device__ __forceinline__ void factor16(double* S, int k0) {
  const int lane = lane_id();
  double d[NB16];
#pragma unroll
  for (int c = 0; c < NB16; ++c) d[c] = lane < NB16 ? S[(k0 + lane) * L128 + k0 + c] : 0.0;
#pragma unroll
  for (int m = 0; m < NB16; ++m) {
    const double inv = rcp_nr(__shfl_sync(0xffffffffu, d[m], m));
    double u[NB16];
#pragma unroll
    for (int c = m + 1; c < NB16; ++c) u[c] = __shfl_sync(0xffffffffu, d[c], m);
    if (lane > m && lane < NB16) {
      const double f = d[m] * inv;
      d[m] = f;
#pragma unroll
      for (int c = m + 1; c < NB16; ++c) d[c] = fma(-f, u[c], d[c]);
    }
  }
  if (lane < NB16) {
#pragma unroll
    for (int c = 0; c < NB16; c += 2)
      *reinterpret_cast<double2*>(&S[(k0 + lane) * L128 + k0 + c]) = make_double2(d[c], d[c + 1]);
  }
}

// (R0, C0) 16 x 16 block of S -= S[R0.., k0..k0+16) S[k0..k0+16, C0..) by one warp (DMMA, K = 16)
__device__ __forceinline__ void schur16(double* S, int k0, int R0, int C0) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  double acc[2][2][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) {
      const double2 v = *reinterpret_cast<const double2*>(&S[(R0 + 8 * mi + g) * L128 + C0 + 8 * nj + 2 * t]);
      acc[mi][nj][0] = v.x;
      acc[mi][nj][1] = v.y;
    }
#pragma unroll
  for (int kk = 0; kk < NB16; kk += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = -S[(R0 + 8 * mi + g) * L128 + k0 + kk + t];
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) bf[nj] = S[(k0 + kk + t) * L128 + C0 + 8 * nj + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
      *reinterpret_cast<double2*>(&S[(R0 + 8 * mi + g) * L128 + C0 + 8 * nj + 2 * t]) =
          make_double2(acc[mi][nj][0], acc[mi][nj][1]);
}
}  // namespace

// The 128 x 128 diagonal tile at a (leading dimension ld), no exchanges, in place, plus the L / U
// inverses of its two 64-blocks into out (4 x 64^2: L11^-1, U11^-1, L22^-1, U22^-1) -- the outputs
// of two 64 leaves and the level between them. 256 threads, the tile in shared memory, blocked
// right-looking LU with 16-wide steps and one step of look-ahead: the lead warp (7) applies the
// Schur update to the next 16 x 16 diagonal block and factors it (pointwise, shuffles) while the
// other warps apply the rest of the trailing update (DMMA); between them, every row of the panel
// below (L21 = A21 U_kk^-1) and every column of the panel to the right (U12 = L_kk^-1 A12) is
// solved by its own thread. Then the two 64-blocks' inverses (lu64_smem's substitution + DMMA
// levels). Global reads bypass L1 (ld.global.cg): the persistent LU calls this on data other SMs
// just wrote.
size_t lu_base128_smem_bytes() { return sizeof(double) * (128 * L128 + 2 * B64 * L64 + 8 * 16 * TSW); }

// inv64_block: the L / U inverses of the factored 64 x 64 block at a (leading dimension ld) into
// out (2 x 64^2) -- the second half of lu128_block as a task of its own (the device-scheduled LU
// runs the two halves' inverses on two SMs, concurrently).
__device__ void inv64_block(const double* a, int64_t ld, double* out, double* smem) {
  double* s = smem;
  double* xl = s + B64 * L64;
  double* xu = xl + B64 * L64;
  double* scratch = xu + B64 * L64;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < B64 * 32; idx += blockDim.x) {
    const int r = idx >> 5, c2 = idx & 31;
    *reinterpret_cast<double2*>(&s[r * L64 + 2 * c2]) = __ldcg(reinterpret_cast<const double2*>(a + (int64_t)r * ld) + c2);
  }
  for (int idx = tid; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    xl[r * L64 + c] = 0.0;
    xu[r * L64 + c] = 0.0;
  }
  __syncthreads();
  lu64_smem(s, xl, xu, scratch, 0, L64);
  for (int idx = tid; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    out[idx] = xl[r * L64 + c];
    out[B64 * B64 + idx] = xu[r * L64 + c];
  }
}

// inverses == false: the factors only (inv64_block supplies the inverses)
__device__ void lu128_block(double* a, int64_t ld, double* out, double* lu_smem, bool inverses = true) {
  double* S = lu_smem;
  double* xl = S + 128 * L128;
  double* xu = xl + B64 * L64;
  double* scratch = xu + B64 * L64;
  const int tid = threadIdx.x, warp = warp_id();
  async_tile64(S, L128, a, ld, 128);
  async_tile64(S + 64, L128, a + 64, ld, 128);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  constexpr int kLead = 7;
  if (warp == kLead) factor16(S, 0);
  __syncthreads();
  for (int k0 = 0; k0 < 128 - NB16; k0 += NB16) {
    const int rest = 128 - k0 - NB16;
    if (tid < rest) {  // row k0 + 16 + tid of L21 = A21 U_kk^-1 (forward over the block's columns)
      const int row = k0 + NB16 + tid;
      double x[NB16], rinv[NB16];
#pragma unroll
      for (int c = 0; c < NB16; ++c) {
        x[c] = S[row * L128 + k0 + c];
        rinv[c] = rcp_nr(S[(k0 + c) * L128 + k0 + c]);
      }
#pragma unroll
      for (int m = 0; m < NB16; ++m) {
        x[m] = x[m] * rinv[m];
#pragma unroll
        for (int c = m + 1; c < NB16; ++c) x[c] = fma(-x[m], S[(k0 + m) * L128 + k0 + c], x[c]);
      }
#pragma unroll
      for (int c = 0; c < NB16; c += 2)
        *reinterpret_cast<double2*>(&S[row * L128 + k0 + c]) = make_double2(x[c], x[c + 1]);
    } else if (tid >= 128 && tid - 128 < rest) {  // column of U12 = L_kk^-1 A12 (unit lower)
      const int col = k0 + NB16 + (tid - 128);
      double y[NB16];
#pragma unroll
      for (int r = 0; r < NB16; ++r) y[r] = S[(k0 + r) * L128 + col];
#pragma unroll
      for (int m = 0; m < NB16 - 1; ++m)
#pragma unroll
        for (int r = m + 1; r < NB16; ++r) y[r] = fma(-S[(k0 + r) * L128 + k0 + m], y[m], y[r]);
#pragma unroll
      for (int r = 1; r < NB16; ++r) S[(k0 + r) * L128 + col] = y[r];
    }
    __syncthreads();
    const int nbk = rest / NB16;
    if (warp == kLead) {
      schur16(S, k0, k0 + NB16, k0 + NB16);
      __syncwarp();
      factor16(S, k0 + NB16);
    } else {
      for (int blk = warp + 1; blk < nbk * nbk; blk += kLead)
        schur16(S, k0, k0 + NB16 + NB16 * (blk / nbk), k0 + NB16 + NB16 * (blk % nbk));
    }
    __syncthreads();
  }
  // the factors out; the 64-blocks' inverses
  for (int idx = tid; idx < 128 * 64; idx += blockDim.x) {
    const int r = idx >> 6, c2 = idx & 63;
    reinterpret_cast<double2*>(a + (int64_t)r * ld)[c2] = *reinterpret_cast<const double2*>(&S[r * L128 + 2 * c2]);
  }
  if (!inverses) return;
  for (int h = 0; h < 2; ++h) {
    for (int idx = tid; idx < B64 * B64; idx += blockDim.x) {
      const int r = idx >> 6, c = idx & 63;
      xl[r * L64 + c] = 0.0;
      xu[r * L64 + c] = 0.0;
    }
    __syncthreads();
    lu64_smem(S + h * B64 * L128 + h * B64, xl, xu, scratch, 0, L128);
    double* o = out + h * 2 * B64 * B64;
    for (int idx = tid; idx < B64 * B64; idx += blockDim.x) {
      const int r = idx >> 6, c = idx & 63;
      o[idx] = xl[r * L64 + c];
      o[B64 * B64 + idx] = xu[r * L64 + c];
    }
    __syncthreads();
  }
}



__global__ void __launch_bounds__(256) lu_base128_kernel(double* M, int64_t ld, int64_t strideM, int off,
                                                         double* inv, int64_t inv_stride) {
  extern __shared__ __align__(16) double lu_smem[];
  const int z = blockIdx.x;
  lu128_block(M + (int64_t)z * strideM + (int64_t)off * ld + off, ld,
              inv + (int64_t)z * inv_stride + (int64_t)(off / B64) * 2 * B64 * B64, lu_smem);
}

// ---------------------------------------------------------------------------------------------
// Triangular solve with a 128 x 128 diagonal block [off, off + 128) in one launch (the three
// launches of the host recursion at that level -- inverse, update, inverse -- fused per chunk):
//   mode 0 (left, L unit lower):  B1 <- L11^-1 B1;            B2 <- L22^-1 (B2 - L21 B1)
//   mode 1 (left, U upper):       B2 <- U22^-1 B2;            B1 <- U11^-1 (B1 - U12 B2)
//   mode 2 (right, U upper):      B1 <- B1 U11^-1;            B2 <- (B2 - B1 U12) U22^-1
// Left modes: CTA = 64 columns of the 128-row panel B; right mode: CTA = 64 rows of the 128-column
// panel. Explicit 64-block inverses from `inv` (as apply_inv64), the coupling block from M.
size_t trsm128_smem_bytes() { return sizeof(double) * (5 * B64 * L64); }

namespace {
// D (64 x 64, smem, stride L64) = X Y (both smem 64 x 64), into registers: two 16 x 16 tiles per warp
// the warp's two tiles (2 warp, 2 warp + 1: the same 16-row block i, columns j and j + 1) in one
// k loop -- shared A fragments and eight independent accumulator chains instead of two passes of four
__device__ __forceinline__ void mm64_regs(const double* X, const double* Y, double (&acc)[2][2][2][2]) {
  const int warp = warp_id(), lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int i = warp >> 1, j0 = 2 * (warp & 1);
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) acc[u][mi][nj][0] = acc[u][mi][nj][1] = 0.0;
  const double* A = X + 16 * i * L64;
  const double* B = Y + 16 * j0;
#pragma unroll 4
  for (int k = 0; k < B64; k += 4) {
    double af[2], bf[2][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = A[(8 * mi + g) * L64 + k + t];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) bf[u][nj] = B[(k + t) * L64 + 16 * u + 8 * nj + g];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) dmma(acc[u][mi][nj], af[mi], bf[u][nj]);
  }
}
// D = base - acc (base == nullptr: D = acc), D smem 64 x 64
__device__ __forceinline__ void store64(double* D, const double* base, const double (&acc)[2][2][2][2]) {
  const int warp = warp_id(), lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int tile = warp * 2 + u, i = tile >> 2, j = tile & 3;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int idx = (16 * i + 8 * mi + g) * L64 + 16 * j + 8 * nj + 2 * t + e;
          D[idx] = base ? base[idx] - acc[u][mi][nj][e] : acc[u][mi][nj][e];
        }
  }
}
}  // namespace

// m: the 128 diagonal block's origin, blkinv: its 64-blocks' inverses, b: the 64-column (left modes)
// or 64-row (right mode) chunk of B, `live` of them in range. Global reads bypass L1 (ld.global.cg).
__device__ void trsm128_chunk(const double* m, int64_t ld, const double* blkinv, int mode, double* b, int64_t ldb,
                              int live, double* t_smem) {
  double* t1 = t_smem;             // first inverse to apply
  double* t2 = t1 + B64 * L64;     // second inverse
  double* cpl = t2 + B64 * L64;    // coupling block (L21 or U12)
  double* b1 = cpl + B64 * L64;    // the chunk's first 64 (rows, or columns in mode 2)
  double* b2 = b1 + B64 * L64;     // ... and second 64
  const bool right = mode == 2;
  // mode 0: t1 = L11^-1, t2 = L22^-1, cpl = L21; modes 1, 2: t1 = U11^-1, t2 = U22^-1, cpl = U12
  const double* i1 = blkinv + (mode == 0 ? 0 : B64 * B64);
  const double* i2 = blkinv + 2 * B64 * B64 + (mode == 0 ? 0 : B64 * B64);
  const double* c0 = mode == 0 ? m + (int64_t)B64 * ld : m + B64;
  if (live == B64 && aligned16(b, ldb) && aligned16(m, ld) && aligned16(blkinv, 0)) {
    async_tile64(t1, L64, i1, B64, B64);
    async_tile64(t2, L64, i2, B64, B64);
    async_tile64(cpl, L64, c0, ld, B64);
    if (!right) {
      async_tile64(b1, L64, b, ldb, B64);
      async_tile64(b2, L64, b + (int64_t)B64 * ldb, ldb, B64);
    } else {
      async_tile64(b1, L64, b, ldb, B64);
      async_tile64(b2, L64, b + B64, ldb, B64);
    }
    cp_async_commit();
    cp_async_wait<0>();
  } else
  for (int idx = threadIdx.x; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    t1[r * L64 + c] = __ldcg(i1 + idx);
    t2[r * L64 + c] = __ldcg(i2 + idx);
    cpl[r * L64 + c] = __ldcg(c0 + (int64_t)r * ld + c);
    if (!right) {  // B rows r and 64 + r, chunk column c
      const bool ok = c < live;
      b1[r * L64 + c] = ok ? __ldcg(b + (int64_t)r * ldb + c) : 0.0;
      b2[r * L64 + c] = ok ? __ldcg(b + (int64_t)(B64 + r) * ldb + c) : 0.0;
    } else {  // B row r of the chunk, columns c and 64 + c
      const bool ok = r < live;
      b1[r * L64 + c] = ok ? __ldcg(b + (int64_t)r * ldb + c) : 0.0;
      b2[r * L64 + c] = ok ? __ldcg(b + (int64_t)r * ldb + B64 + c) : 0.0;
    }
  }
  __syncthreads();
  double acc[2][2][2][2];
  if (mode == 0) {
    mm64_regs(t1, b1, acc);  // B1' = L11^-1 B1
    __syncthreads();
    store64(b1, nullptr, acc);
    __syncthreads();
    mm64_regs(cpl, b1, acc);  // B2 - L21 B1'
    __syncthreads();
    store64(b2, b2, acc);
    __syncthreads();
    mm64_regs(t2, b2, acc);  // L22^-1 (...)
    __syncthreads();
    store64(b2, nullptr, acc);
  } else if (mode == 1) {
    mm64_regs(t2, b2, acc);  // B2' = U22^-1 B2
    __syncthreads();
    store64(b2, nullptr, acc);
    __syncthreads();
    mm64_regs(cpl, b2, acc);  // B1 - U12 B2'
    __syncthreads();
    store64(b1, b1, acc);
    __syncthreads();
    mm64_regs(t1, b1, acc);  // U11^-1 (...)
    __syncthreads();
    store64(b1, nullptr, acc);
  } else {
    mm64_regs(b1, t1, acc);  // B1' = B1 U11^-1
    __syncthreads();
    store64(b1, nullptr, acc);
    __syncthreads();
    mm64_regs(b1, cpl, acc);  // B2 - B1' U12
    __syncthreads();
    store64(b2, b2, acc);
    __syncthreads();
    mm64_regs(b2, t2, acc);  // (...) U22^-1
    __syncthreads();
    store64(b2, nullptr, acc);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    if (!right) {
      if (c < live) {
        b[(int64_t)r * ldb + c] = b1[r * L64 + c];
        b[(int64_t)(B64 + r) * ldb + c] = b2[r * L64 + c];
      }
    } else if (r < live) {
      b[(int64_t)r * ldb + c] = b1[r * L64 + c];
      b[(int64_t)r * ldb + B64 + c] = b2[r * L64 + c];
    }
  }
}

__global__ void __launch_bounds__(256) trsm128_kernel(const double* M, int64_t ld, int64_t strideM, int off,
                                                      const double* inv, int64_t inv_stride, int mode, double* Bm,
                                                      int64_t ldb, int64_t strideB, int extent) {
  extern __shared__ __align__(16) double t_smem[];
  const int z = blockIdx.y, tile = blockIdx.x;
  const bool right = mode == 2;
  trsm128_chunk(M + (int64_t)z * strideM + (int64_t)off * ld + off, ld,
                inv + (int64_t)z * inv_stride + (int64_t)(off / B64) * 2 * B64 * B64, mode,
                Bm + (int64_t)z * strideB + (right ? (int64_t)tile * B64 * ldb : (int64_t)tile * B64), ldb,
                min(B64, extent - tile * B64), t_smem);
}

// ---------------------------------------------------------------------------------------------
// In-place block solve with an explicit 64 x 64 inverse T (T = Linv or Uinv of diagonal block blk):
//   left : B[64 x cols] <- T B     (CTA = 64 columns)
//   right: B[rows x 64] <- B T     (CTA = 64 rows)
// 8 warps, each a 16 x 32 output tile (2 x 4 DMMA tiles), K = 64.
__global__ void __launch_bounds__(256) apply_inv64_kernel(const double* inv, int64_t inv_stride, int blk, int upper,
                                                          int right, double* Bm, int64_t ld, int64_t strideB,
                                                          int extent) {
  extern __shared__ __align__(16) double inv_smem[];
  double* t = inv_smem;
  double* bt = inv_smem + B64 * L64;
  const int z = blockIdx.y;
  const int tile = blockIdx.x;
  const double* T = inv + (int64_t)z * inv_stride + (int64_t)blk * 2 * B64 * B64 + (upper ? B64 * B64 : 0);
  double* b = Bm + (int64_t)z * strideB + (right ? (int64_t)tile * B64 * ld : (int64_t)tile * B64);
  const int live = min(B64, extent - tile * B64);  // columns (left) or rows (right) in range
  if (live == B64 && aligned16(b, ld) && aligned16(T, 0)) {
    async_tile64(t, L64, T, B64, B64);
    async_tile64(bt, L64, b, ld, B64);
    cp_async_commit();
    cp_async_wait<0>();
  } else
  for (int idx = threadIdx.x; idx < B64 * B64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    t[r * L64 + c] = T[r * B64 + c];
    const bool ok = right ? (r < live) : (c < live);
    bt[r * L64 + c] = ok ? b[(int64_t)r * ld + c] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int rb = 16 * (warp >> 1), cb = 32 * (warp & 1);
  const double* As = right ? bt : t;  // left: T * Bt ; right: Bt * T
  const double* Bs = right ? t : bt;
  double acc[2][4][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
#pragma unroll 4
  for (int k = 0; k < B64; k += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = As[(rb + 8 * mi + g) * L64 + k + tq];
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) bf[nj] = Bs[(k + tq) * L64 + cb + 8 * nj + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 4; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = rb + 8 * mi + g, c = cb + 8 * nj + 2 * tq + e;
        const bool ok = right ? (r < live) : (c < live);
        if (ok) b[(int64_t)r * ld + c] = acc[mi][nj][e];
      }
}

// ---------------------------------------------------------------------------------------------
// Genuine partial pivoting (reference operation order, dense.cpp:105-132) on the leading n x n of
// each np x np system; one CTA of 1024 threads per system, global memory. Fallback only.
__global__ void __launch_bounds__(1024) lu_pivot_kernel(double* M, int64_t ld, int64_t strideM, int n, int* piv,
                                                        const double* tol, DevStatus* status, int* first_error,
                                                        const int* zlist) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_p;
  __shared__ double s_best;
  const int z = zlist ? zlist[blockIdx.x] : blockIdx.x;
  double* a = M + (int64_t)z * strideM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int col = 0; col < n; ++col) {
    double best = -1.0;
    int p = INT_MAX;
    for (int r = col + threadIdx.x; r < n; r += blockDim.x) {
      const double v = fabs(a[(int64_t)r * ld + col]);
      if (v > best) {
        best = v;
        p = r;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      if (ob > best || (ob == best && op < p)) {
        best = ob;
        p = op;
      }
    }
    if (lane == 0) {
      red_v[warp] = best;
      red_i[warp] = p;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = red_v[0];
      int pp = red_i[0];
      for (int w = 1; w < nw; ++w)
        if (red_v[w] > bb || (red_v[w] == bb && red_i[w] < pp)) {
          bb = red_v[w];
          pp = red_i[w];
        }
      s_best = bb;
      s_p = pp;
    }
    __syncthreads();
    const int pp = s_p;
    const double bb = s_best;
    if (bb <= tol[z]) {
      if (threadIdx.x == 0) {
        status[z].code = PF_ERR_SINGULAR_SHIFT;
        status[z].column = col;
        status[z].pivot_magnitude = bb;
        atomicMin(first_error, z);
      }
      return;
    }
    if (pp != col)
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const double tmp = a[(int64_t)pp * ld + c];
        a[(int64_t)pp * ld + c] = a[(int64_t)col * ld + c];
        a[(int64_t)col * ld + c] = tmp;
      }
    if (threadIdx.x == 0) piv[(int64_t)z * n + col] = pp;
    __syncthreads();
    const double inv_piv = 1.0 / a[(int64_t)col * ld + col];
    for (int r = col + 1 + threadIdx.x; r < n; r += blockDim.x)
      a[(int64_t)r * ld + col] = __dmul_rn(a[(int64_t)r * ld + col], inv_piv);
    __syncthreads();
    const int w = n - col - 1;
    for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += blockDim.x) {
      const int r = col + 1 + (int)(idx / w), c = col + 1 + (int)(idx % w);
      const double f = a[(int64_t)r * ld + col];
      if (f != 0.0) a[(int64_t)r * ld + c] = __dsub_rn(a[(int64_t)r * ld + c], __dmul_rn(f, a[(int64_t)col * ld + c]));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// System z = i * batch + b (shift i, matrix b). M_z = (-c_i) 2^-j_b A_b + I (padding: identity);
// also max|M_z| over the true block -> mx[z] (atomicMax on the bit pattern of a non-negative double).
__global__ void form_shifted_kernel(const double* A, int64_t lda, int64_t strideA, int n, int np, int batch,
                                    const double* shifts, const int* j, double* M, unsigned long long* mx) {
  const int z = blockIdx.y;
  const int b = z % batch, i = z / batch;
  const double c = shifts[i];
  const int jb = j ? j[b] : 0;
  const double* a = A + (int64_t)b * strideA;
  double* m = M + (int64_t)z * np * np;
  double loc = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)np * np;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / np), col = (int)(idx % np);
    double v;
    if (r < n && col < n) {
      v = __dmul_rn(ldexp_j(a[(int64_t)r * lda + col], jb), -c);  // (-c) B + I (dense.cpp:211-213)
      if (r == col) v = __dadd_rn(v, 1.0);
      loc = fmax(loc, fabs(v));
    } else {
      v = (r == col) ? 1.0 : 0.0;
    }
    m[idx] = v;
  }
  for (int o = 16; o > 0; o >>= 1) loc = fmax(loc, __shfl_xor_sync(0xffffffffu, loc, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx + z, (unsigned long long)__double_as_longlong(loc));
}

// Strict column diagonal dominance with margin (see small_eval.cu): ok[z] stays 1 only if every
// column passes. Off-diagonal column sums in two passes: certificate_partial_kernel sums row chunk
// blockIdx.y of every column (one thread per column, coalesced rows), certificate_kernel adds the
// chunks in ascending order -- a fixed order, so the decision is deterministic. (One thread summing
// all n rows of its column took 1.8 ms for 8 x 4096^2: a 4096-long dependent add chain per thread.)
__global__ void certificate_partial_kernel(const double* M, int np, int n, int chunk, double* part) {
  const int z = blockIdx.z, q = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  const double* m = M + (int64_t)z * np * np;
  const int r0 = q * chunk, r1 = min(n, r0 + chunk);
  double s0 = 0.0, s1 = 0.0;  // two interleaved chains, combined at the end
  int r = r0;
  for (; r + 1 < r1; r += 2) {
    const double a0 = (r != col) ? fabs(m[(int64_t)r * np + col]) : 0.0;
    const double a1 = (r + 1 != col) ? fabs(m[(int64_t)(r + 1) * np + col]) : 0.0;
    s0 += a0;
    s1 += a1;
  }
  if (r < r1 && r != col) s0 += fabs(m[(int64_t)r * np + col]);
  part[((int64_t)z * gridDim.y + q) * n + col] = s0 + s1;
}

__global__ void certificate_kernel(const double* M, int np, int n, int nchunks, const double* part,
                                   const unsigned long long* mx, double rel_tol, int* ok) {
  const int z = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  const double* m = M + (int64_t)z * np * np;
  double off = 0.0;
  for (int q = 0; q < nchunks; ++q) off += part[((int64_t)z * nchunks + q) * n + col];
  const double mxz = __longlong_as_double((long long)mx[z]);
  const double margin = fabs(m[(int64_t)col * np + col]) - off;
  const bool pass = (margin >= 1e-10 * mxz) && (margin > 2.0 * rel_tol * fmax(mxz, 1e-300)) && (mxz > 1e-250) &&
                    (mxz < 1e250);
  if (!pass) atomicAnd(ok + z, 0);
}

// Pair mode (pf_large.cu large_eval_pairs): the reference's systems I - cB and I + cB must be
// certified for every pair c. Column statistics of B in two passes like the certificate above:
// off-diagonal |b| sums per row chunk, and max|B| per matrix (atomicMax on the bit pattern).
__global__ void colstat_partial_kernel(const double* B, int64_t ld, int64_t strideB, int n, int chunk, double* part,
                                       unsigned long long* bmax) {
  const int z = blockIdx.z, q = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0;
  if (col < n) {
    const double* m = B + (int64_t)z * strideB;
    const int r0 = q * chunk, r1 = min(n, r0 + chunk);
    double s0 = 0.0;
    for (int r = r0; r < r1; ++r) {
      const double a = fabs(m[(int64_t)r * ld + col]);
      mx = fmax(mx, a);
      if (r != col) s0 += a;
    }
    part[((int64_t)z * gridDim.y + q) * n + col] = s0;
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(bmax + z, (unsigned long long)__double_as_longlong(mx));
}

// |1 -/+ c b_jj| - |c| sum_{i != j} |b_ij| > bound (1 + |c| max|B|) for every pair c and column j:
// strict column diagonal dominance of I - cB and I + cB with the per-shift certificate's margin
// taken at the upper bound 1 + |c| max|B| of max|I -/+ cB|.
__global__ void pair_certificate_kernel(const double* B, int64_t ld, int64_t strideB, int n, int nchunks,
                                        const double* part, const unsigned long long* bmax, const double* c, int npairs,
                                        double rel, int* ok) {
  const int z = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  double off = 0.0;
  for (int q = 0; q < nchunks; ++q) off += part[((int64_t)z * nchunks + q) * n + col];
  const double d = B[(int64_t)z * strideB + (int64_t)col * ld + col];
  const double bm = __longlong_as_double((long long)bmax[z]);
  bool pass = bm < 1e250;
  for (int p = 0; p < npairs && pass; ++p) {
    const double cc = c[p], scale = 1.0 + fabs(cc) * bm;
    const double bound = fmax(1e-10, 2.0 * rel) * scale;
    const double o = fabs(cc) * off;
    pass = (fabs(1.0 - cc * d) - o > bound) && (fabs(1.0 + cc * d) - o > bound);
  }
  if (!pass) atomicAnd(ok + z, 0);
}

// R_z = c_i 2^-j A_b[perm] (residual) or P I (plain), padded np x cols (cols = np for matrices).
// For the action, A_b is replaced by the block V (n x k): src_ld / src_stride describe it.
__global__ void form_rhs_kernel(const double* src, int64_t lds, int64_t strideS, int n, int np, int cols, int ncols_true,
                                int batch, const double* shifts, const int* j, int residual, const int* perm,
                                double* R, int64_t strideR) {
  const int z = blockIdx.y;
  const int b = z % batch, i = z / batch;
  const double c = shifts[i];
  const int jb = j ? j[b] : 0;
  const double* s = src + (int64_t)b * strideS;
  double* rz = R + (int64_t)z * strideR;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)np * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / cols), col = (int)(idx % cols);
    double v = 0.0;
    if (r < n && col < ncols_true) {
      const int pr = perm ? perm[(int64_t)z * n + r] : r;
      if (residual)
        v = __dmul_rn(ldexp_j(s[(int64_t)pr * lds + col], jb), c);
      else
        v = (pr == col) ? 1.0 : 0.0;
    }
    rz[idx] = v;
  }
}

// out_s[b] = sum_i (w_{s,i} X_{i,b}) in ascending i, then + poly (const I + d1 B + d2 B^2) -- the
// fixed-order reduction and poly_part of eval_dense (dense.cpp:176-189, 217, 245-250).
// term_z[t] = system slot of term t (the X of shift t lives at X + (slot * batch + b) * strideX),
// or -1 for a plain-form zero shift (the w I term).
__global__ void accumulate_kernel(const double* X, int64_t xld, int64_t strideX, int n, int cols, int batch,
                                  int n_terms, const int* term_z, const double* w, int add_poly, double constant,
                                  double d1, double d2, const double* Bsrc, int64_t bld, int64_t strideBs,
                                  const int* j, const double* B2, int64_t b2ld, int64_t strideB2, double* out,
                                  int64_t ldo, int64_t strideOut) {
  const int b = blockIdx.y;
  const int jb = j ? j[b] : 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / cols), col = (int)(idx % cols);
    double acc = 0.0;
    for (int t = 0; t < n_terms; ++t) {
      const int z = term_z[t];
      double tv;
      if (z < 0)
        tv = (r == col) ? __dadd_rn(0.0, w[t]) : 0.0;
      else
        tv = __dmul_rn(X[(int64_t)(z * batch + b) * strideX + (int64_t)r * xld + col], w[t]);
      acc = (t == 0) ? tv : __dadd_rn(acc, tv);
    }
    if (add_poly) {
      double poly = (r == col) ? __dadd_rn(0.0, constant) : 0.0;
      if (d1 != 0.0 || d2 != 0.0)
        poly = __dadd_rn(poly, __dmul_rn(d1, ldexp_j(Bsrc[(int64_t)b * strideBs + (int64_t)r * bld + col], jb)));
      if (d2 != 0.0) poly = __dadd_rn(poly, __dmul_rn(d2, B2[(int64_t)b * strideB2 + (int64_t)r * b2ld + col]));
      acc = __dadd_rn(acc, poly);
    }
    out[(int64_t)b * strideOut + (int64_t)r * ldo + col] = acc;
  }
}

// Up to four weighted sums of the same solutions in ONE pass over them (every X element read once):
// output o = sum_t w_o[t] X_t in ascending t (plus its poly part), rounded exactly as
// accumulate_kernel -- the weight sets of a method and the pair path's E_A / E_B share the reads.
__global__ void accumulate_sets_kernel(const double* X, int64_t xld, int64_t strideX, int n, int cols, int batch,
                                       int n_terms, const int* term_z, AccSets sets, const double* Bsrc, int64_t bld,
                                       int64_t strideBs, const int* j, const double* B2, int64_t b2ld,
                                       int64_t strideB2) {
  const int b = blockIdx.y;
  const int jb = j ? j[b] : 0;
  const int no = sets.n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / cols), col = (int)(idx % cols);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < n_terms; ++t) {
      const int z = term_z[t];
      const double x = z < 0 ? 0.0 : X[(int64_t)(z * batch + b) * strideX + (int64_t)r * xld + col];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        if (o >= no) break;
        const double w = sets.s[o].w[t];
        const double tv = z < 0 ? ((r == col) ? __dadd_rn(0.0, w) : 0.0) : __dmul_rn(x, w);
        acc[o] = (t == 0) ? tv : __dadd_rn(acc[o], tv);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      if (o >= no) break;
      const AccSet& q = sets.s[o];
      double v = acc[o];
      if (q.add_poly) {
        double poly = (r == col) ? __dadd_rn(0.0, q.constant) : 0.0;
        if (q.d1 != 0.0 || q.d2 != 0.0)
          poly = __dadd_rn(poly, __dmul_rn(q.d1, ldexp_j(Bsrc[(int64_t)b * strideBs + (int64_t)r * bld + col], jb)));
        if (q.d2 != 0.0) poly = __dadd_rn(poly, __dmul_rn(q.d2, B2[(int64_t)b * strideB2 + (int64_t)r * b2ld + col]));
        v = __dadd_rn(v, poly);
      }
      q.out[(int64_t)b * q.strideOut + (int64_t)r * q.ldo + col] = v;
    }
  }
}

// perm_z from the swap sequence piv_z (LAPACK style): perm[r] = row of the original RHS in row r.
// the row permutation of a swap sequence: one warp per system, the sequence applied by lane 0 in
// shared memory (chunks of 4096 rows' swaps staged by the warp; larger n walks global memory)
__global__ void perm_from_piv_kernel(const int* piv, int n, int* perm, const int* zlist) {
  constexpr int S = 4096;
  __shared__ int p_s[S], q_s[S];
  const int z = zlist ? zlist[blockIdx.x] : blockIdx.x;
  int* p = perm + (int64_t)z * n;
  const int* pv = piv + (int64_t)z * n;
  if (n <= S) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      p_s[r] = r;
      q_s[r] = pv[r];
    }
    __syncwarp();
    if (threadIdx.x == 0)
      for (int r = 0; r < n; ++r) {
        const int q = q_s[r];
        const int t = p_s[r];
        p_s[r] = p_s[q];
        p_s[q] = t;
      }
    __syncwarp();
    for (int r = threadIdx.x; r < n; r += blockDim.x) p[r] = p_s[r];
    return;
  }
  if (threadIdx.x != 0) return;
  for (int r = 0; r < n; ++r) p[r] = r;
  for (int r = 0; r < n; ++r) {
    const int q = pv[r];
    const int t = p[r];
    p[r] = p[q];
    p[q] = t;
  }
}

// copy (strided 2-D, batched) with optional scale: Y = s X
__global__ void copy2d_kernel(int rows, int cols, double s, const double* X, int64_t ldx, int64_t strideX, double* Y,
                              int64_t ldy, int64_t strideY) {
  const int b = blockIdx.y;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)rows * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / cols), c = (int)(idx % cols);
    const double v = X[(int64_t)b * strideX + (int64_t)r * ldx + c];
    Y[(int64_t)b * strideY + (int64_t)r * ldy + c] = s == 1.0 ? v : __dmul_rn(s, v);
  }
}

// B = A * inv elementwise (substep_action's A * (1.0 / N), action.cpp:330-334), padded with zeros.
__global__ void scale_pad_kernel(const double* A, int64_t lda, int n, int np, double s, double* B) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)np * np;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / np), c = (int)(idx % np);
    B[idx] = (r < n && c < n) ? __dmul_rn(A[(int64_t)r * lda + c], s) : 0.0;
  }
}

// M_z = A_z with identity padding; max|a| over the true block -> mx[z]
__global__ void load_padded_kernel(const double* A, int64_t lda, int64_t strideA, int n, int np, double* M,
                                   unsigned long long* mx) {
  const int z = blockIdx.y;
  const double* a = A + (int64_t)z * strideA;
  double* m = M ? M + (int64_t)z * np * np : nullptr;  // M null: max |a| only (in-place factorisation)
  double loc = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)np * np;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / np), c = (int)(idx % np);
    double v;
    if (r < n && c < n) {
      v = a[(int64_t)r * lda + c];
      loc = fmax(loc, fabs(v));
    } else {
      v = (r == c) ? 1.0 : 0.0;
    }
    if (m) m[idx] = v;
  }
  for (int o = 16; o > 0; o >>= 1) loc = fmax(loc, __shfl_xor_sync(0xffffffffu, loc, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx + z, (unsigned long long)__double_as_longlong(loc));
}

__global__ void iota_kernel(int* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[(int64_t)blockIdx.y * n + i] = i;
}

size_t apply_inv64_smem_bytes() { return sizeof(double) * 2 * B64 * L64; }

__global__ void fill_int_kernel(int* p, int count, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) p[i] = v;
}

}  // namespace pf

namespace pf {
// action step: out = sum_t w_t T_t (T_t = R_z, or X itself for a plain-form zero shift), then
// + constant X (+ d1 BX + d2 B(BX)) -- assemble_action's fixed-order reduction (action.cpp:265-282).
__global__ void action_accumulate_kernel(const double* R, int64_t rld, int64_t strideR, const double* X, int64_t xld,
                                         int n, int k, int n_terms, const int* term_z, const double* w, int add_poly,
                                         double constant, int hybrid, double d1, double d2, const double* BX,
                                         const double* B2X, double* out, int64_t ldo) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * k;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / k), c = (int)(idx % k);
    const double xv = X[(int64_t)r * xld + c];
    double acc = 0.0;
    for (int t = 0; t < n_terms; ++t) {
      const int z = term_z[t];
      const double tv = __dmul_rn(z < 0 ? xv : R[(int64_t)z * strideR + (int64_t)r * rld + c], w[t]);
      acc = (t == 0) ? tv : __dadd_rn(acc, tv);
    }
    if (add_poly) {
      acc = __dadd_rn(acc, __dmul_rn(constant, xv));
      if (hybrid) {
        const double bx = BX[(int64_t)r * xld + c], b2x = B2X[(int64_t)r * xld + c];
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(d1, bx), __dmul_rn(d2, b2x)));
      }
    }
    out[(int64_t)r * ldo + c] = acc;
  }
}

// out = d1 X + d2 Y (each product rounded, then the sum): the hybrid poly term of assemble_action
// (action.cpp:279-281), kept separate for the deterministic multi-rank reduction.
__global__ void lincomb2_kernel(int n, int k, double d1, const double* X, double d2, const double* Y, int64_t ld,
                                double* out, int64_t ldo) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * k;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / k), c = (int)(idx % k);
    out[(int64_t)r * ldo + c] = __dadd_rn(__dmul_rn(d1, X[(int64_t)r * ld + c]), __dmul_rn(d2, Y[(int64_t)r * ld + c]));
  }
}
// ---------------------------------------------------------------------------------------------
// Device-scheduled tile-DAG LU (no exchanges: the certified systems) of nsys systems of order np
// (a multiple of 128), one persistent CTA per SM. The 128 x 128 tiles of every system form the DAG
//   F(k)      LU of the diagonal tile (k, k) + its 64-block L / U inverses      (lu128_block)
//   R(k, j)   U_kj = L_kk^-1 A_kj,  C(i, k)  L_ik = A_ik U_kk^-1                 (trsm128_chunk)
//   G(i,j,k)  A_ij -= L_ik U_kj                                                  (gemm_tile, DMMA)
// listed by the host in a topological order with one step of look-ahead (the tiles of row / column
// k + 1 are updated, F(k + 1) and its panel solved before the rest of step k's trailing update). CTAs
// pull the next task from a global counter, wait (acquire) until its inputs are final, run it and
// publish (release) the tile's new state = the number of steps applied to it. Every CTA only waits
// for tasks listed earlier, all of which are held by running CTAs: no deadlock. The 8 systems of a
// batch share every wave, and the whole factorisation is one launch instead of the recursion's
// hundreds of dependent ones. Each tile's updates run in step order, so the result does not depend
// on which CTA runs which task. A spin limit turns a scheduling bug into an error flag, not a hang.
namespace {
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ bool wait_ge(const int* p, int need, int* err) {
  unsigned spins = 0;
  while (ld_acquire(p) < need) {
    if (ld_acquire(err)) return false;
    __nanosleep(64);
    if (++spins > (1u << 25)) {
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}
}  // namespace

// G task on TMA: C (128 x 128 tile) -= A B, A = the L tile (i, k), B = the U tile (k, j) of system z,
// staged by the tensor-memory accelerator in a two-stage ring (box A 16 x 128, B eight 16 x 16 boxes,
// 128-byte swizzle, k-permuted fragments as gemm_tma.cu), 8 warps of 32 x 64. `fills` counts the
// CTA's ring fills over all its G tasks (stage = fill % 2, phase = fill / 2) -- the ring's mbarriers
// live for the whole persistent kernel.
namespace {
constexpr int DG_A_BYTES = 128 * 16 * 8, DG_STAGE = 2 * DG_A_BYTES;
#ifndef PF_DAG_STAGES
#define PF_DAG_STAGES 3
#endif
constexpr unsigned DG_NS = PF_DAG_STAGES;  // ring stages
__device__ void dag_gemm_tma(const DagMaps& maps, int z, int i, int j, int k0, int steps, double* C, int ldc,
                             unsigned char* ring, unsigned fullb, unsigned emptyb, unsigned& fills) {
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wm = 32 * (warp >> 1), wn = 64 * (warp & 1);
  const unsigned base = su32(ring);
  const int NK = 8 * steps;  // 16-wide k tiles over the steps k0 .. k0 + steps - 1
  auto issue = [&](unsigned f, int kt) {
    const unsigned s = f % DG_NS, sa = base + s * DG_STAGE, sb = sa + DG_A_BYTES, bar = fullb + 8 * s;
    if (f >= DG_NS) mb_wait(emptyb + 8 * s, ((f / DG_NS) - 1) & 1u);
    mb_expect(bar, DG_STAGE);
    tma3(sa, &maps.a, 128 * k0 + 16 * kt, 128 * i, z, bar);
#pragma unroll
    for (int q = 0; q < 8; ++q) tma3(sb + q * 2048, &maps.b, 128 * j + 16 * q, 128 * k0 + 16 * kt, z, bar);
  };
  if (tid == 0) {
    fence_proxy_async_all();  // the tiles other CTAs published (generic stores) before these async reads;
                              // this CTA's earlier generic use of the ring before its async refills
    for (int kt = 0; kt < (int)DG_NS - 1 && kt < NK; ++kt) issue(fills + kt, kt);
  }
  unsigned offA[4], offB[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int kt_ = 2 * (s & 1) + 8 * (s >> 1) + (t & 1) + 4 * (t >> 1);
    offA[s] = (unsigned)((wm + g) * 128 + ((((kt_ >> 1) ^ g) & 7) << 4) + ((kt_ & 1) << 3));
    offB[s] = (unsigned)(DG_A_BYTES + (wn / 16) * 2048 + kt_ * 128 + ((((g >> 1) ^ (kt_ & 7)) & 7) << 4) + ((g & 1) << 3));
  }
  double acc[4][8][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
  for (int kt = 0; kt < NK; ++kt) {
    const unsigned f = fills + kt;
    if (tid == 0 && kt + (int)DG_NS - 1 < NK) issue(f + DG_NS - 1, kt + DG_NS - 1);
    mb_wait(fullb + 8 * (f % DG_NS), (f / DG_NS) & 1u);
    const unsigned char* sp = ring + (f % DG_NS) * DG_STAGE;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double af[4], bf[8];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = *reinterpret_cast<const double*>(sp + offA[ks] + mi * 1024);
#pragma unroll
      for (int nj = 0; nj < 8; ++nj)
        bf[nj] = *reinterpret_cast<const double*>(sp + ((offB[ks] + (nj >> 1) * 2048) ^ ((nj & 1) << 6)));
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 8; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
    }
    __syncwarp();
    if (lane == 0) mb_arrive(emptyb + 8 * (f % DG_NS));
  }
  fills += NK;
  // C - acc, rounded as gemm_tile's alpha = -1, beta = 1 epilogue
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 8; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double* dst = C + (int64_t)(wm + 8 * mi + g) * ldc + wn + 8 * nj + 2 * t + e;
        *dst = __dadd_rn(__ldcg(dst), -acc[mi][nj][e]);
      }
}
// A quarter of the look-ahead update: rows r0 .. r0 + 63, columns c0 .. c0 + 63 of tile (i, j),
// K = 128 (step k), on the same TMA ring: the A box (128 rows from row 128 i + r0; the first 64 are
// used) and four B boxes per stage, 8 warps of 16 x 32.
__device__ void dag_gemm_tma_quarter(const DagMaps& maps, int z, int i, int j, int k, int r0, int c0, double* C,
                                     int ldc, unsigned char* ring, unsigned fullb, unsigned emptyb, unsigned& fills) {
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wm = 16 * (warp >> 1), wn = 32 * (warp & 1);
  const unsigned base = su32(ring);
  constexpr int NK = 8;
  constexpr unsigned BYTES = DG_A_BYTES + 4 * 2048;
  auto issue = [&](unsigned f, int kt) {
    const unsigned s = f % DG_NS, sa = base + s * DG_STAGE, sb = sa + DG_A_BYTES, bar = fullb + 8 * s;
    if (f >= DG_NS) mb_wait(emptyb + 8 * s, ((f / DG_NS) - 1) & 1u);
    mb_expect(bar, BYTES);
    tma3(sa, &maps.a, 128 * k + 16 * kt, 128 * i + r0, z, bar);
#pragma unroll
    for (int q = 0; q < 4; ++q) tma3(sb + q * 2048, &maps.b, 128 * j + c0 + 16 * q, 128 * k + 16 * kt, z, bar);
  };
  if (tid == 0) {
    fence_proxy_async_all();
    for (int kt = 0; kt < (int)DG_NS - 1 && kt < NK; ++kt) issue(fills + kt, kt);
  }
  unsigned offA[4], offB[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int kt_ = 2 * (s & 1) + 8 * (s >> 1) + (t & 1) + 4 * (t >> 1);
    offA[s] = (unsigned)((wm + g) * 128 + ((((kt_ >> 1) ^ g) & 7) << 4) + ((kt_ & 1) << 3));
    offB[s] = (unsigned)(DG_A_BYTES + (wn / 16) * 2048 + kt_ * 128 + ((((g >> 1) ^ (kt_ & 7)) & 7) << 4) + ((g & 1) << 3));
  }
  double acc[2][4][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
  for (int kt = 0; kt < NK; ++kt) {
    const unsigned f = fills + kt;
    if (tid == 0 && kt + (int)DG_NS - 1 < NK) issue(f + DG_NS - 1, kt + DG_NS - 1);
    mb_wait(fullb + 8 * (f % DG_NS), (f / DG_NS) & 1u);
    const unsigned char* sp = ring + (f % DG_NS) * DG_STAGE;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double af[2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) af[mi] = *reinterpret_cast<const double*>(sp + offA[ks] + mi * 1024);
#pragma unroll
      for (int nj = 0; nj < 4; ++nj)
        bf[nj] = *reinterpret_cast<const double*>(sp + ((offB[ks] + (nj >> 1) * 2048) ^ ((nj & 1) << 6)));
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
    }
    __syncwarp();
    if (lane == 0) mb_arrive(emptyb + 8 * (f % DG_NS));
  }
  fills += NK;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double* dst = C + (int64_t)(r0 + wm + 8 * mi + g) * ldc + c0 + wn + 8 * nj + 2 * t + e;
        *dst = __dadd_rn(__ldcg(dst), -acc[mi][nj][e]);
      }
}
}  // namespace

size_t lu_dag_smem_bytes() {
  size_t b = lu_base128_smem_bytes();
  b = b > trsm128_smem_bytes() ? b : trsm128_smem_bytes();
  b = b > sizeof(GemmSmem<128, 128, 16>) ? b : sizeof(GemmSmem<128, 128, 16>);
  const size_t ring = DG_NS * DG_STAGE + 1024 + 64;  // the TMA ring (1024-aligned)
  return b > ring ? b : ring;
}

// optional per-task timeline (PF_DAG_TRACE, pf_large.cu): globaltimer at pull / start / end
__device__ long long* g_dag_trace = nullptr;
void set_dag_trace(long long* p) { cudaMemcpyToSymbol(g_dag_trace, &p, sizeof(p)); }
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256, 1) lu_dag_kernel(double* M, int np, int64_t strideM, double* inv,
                                                        int64_t inv_stride, const int4* tasks, int ntasks, int* next,
                                                        int* state, int nt, int* err,
                                                        const __grid_constant__ DagMaps maps, int use_tma) {
  extern __shared__ __align__(16) unsigned char dag_smem[];
  double* dsm = reinterpret_cast<double*>(dag_smem);
  __shared__ int s_task, s_ok;
  __shared__ __align__(8) unsigned long long ring_bar[2 * DG_NS];  // full[NS], empty[NS] of the G tasks' TMA ring
  constexpr int T = 128;
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dag_smem) + 1023) & ~uintptr_t(1023));
  const unsigned fullb = su32(&ring_bar[0]), emptyb = su32(&ring_bar[DG_NS]);
  unsigned fills = 0;
  if (use_tma && threadIdx.x == 0) {
    for (unsigned q = 0; q < DG_NS; ++q) {
      mb_init(fullb + 8 * q, 1);
      mb_init(emptyb + 8 * q, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(next, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= ntasks) return;
    long long* const trace = g_dag_trace;
    if (trace && threadIdx.x == 0) trace[3 * (int64_t)t] = gtimer();
    const int4 tk = tasks[t];
    // type (bits 24-27), part (bits 28-29: R / C tasks split into their two 64-wide chunks, the
    // look-ahead update of the next diagonal tile into four 64 x 64 quarters, so the critical path's
    // tasks run on several SMs each), system (bits 0-23)
    const int type = (tk.x >> 24) & 15, part = (tk.x >> 28) & 3, z = tk.x & 0xff, i = tk.y, j = tk.z, k = tk.w;
    const int k0 = type == 3 ? (tk.x >> 8) & 0xffff : k;  // a G task applies steps k0 .. k
    const bool quarter = type == 4;  // a quarter of G(k + 1, k + 1, k)
    int* st = state + (int64_t)z * nt * nt;
    // tile states count quarter-steps: an F or G task moves its tile from 4k to 4k + 4, each R / C
    // chunk adds 2, each G quarter 1
    if (threadIdx.x == 0) {
      // (an inverse task waits for the factored tile: F moved it to 4k + 2)
      bool ok = wait_ge(st + i * nt + j, type == 5 ? 4 * k + 2 : 4 * k0, err);  // steps 0 .. k0-1 received
      if (ok && (type == 1 || type == 2)) ok = wait_ge(st + k * nt + k, 4 * k + 4, err);  // F(k) done
      if (type == 3 || quarter)  // the L tiles (i, kk) and U tiles (kk, j) of every step applied
        for (int kk = k0; ok && kk <= k; ++kk)
          ok = wait_ge(st + i * nt + kk, 4 * kk + 4, err) && wait_ge(st + kk * nt + j, 4 * kk + 4, err);
      s_ok = ok;
    }
    __syncthreads();
    if (!s_ok) return;
    if (trace && threadIdx.x == 0) trace[3 * (int64_t)t + 1] = gtimer();
    double* Mz = M + (int64_t)z * strideM;
    double* dblk = Mz + (int64_t)T * k * np + T * k;  // diagonal tile of step k
    double* bi = inv + (int64_t)z * inv_stride + (int64_t)(2 * k) * 2 * B64 * B64;
    double* tile = Mz + (int64_t)T * i * np + T * j;
    if (type == 0) {
      lu128_block(dblk, np, bi, dsm, false);
    } else if (type == 5) {  // the L / U inverses of 64-half `part` of the factored diagonal tile
      inv64_block(dblk + (int64_t)B64 * part * np + B64 * part, np, bi + part * 2 * B64 * B64, dsm);
    } else if (type == 1 || type == 2) {  // one 64-column (R) / 64-row (C) chunk
      trsm128_chunk(dblk, np, bi, type == 1 ? 0 : 2, type == 1 ? tile + B64 * part : tile + (int64_t)B64 * part * np,
                    np, B64, dsm);
    } else if (quarter && use_tma) {  // rows / columns 64 (part >> 1) / 64 (part & 1) of the tile
      dag_gemm_tma_quarter(maps, z, i, j, k, B64 * (part >> 1), B64 * (part & 1), tile, np, ring, fullb, emptyb, fills);
    } else if (quarter) {  // rows / columns 64 (part >> 1) / 64 (part & 1) of the tile, K = 128
      const int r0 = B64 * (part >> 1), c0 = B64 * (part & 1);
      GemmParams p{};
      p.m = p.n = B64;
      p.k = T;
      p.batch = 1;
      p.alpha = -1.0;
      p.beta = 1.0;
      p.A = Mz + (int64_t)(T * i + r0) * np + T * k;
      p.lda = np;
      p.B = Mz + (int64_t)T * k * np + T * j + c0;
      p.ldb = np;
      p.C = tile + (int64_t)r0 * np + c0;
      p.ldc = np;
      gemm_tile<64, 64, 16, 16, 32, true>(p, *reinterpret_cast<GemmSmem<64, 64, 16>*>(dag_smem), 0, 0, 1);
    } else if (use_tma) {
      dag_gemm_tma(maps, z, i, j, k0, k - k0 + 1, tile, np, ring, fullb, emptyb, fills);
    } else {
      GemmParams p{};
      p.m = p.n = T;
      p.k = T * (k - k0 + 1);
      p.batch = 1;
      p.alpha = -1.0;
      p.beta = 1.0;
      p.A = Mz + (int64_t)T * i * np + T * k0;
      p.lda = np;
      p.B = Mz + (int64_t)T * k0 * np + T * j;
      p.ldb = np;
      p.C = tile;
      p.ldc = np;
      gemm_tile<128, 128, 16, 32, 64, true>(p, *reinterpret_cast<GemmSmem<128, 128, 16>*>(dag_smem), 0, 0, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (trace) trace[3 * (int64_t)t + 2] = gtimer();
      if (type == 1 || type == 2 || quarter || type == 5)
        atomicAdd(st + i * nt + j, quarter || type == 5 ? 1 : 2);  // ordered after the fence; the waiter acquires
      else
        st_release(st + i * nt + j, type == 0 ? 4 * k + 2 : 4 * k + 4);  // F: +2, its two inverse tasks +1 each
    }
  }
}
}  // namespace pf
