// Blocked partial-pivoting LU for n > 128 (DenseLu, dense.cpp:102-133): recursive (column-split)
// factorisation whose big work is the DMMA TRSM / GEMM of pf_large.cu, with two kernels here:
//
//   panel_lu_cluster_kernel  the rows [off, np) x columns [off, off + w) panel (w <= 64) of one system,
//                            factored column by column with the reference's pivot rule (strict '>'
//                            over the column, first maximum wins), row exchanges inside the panel,
//                            multipliers a * (1 / pivot), the f == 0 skip. The panel lives in the
//                            shared memory of a thread-block CLUSTER (up to 16 CTAs, DSMEM): each CTA
//                            owns a contiguous row range; per column one cluster barrier publishes the
//                            CTAs' candidates, every CTA reads them over DSMEM and agrees on the
//                            pivot, the pivot row is read once over DSMEM and the swap partner row is
//                            written back after a second barrier. No global-memory round trip per
//                            column (the unblocked fallback streamed the whole trailing matrix per
//                            column from one SM).
//   panel_lu_global_kernel   the same panel in global memory (one CTA) when it does not fit the
//                            cluster's shared memory.
//   laswp_kernel             applies a range of the swap sequence to a column range (LAPACK laswp).
//
// A failing pivot (best <= 1e-14 max|A|) records SingularShift (column, magnitude) for the system and
// stops its remaining panels; the host reports the first failure.
#include <climits>
#include <cstdlib>
#include <cooperative_groups.h>

#include "pf_common.cuh"
#include "pf_kernels.h"

namespace cg = cooperative_groups;

namespace pf {

namespace {
constexpr unsigned FULL = 0xffffffffu;
constexpr int PW = 64;        // panel width
constexpr int PLS = PW + 1;   // smem row stride (odd: column walks are conflict free)

__device__ __forceinline__ void better(double& bv, int& bi, double v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}
}  // namespace

size_t panel_lu_smem_bytes(int rows_per_cta) {
  return sizeof(double) * ((size_t)rows_per_cta * PLS + 2 * PW + 64) + sizeof(int) * 64;
}

// blockIdx.x = CTA within the cluster (rank), blockIdx.y = system. Rows [off + rank * R, ...).
__global__ void __launch_bounds__(512) panel_lu_cluster_kernel(double* M, int64_t ld, int64_t strideM, int np,
                                                                int off, int w, int R, int* piv, int npiv,
                                                                const double* tol, const int* zorig, int* failed,
                                                                DevStatus* status, int* first_error) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* P = reinterpret_cast<double*>(smem_raw);  // R x PLS
  double* prow = P + (size_t)R * PLS;               // the pivot row (after the swap: row col)
  double* oldc = prow + PW;                         // the old row col (goes to row p)
  double* cand_v = oldc + PW;                       // [0] this CTA's candidate
  int* cand_i = reinterpret_cast<int*>(cand_v + 64);
  const int z = blockIdx.y;
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int r_lo = off + rank * R;                  // first owned row
  const int r_hi = min(np, r_lo + R);
  const int nr = max(0, r_hi - r_lo);
  double* a = M + (int64_t)z * strideM;
  const bool dead = failed[z] != 0;  // an earlier panel of this system failed: nothing to do
  // load the owned rows of the panel
  for (int idx = threadIdx.x; idx < nr * w; idx += blockDim.x) {
    const int r = idx / w, c = idx % w;
    P[r * PLS + c] = a[(int64_t)(r_lo + r) * ld + off + c];
  }
  cluster.sync();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  bool singular = false;  // uniform over the cluster: every CTA reduces the same candidates
  for (int c = 0; c < w && !dead; ++c) {
    const int col = off + c;
    // ---- this CTA's candidate over its rows >= col (strict '>', smallest row on ties)
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = max(col, r_lo) - r_lo + threadIdx.x; r < nr; r += blockDim.x) better(bv, bi, fabs(P[r * PLS + c]), r_lo + r);
    for (int o = 16; o > 0; o >>= 1) better(bv, bi, __shfl_xor_sync(FULL, bv, o), __shfl_xor_sync(FULL, bi, o));
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < nw; ++q) better(bv, bi, red_v[q], red_i[q]);
      cand_v[0] = bv;
      cand_i[0] = bi;
    }
    cluster.sync();  // (1) every candidate published
    // ---- the pivot: every CTA reduces the same candidates in the same order
    double gv = -1.0;
    int gi = INT_MAX;
    for (int q = 0; q < C; ++q) {
      const double* cv = cluster.map_shared_rank(cand_v, q);
      const int* ci = cluster.map_shared_rank(cand_i, q);
      better(gv, gi, cv[0], ci[0]);
    }
    if (gv <= tol[z]) {  // SingularShift (dense.cpp:116-119), reported once
      if (rank == 0 && threadIdx.x == 0) {
        status[zorig[z]].code = PF_ERR_SINGULAR_SHIFT;
        status[zorig[z]].column = col;
        status[zorig[z]].pivot_magnitude = gv;
        failed[z] = 1;
        atomicMin(first_error, zorig[z]);
      }
      singular = true;
      break;
    }
    const int p = gi;
    const int own_p = (p - off) / R, own_c = (col - off) / R;
    // the pivot row (and, for its new owner, the old row col) over DSMEM
    {
      const double* src = cluster.map_shared_rank(P, own_p) + (size_t)(p - off - own_p * R) * PLS;
      for (int j = threadIdx.x; j < w; j += blockDim.x) prow[j] = src[j];
      if (rank == own_p && p != col) {
        const double* s2 = cluster.map_shared_rank(P, own_c) + (size_t)(col - off - own_c * R) * PLS;
        for (int j = threadIdx.x; j < w; j += blockDim.x) oldc[j] = s2[j];
      }
    }
    cluster.sync();  // (2) all reads done before the swap writes
    if (p != col) {
      if (rank == own_c)
        for (int j = threadIdx.x; j < w; j += blockDim.x) P[(size_t)(col - r_lo) * PLS + j] = prow[j];
      if (rank == own_p)
        for (int j = threadIdx.x; j < w; j += blockDim.x) P[(size_t)(p - r_lo) * PLS + j] = oldc[j];
    }
    if (rank == 0 && threadIdx.x == 0) piv[(int64_t)z * npiv + col] = p;
    __syncthreads();
    // ---- multipliers f = a * (1 / pivot) and the rank-1 update of the owned rows below col
    const double inv_piv = 1.0 / prow[c];
    const int r0 = max(col + 1, r_lo) - r_lo;
    const int wc = w - c - 1;
    for (int r = r0 + threadIdx.x; r < nr; r += blockDim.x) P[r * PLS + c] = __dmul_rn(P[r * PLS + c], inv_piv);
    __syncthreads();
    if (wc > 0)
      for (int idx = threadIdx.x; idx < (nr - r0) * wc; idx += blockDim.x) {
        const int r = r0 + idx / wc, j = c + 1 + idx % wc;
        const double f = P[r * PLS + c];
        if (f != 0.0) P[r * PLS + j] = __dsub_rn(P[r * PLS + j], __dmul_rn(f, prow[j]));
      }
    __syncthreads();
  }
  cluster.sync();  // no CTA leaves while others may still read its shared memory
  if (dead || singular) return;
  for (int idx = threadIdx.x; idx < nr * w; idx += blockDim.x) {
    const int r = idx / w, c = idx % w;
    a[(int64_t)(r_lo + r) * ld + off + c] = P[r * PLS + c];
  }
}

// The same panel in global memory, one CTA per system (fallback for panels taller than the
// cluster's shared memory).
__global__ void __launch_bounds__(1024) panel_lu_global_kernel(double* M, int64_t ld, int64_t strideM, int np,
                                                                int off, int w, int* piv, int npiv, const double* tol,
                                                                const int* zorig, int* failed, DevStatus* status,
                                                                int* first_error) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_p;
  __shared__ double s_best;
  const int z = blockIdx.x;
  if (failed[z]) return;
  double* a = M + (int64_t)z * strideM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = 0; c < w; ++c) {
    const int col = off + c;
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = col + threadIdx.x; r < np; r += blockDim.x) better(bv, bi, fabs(a[(int64_t)r * ld + col]), r);
    for (int o = 16; o > 0; o >>= 1) better(bv, bi, __shfl_xor_sync(FULL, bv, o), __shfl_xor_sync(FULL, bi, o));
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < nw; ++q) better(bv, bi, red_v[q], red_i[q]);
      s_best = bv;
      s_p = bi;
    }
    __syncthreads();
    const int p = s_p;
    if (s_best <= tol[z]) {
      if (threadIdx.x == 0) {
        status[zorig[z]].code = PF_ERR_SINGULAR_SHIFT;
        status[zorig[z]].column = col;
        status[zorig[z]].pivot_magnitude = s_best;
        failed[z] = 1;
        atomicMin(first_error, zorig[z]);
      }
      return;
    }
    if (p != col)
      for (int j = threadIdx.x; j < w; j += blockDim.x) {
        const double t = a[(int64_t)p * ld + off + j];
        a[(int64_t)p * ld + off + j] = a[(int64_t)col * ld + off + j];
        a[(int64_t)col * ld + off + j] = t;
      }
    if (threadIdx.x == 0) piv[(int64_t)z * npiv + col] = p;
    __syncthreads();
    const double inv_piv = 1.0 / a[(int64_t)col * ld + col];
    for (int r = col + 1 + threadIdx.x; r < np; r += blockDim.x)
      a[(int64_t)r * ld + col] = __dmul_rn(a[(int64_t)r * ld + col], inv_piv);
    __syncthreads();
    const int wc = w - c - 1;
    if (wc > 0)
      for (int64_t idx = threadIdx.x; idx < (int64_t)(np - col - 1) * wc; idx += blockDim.x) {
        const int r = col + 1 + (int)(idx / wc), j = col + 1 + (int)(idx % wc);
        const double f = a[(int64_t)r * ld + col];
        if (f != 0.0) a[(int64_t)r * ld + j] = __dsub_rn(a[(int64_t)r * ld + j], __dmul_rn(f, a[(int64_t)col * ld + j]));
      }
    __syncthreads();
  }
}

// Swaps k = k0 .. k1-1 of every system's sequence applied in order to columns [c0, c1): one thread per
// column, the rows of each swap contiguous across the warp.
__global__ void laswp_kernel(double* M, int64_t ld, int64_t strideM, const int* piv, int npiv, int k0, int k1, int c0,
                             int c1, const int* failed) {
  const int z = blockIdx.y;
  if (failed && failed[z]) return;
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double* a = M + (int64_t)z * strideM;
  const int* pz = piv + (int64_t)z * npiv;
  for (int k = k0; k < k1; ++k) {
    const int p = pz[k];
    if (p != k) {
      const double t = a[(int64_t)p * ld + c];
      a[(int64_t)p * ld + c] = a[(int64_t)k * ld + c];
      a[(int64_t)k * ld + c] = t;
    }
  }
}

cudaError_t launch_panel_lu(double* M, int64_t ld, int64_t strideM, int np, int off, int w, int nsys, int* piv,
                            int npiv, const double* tol, const int* zorig, int* failed, DevStatus* status,
                            int* first_error, cudaStream_t stream) {
  const int rows = np - off;
  // smallest cluster whose CTAs hold <= 384 rows each (<= 197 KB of shared memory), up to 16 CTAs
  int C = 1;
  while (C < 16 && (rows + C - 1) / C > 384) C *= 2;
  const int R = (rows + C - 1) / C;
  static const bool no_cluster = std::getenv("PF_PANEL_GLOBAL") != nullptr;
  if (R <= 384 && !no_cluster) {
    const size_t smem = panel_lu_smem_bytes(R);
    static bool attrs = false;
    if (!attrs) {
      cudaFuncSetAttribute(panel_lu_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      attrs = true;
    }
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(panel_lu_cluster_kernel),
                                       (int)panel_lu_smem_bytes(384));
    if (e == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C, nsys);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e = cudaLaunchKernelEx(&cfg, panel_lu_cluster_kernel, M, ld, strideM, np, off, w, R, piv, npiv, tol, zorig,
                             failed, status, first_error);
      if (e == cudaSuccess) return e;
    }
    cudaGetLastError();  // cluster launch unavailable: the global-memory panel
  }
  panel_lu_global_kernel<<<nsys, 1024, 0, stream>>>(M, ld, strideM, np, off, w, piv, npiv, tol, zorig, failed, status,
                                                    first_error);
  return cudaGetLastError();
}

void launch_laswp(double* M, int64_t ld, int64_t strideM, const int* piv, int npiv, int k0, int k1, int c0, int c1,
                  int nsys, const int* failed, cudaStream_t stream) {
  if (k1 <= k0 || c1 <= c0 || nsys == 0) return;
  laswp_kernel<<<dim3((c1 - c0 + 127) / 128, nsys), 128, 0, stream>>>(M, ld, strideM, piv, npiv, k0, k1, c0, c1,
                                                                       failed);
}

}  // namespace pf
