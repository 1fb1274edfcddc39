// Blocked partial-pivoting LU for n > 128 (DenseLu, dense.cpp:102-133): recursive (column-split)
// factorisation whose big work is the DMMA TRSM / GEMM of pf_large.cu, with these kernels:
//
//   panel_lu_reg_kernel      (the default for 64-wide panels of up to 4096 rows) the rows [off, np) x
//                            columns [off, off + 64) of one system, factored column by column with the
//                            reference's pivot rule (the largest |a| of the column, the first such row
//                            in the current row order on ties), multipliers a * (1 / pivot) and the
//                            f == 0 skip. One row per thread, its 64 values in registers, a thread-block
//                            CLUSTER of up to 16 CTAs of 256 rows. Row exchanges are not moved: every
//                            row carries its current position in the exchanged order (the reference's
//                            full-row swaps are a permutation of these positions), and the pivot row
//                            of a column is final from then on. Per column: a redux argmax per warp,
//                            one CTA barrier, the CTA's candidate pushed into every CTA's shared memory
//                            by st.async with mbarrier completion (details at the kernel). Rows are
//                            written back in exchanged order and the moves listed for row_move_kernel.
//   panel_lu_cluster_kernel  the same panel in the clusters' shared memory (narrower panels, or up to
//                            16 x 384 rows).
//   panel_lu_global_kernel   the same panel in global memory, one CTA (anything taller).
//   row_move_kernel          applies a panel's row moves (at most 2 w rows) to every column outside the
//                            panel: after each panel the whole matrix has the reference's row order.
//
// A failing pivot (best <= 1e-14 max|A|) records SingularShift (column, magnitude) for the system and
// stops its remaining panels; the host reports the first failure.
#include <climits>
#include <cooperative_groups.h>
#include <cstdlib>

#include "pf_common.cuh"
#include "pf_kernels.h"

namespace cg = cooperative_groups;

namespace pf {

namespace {
constexpr unsigned FULL = 0xffffffffu;
constexpr int PW = 64;       // panel width
constexpr int PLS = PW + 1;  // smem row stride (odd: column walks are conflict free)
constexpr int PT = 256;      // threads per panel CTA
constexpr int MAX_ROWS_PER_CTA = 384;

// candidate order: larger |a|, then the earlier row in the exchanged order
__device__ __forceinline__ void better(double& bv, int& bl, int& br, double v, int l, int r) {
  if (v > bv || (v == bv && l < bl)) {
    bv = v;
    bl = l;
    br = r;
  }
}

struct PanelShared {
  double cand_v[2];
  int cand_l[2];        // exchanged-order position (relative to off)
  int cand_r[2];        // local row in the owning CTA
  double crow[2][PW];   // the candidate row's values (read by every CTA over DSMEM)
  double cv[16];        // the cluster's candidates, gathered
  int cl[16];
};
}  // namespace

size_t panel_lu_smem_bytes(int rows_per_cta) {
  return sizeof(double) * ((size_t)rows_per_cta * PLS + 16 * PW) + sizeof(int) * 2 * (size_t)rows_per_cta +
         sizeof(PanelShared) + 64;
}

// blockIdx.x = CTA within the cluster (rank), blockIdx.y = system. Physical rows [off + rank R, ...).
// moves[z * 2 PW ...]: (dst, src) absolute row pairs, count in moves_n[z].
__global__ void __launch_bounds__(PT) panel_lu_cluster_kernel(double* M, int64_t ld, int64_t strideM, int np,
                                                               int off, int w, int R, int* piv, int npiv,
                                                               const double* tol, const int* zorig, int* failed,
                                                               DevStatus* status, int* first_error, int2* moves,
                                                               int* moves_n) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* P = reinterpret_cast<double*>(smem_raw);  // R x PLS
  double* rows_buf = P + (size_t)R * PLS;           // 16 x PW: the cluster's candidate rows, gathered
  int* pos = reinterpret_cast<int*>(rows_buf + 16 * PW);  // exchanged-order position of each owned row
  int* done = pos + R;                              // 1 once the row is a pivot row
  PanelShared& sh = *reinterpret_cast<PanelShared*>(done + R);
  __shared__ double red_v[PT / 32];
  __shared__ int red_l[PT / 32], red_r[PT / 32];
  const int z = blockIdx.y;
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int r_lo = rank * R;  // relative to off
  const int nr = max(0, min(np - off, r_lo + R) - r_lo);
  double* a = M + (int64_t)z * strideM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool dead = failed[z] != 0;  // an earlier panel of this system failed: nothing to do
  for (int idx = tid; idx < nr * w; idx += PT) {
    const int r = idx / w, c = idx - r * w;
    P[r * PLS + c] = a[(int64_t)(off + r_lo + r) * ld + off + c];
  }
  for (int r = tid; r < nr; r += PT) {
    pos[r] = r_lo + r;
    done[r] = 0;
  }
  if (tid == 0 && rank == 0) moves_n[z] = 0;
  cluster.sync();
  bool singular = false;
  const int uj = tid & (PW - 1), ur = tid / PW;  // update mapping: column lane, row phase
  double inv_prev = 0.0;                          // 1 / pivot of the previous column
  // Four barriers per column (one of them cluster-wide). The multipliers of column c are scaled in
  // column c + 1's first phase (the update of column c computes f = a * (1 / pivot) itself), so no
  // barrier separates the scaling from the update.
  for (int c = 0; c < w && !dead; ++c) {
    const int slot = c & 1;
    // ---- (A) column c - 1's multipliers; this CTA's candidate among its rows not yet pivoted
    double bv = -1.0;
    int bl = INT_MAX, br = -1;
    for (int r = tid; r < nr; r += PT) {
      if (done[r]) continue;
      if (c > 0) P[r * PLS + c - 1] = __dmul_rn(P[r * PLS + c - 1], inv_prev);
      better(bv, bl, br, fabs(P[r * PLS + c]), pos[r], r);
    }
    for (int o = 16; o > 0; o >>= 1)
      better(bv, bl, br, __shfl_xor_sync(FULL, bv, o), __shfl_xor_sync(FULL, bl, o), __shfl_xor_sync(FULL, br, o));
    if (lane == 0) {
      red_v[warp] = bv;
      red_l[warp] = bl;
      red_r[warp] = br;
    }
    __syncthreads();
    // ---- (B) warp 0: the CTA's candidate and a copy of its row
    if (warp == 0) {
      bv = lane < PT / 32 ? red_v[lane] : -1.0;
      bl = lane < PT / 32 ? red_l[lane] : INT_MAX;
      br = lane < PT / 32 ? red_r[lane] : -1;
      for (int o = 16; o > 0; o >>= 1)
        better(bv, bl, br, __shfl_xor_sync(FULL, bv, o), __shfl_xor_sync(FULL, bl, o), __shfl_xor_sync(FULL, br, o));
      if (lane == 0) {
        sh.cand_v[slot] = bv;
        sh.cand_l[slot] = bl;
        sh.cand_r[slot] = br;
      }
      if (br >= 0)
        for (int j = lane; j < w; j += 32) sh.crow[slot][j] = P[br * PLS + j];
    }
    if (C > 1)
      cluster.sync();  // every CTA's candidate and its row published (slot c & 1)
    else
      __syncthreads();
    // ---- (C) one DSMEM round trip: every candidate row and value, in parallel
    for (int t = tid; t < C * PW; t += PT) {
      const PanelShared* o = C > 1 ? cluster.map_shared_rank(&sh, t / PW) : &sh;
      const int j = t % PW;
      if (j < w) rows_buf[t] = o->crow[slot][j];
      if (j == 0) {
        sh.cv[t / PW] = o->cand_v[slot];
        sh.cl[t / PW] = o->cand_l[slot];
      }
    }
    __syncthreads();
    // ---- (D) the pivot (every thread reduces the same C candidates in the same order), the
    // exchange c <-> p of the positions, and the rank-1 update of the rows not yet pivoted
    double gv = -1.0;
    int p = INT_MAX, q = -1;
    for (int k = 0; k < C; ++k) better(gv, p, q, sh.cv[k], sh.cl[k], k);
    if (gv <= tol[z]) {  // SingularShift (dense.cpp:116-119), reported once
      if (rank == 0 && tid == 0) {
        status[zorig[z]].code = PF_ERR_SINGULAR_SHIFT;
        status[zorig[z]].column = off + c;
        status[zorig[z]].pivot_magnitude = gv;
        failed[z] = 1;
        atomicMin(first_error, zorig[z]);
      }
      singular = true;
      break;
    }
    const double* prow = rows_buf + q * PW;  // the pivot row, final from now on
    const int my_r = rank == q ? sh.cand_r[slot] : -1;  // the pivot row, if it is this CTA's
    for (int r = tid; r < nr; r += PT) {
      if (r == my_r) {
        pos[r] = c;
        done[r] = 1;  // (the update below excludes my_r explicitly)
      } else if (pos[r] == c) {
        pos[r] = p;
      }
    }
    if (rank == 0 && tid == 0) piv[(int64_t)z * npiv + off + c] = off + p;
    const double inv_piv = 1.0 / prow[c];
    const int j = c + 1 + uj;
    if (j < w) {
      const double u = prow[j];
      for (int r = ur; r < nr; r += PT / PW) {
        if (done[r] || r == my_r) continue;
        const double f = __dmul_rn(P[r * PLS + c], inv_piv);
        if (f != 0.0) P[r * PLS + j] = __dsub_rn(P[r * PLS + j], __dmul_rn(f, u));
      }
    }
    __syncthreads();
    inv_prev = inv_piv;
  }
  // the last column's multipliers
  if (!dead && !singular && w > 0) {
    __syncthreads();
    for (int r = tid; r < nr; r += PT)
      if (!done[r]) P[r * PLS + w - 1] = __dmul_rn(P[r * PLS + w - 1], inv_prev);
    __syncthreads();
  }
  cluster.sync();  // no CTA leaves while others may still read its shared memory
  if (dead || singular) return;
  // write back in exchanged order; list the moved rows for the columns outside the panel
  for (int idx = tid; idx < nr * w; idx += PT) {
    const int r = idx / w, c = idx - r * w;
    a[(int64_t)(off + pos[r]) * ld + off + c] = P[r * PLS + c];
  }
  for (int r = tid; r < nr; r += PT)
    if (pos[r] != r_lo + r) {
      const int k = atomicAdd(moves_n + z, 1);
      moves[(int64_t)z * 2 * PW + k] = make_int2(off + pos[r], off + r_lo + r);
    }
}

// The panel in REGISTERS: one row per thread (256 rows per CTA, up to 16 CTAs per cluster: panels of
// up to 4096 rows). Each thread keeps its row's 64 values in registers for the whole panel, so the
// rank-1 update of a column is register FMAs against the pivot row (read from shared memory as a
// broadcast). Per column: each warp's candidate (shuffles) stages its row in shared memory, ONE CTA
// barrier, every warp reduces the 8 warp candidates to the CTA's (whose row is already staged). With
// one CTA that is the pivot. In a cluster the CTA's candidate (value, position, row) is pushed into
// every CTA's slot [parity][rank] with st.async (remote stores that complete a transaction count on
// the receiver's mbarrier), and each CTA waits on its own mbarrier only -- no cluster-wide barrier
// per column; every CTA then picks the pivot from its local copies. All buffers are double-buffered
// by column parity: a slot of column c is rewritten at c + 2 only after every reader passed the
// barrier (or the exchange) of column c + 1.
// Register indices are compile-time constants: the column value is picked by a uniform switch, the
// update runs over the 8-column block containing c (predicated j > c) and the blocks after it.
constexpr int RT = 256;  // threads (= rows) per CTA
constexpr int RW = RT / 32;
constexpr int CW = PW + 4;                       // candidate payload (doubles): row, {key, pos}, {1/pivot, -}
constexpr unsigned kCandBytes = 8u * CW;
struct RegPanelShared {
  double wrows[2][RW][CW];  // [parity][warp] each warp's candidate payload
  double rows[2][16][CW];   // [parity][rank] the cluster's candidate payloads
  unsigned long long red_key[2][RW];
  unsigned red_pos[2][RW];
  unsigned long long bar[2];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cluster_addr(const void* p, int q) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(q));
  return r;
}
__device__ __forceinline__ void st_async2(unsigned addr, double x, double y, unsigned bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(x), "d"(y), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void cbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Candidate order as a 64-bit key: |a| + 1 ulp-steps above the "no candidate" key 0 (pivot rows,
// rows past the matrix, NaN); larger |a| wins, then the smaller position (the reference's strict
// '>' over rows in order). The argmax over a warp is three redux instructions and a ballot.
__device__ __forceinline__ unsigned long long cand_key(double x, bool live) {
  const double ax = fabs(x);
  return (live && ax >= 0.0) ? (unsigned long long)__double_as_longlong(ax) + 1ull : 0ull;
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  return k == 0ull ? -1.0 : __longlong_as_double((long long)(k - 1ull));
}
// the lane holding the best (key, pos); every lane gets the same answer
__device__ __forceinline__ int lane_argmax(unsigned long long key, unsigned pos) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(FULL, hi);
  const unsigned mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
  const bool c = hi == mhi && lo == mlo;
  const unsigned mp = __reduce_min_sync(FULL, c ? pos : 0xFFFFFFFFu);
  return __ffs(__ballot_sync(FULL, c && pos == mp)) - 1;
}

// v[c] <- f (the multiplier) and v[j] -= f prow[j] for j > c (skipped when f == 0); nx <- the new
// v[c + 1] (the next column's value, so the next step needs no dynamic register index); B = c / 8
template <int B>
__device__ __forceinline__ void update_from_block(double (&v)[PW], int c, double f, const double* prow, double& nx) {
  const bool nz = f != 0.0;
#pragma unroll
  for (int j = 8 * B; j < PW; ++j) {
    if (j > c && nz) v[j] = __dsub_rn(v[j], __dmul_rn(f, prow[j]));
    if (j < 8 * B + 8 && j == c) v[j] = f;
    if (j < 8 * B + 9 && j == c + 1) nx = v[j];
  }
}

// the candidate row's columns [8 B, 64) into the staging slot (16-byte stores)
template <int B>
__device__ __forceinline__ void stage_from_block(const double (&v)[PW], double2* w2) {
#pragma unroll
  for (int j = 4 * B; j < PW / 2; ++j) w2[j] = make_double2(v[2 * j], v[2 * j + 1]);
}

// ASYNC: candidates exchanged by st.async into the receivers' mbarriers; otherwise plain remote
// stores and one cluster barrier per column (the A/B variant, PF_PANEL_CLUSTER_SYNC). Per column:
// each warp's argmax (redux) -- its winner stages (row, key, position, 1/pivot) in shared memory --
// ONE CTA barrier, every warp reduces the 8 warp candidates the same way; in a cluster the CTA's
// candidate goes to every CTA's slot [parity][rank] and each CTA waits on its own mbarrier only.
// The reciprocal of a candidate pivot is computed by its owner before the exchange (off the chain).
// Buffers are double-buffered by column parity: a slot of column c is rewritten at c + 2 only after
// every reader passed the barrier (or the exchange) of column c + 1.
template <bool ASYNC>
__global__ void __launch_bounds__(RT, 1) panel_lu_reg_kernel(double* M, int64_t ld, int64_t strideM, int np, int off,
                                                             int* piv, int npiv, const double* tol, const int* zorig,
                                                             int* failed, DevStatus* status, int* first_error,
                                                             int2* moves, int* moves_n) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ __align__(16) RegPanelShared sh;
  const int z = blockIdx.y;
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = rank * RT + tid;  // relative to off
  const bool have = row < np - off;
  double* a = M + (int64_t)z * strideM;
  const bool dead = failed[z] != 0;
  double v[PW];
  if (have) {
    const double2* src = reinterpret_cast<const double2*>(a + (int64_t)(off + row) * ld + off);
#pragma unroll
    for (int j = 0; j < PW / 2; ++j) {
      const double2 t = src[j];
      v[2 * j] = t.x;
      v[2 * j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < PW; ++j) v[j] = 0.0;
  }
  int pos = row;      // position in the exchanged order
  bool done = !have;  // pivot rows (and rows past the matrix) take no further part
  double vc = v[0];   // the current column's value
  if (tid == 0 && rank == 0) moves_n[z] = 0;
  if (ASYNC && C > 1 && tid == 0) {
    cbar_init(smem_u32(&sh.bar[0]), 1);
    cbar_init(smem_u32(&sh.bar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    cbar_expect(smem_u32(&sh.bar[0]), kCandBytes * C);  // columns 0 and 1
    cbar_expect(smem_u32(&sh.bar[1]), kCandBytes * C);
  }
  cluster.sync();
  bool singular = false;
  // the column loop stays rolled (a fully unrolled panel is instruction-fetch bound); uniform over
  // the cluster, so no thread diverges from the barriers
#pragma unroll 1
  for (int c = 0; c < PW; ++c) {
    if (dead || singular) continue;
    const int par = c & 1;
    // ---- this warp's candidate: the winner stages its payload; then the CTA's
    const unsigned long long key = cand_key(vc, !done);
    const int wl = lane_argmax(key, done ? 0xFFFFFFFFu : (unsigned)pos);
    if (lane == wl) {
      double2* w2 = reinterpret_cast<double2*>(sh.wrows[par][warp]);
      // only columns >= 8 (c / 8) are read by the update (the earlier ones are final multipliers)
      switch (c >> 3) {
        case 0: stage_from_block<0>(v, w2); break;
        case 1: stage_from_block<1>(v, w2); break;
        case 2: stage_from_block<2>(v, w2); break;
        case 3: stage_from_block<3>(v, w2); break;
        case 4: stage_from_block<4>(v, w2); break;
        case 5: stage_from_block<5>(v, w2); break;
        case 6: stage_from_block<6>(v, w2); break;
        default: stage_from_block<7>(v, w2); break;
      }
      w2[PW / 2] = make_double2(__longlong_as_double((long long)key), __longlong_as_double((long long)(((unsigned long long)(unsigned)pos << 32) | (unsigned)tid)));
      w2[PW / 2 + 1] = make_double2(1.0 / vc, 0.0);
      sh.red_key[par][warp] = key;
      sh.red_pos[par][warp] = done ? 0xFFFFFFFFu : (unsigned)pos;
    }
    __syncthreads();
    const int ww = lane_argmax(lane < RW ? sh.red_key[par][lane] : 0ull, lane < RW ? sh.red_pos[par][lane] : 0xFFFFFFFFu);
    const double* prow = sh.wrows[par][ww];
    if (C > 1) {
      // ---- exchange: the CTA's candidate payload into every CTA's slot [par][rank]
      constexpr int E = CW / 2;  // 16-byte pieces per payload
      const double2* c2 = reinterpret_cast<const double2*>(prow);
      if (ASYNC) {
        for (int k = tid; k < C * E; k += RT) {
          const int q = k / E, e = k - q * E;
          const double2 t = c2[e];
          st_async2(cluster_addr(&sh.rows[par][rank][2 * e], q), t.x, t.y, cluster_addr(&sh.bar[par], q));
        }
        cbar_wait(smem_u32(&sh.bar[par]), (c >> 1) & 1);
        if (tid == 0 && c + 2 < PW) cbar_expect(smem_u32(&sh.bar[par]), kCandBytes * C);
      } else {
        for (int k = tid; k < C * E; k += RT) {
          const int q = k / E, e = k - q * E;
          RegPanelShared* o = cluster.map_shared_rank(&sh, q);
          reinterpret_cast<double2*>(o->rows[par][rank])[e] = c2[e];
        }
        cluster.sync();  // release / acquire: every pushed candidate is visible to every CTA
      }
      // ---- the pivot, from the local copies (every warp reduces the same C candidates)
      const double* meta = sh.rows[par][lane < C ? lane : 0] + PW;
      const unsigned long long mk = lane < C ? (unsigned long long)__double_as_longlong(meta[0]) : 0ull;
      const unsigned mpos = lane < C ? (unsigned)((unsigned long long)__double_as_longlong(meta[1]) >> 32) : 0xFFFFFFFFu;
      prow = sh.rows[par][lane_argmax(mk, mk ? mpos : 0xFFFFFFFFu)];
    }
    const unsigned long long pk = (unsigned long long)__double_as_longlong(prow[PW]);
    const unsigned long long pm = (unsigned long long)__double_as_longlong(prow[PW + 1]);
    const double gv = key_value(pk);
    const int p = (int)(pm >> 32);
    const bool me = !done && (unsigned)pos == (unsigned)p && pk != 0ull;
    if (gv <= tol[z]) {
      if (rank == 0 && tid == 0) {
        status[zorig[z]].code = PF_ERR_SINGULAR_SHIFT;
        status[zorig[z]].column = off + c;
        status[zorig[z]].pivot_magnitude = gv;
        failed[z] = 1;
        atomicMin(first_error, zorig[z]);
      }
      singular = true;
      continue;
    }
    if (rank == 0 && tid == 0) piv[(int64_t)z * npiv + off + c] = off + p;
    if (me) {
      pos = c;
      done = true;
    } else if (!done) {
      if (pos == c) pos = p;
      const double f = __dmul_rn(vc, prow[PW + 2]);  // a * (1 / pivot)
      double nx = 0.0;
      switch (c >> 3) {
        case 0: update_from_block<0>(v, c, f, prow, nx); break;
        case 1: update_from_block<1>(v, c, f, prow, nx); break;
        case 2: update_from_block<2>(v, c, f, prow, nx); break;
        case 3: update_from_block<3>(v, c, f, prow, nx); break;
        case 4: update_from_block<4>(v, c, f, prow, nx); break;
        case 5: update_from_block<5>(v, c, f, prow, nx); break;
        case 6: update_from_block<6>(v, c, f, prow, nx); break;
        default: update_from_block<7>(v, c, f, prow, nx); break;
      }
      vc = nx;
    } else if (pos == c) {
      pos = p;
    }
  }
  cluster.sync();  // no CTA leaves while others may still write into its shared memory
  if (dead || singular || !have) return;
  double2* dst = reinterpret_cast<double2*>(a + (int64_t)(off + pos) * ld + off);
#pragma unroll
  for (int j = 0; j < PW / 2; ++j) dst[j] = make_double2(v[2 * j], v[2 * j + 1]);
  if (pos != row) {
    const int k = atomicAdd(moves_n + z, 1);
    moves[(int64_t)z * 2 * PW + k] = make_int2(off + pos, off + row);
  }
}

// The same panel in global memory, one CTA per system (panels taller than the cluster's shared
// memory): explicit exchanges inside the panel columns, the moves listed from the swap sequence.
__global__ void __launch_bounds__(1024) panel_lu_global_kernel(double* M, int64_t ld, int64_t strideM, int np,
                                                                int off, int w, int* piv, int npiv, const double* tol,
                                                                const int* zorig, int* failed, DevStatus* status,
                                                                int* first_error, int2* moves, int* moves_n) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_p;
  __shared__ double s_best;
  __shared__ int rows[2 * PW], srcs[2 * PW], nrow;
  const int z = blockIdx.x;
  if (failed[z]) return;
  double* a = M + (int64_t)z * strideM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) nrow = 0;
  for (int c = 0; c < w; ++c) {
    const int col = off + c;
    double bv = -1.0;
    int bi = INT_MAX, dummy = 0;
    for (int r = col + threadIdx.x; r < np; r += blockDim.x) better(bv, bi, dummy, fabs(a[(int64_t)r * ld + col]), r, r);
    for (int o = 16; o > 0; o >>= 1)
      better(bv, bi, dummy, __shfl_xor_sync(FULL, bv, o), __shfl_xor_sync(FULL, bi, o), 0);
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < nw; ++q) better(bv, bi, dummy, red_v[q], red_i[q], 0);
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
    if (threadIdx.x == 0) {
      piv[(int64_t)z * npiv + col] = p;
      // track where each touched row's original content now is: rows[] holds the touched rows,
      // srcs[] the original row whose data sits there
      int ic = -1, ip = -1;
      for (int t = 0; t < nrow; ++t) {
        if (rows[t] == col) ic = t;
        if (rows[t] == p) ip = t;
      }
      if (ic < 0) {
        ic = nrow++;
        rows[ic] = col;
        srcs[ic] = col;
      }
      if (ip < 0) {
        ip = nrow++;
        rows[ip] = p;
        srcs[ip] = p;
      }
      const int t = srcs[ic];
      srcs[ic] = srcs[ip];
      srcs[ip] = t;
    }
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
  if (threadIdx.x == 0) {
    int k = 0;
    for (int t = 0; t < nrow; ++t)
      if (rows[t] != srcs[t]) moves[(int64_t)z * 2 * PW + k++] = make_int2(rows[t], srcs[t]);
    moves_n[z] = k;
  }
}

// The panel's row moves (dst <- src) applied to the columns outside [off, off + w): CTA = 32 columns
// of one system; all sources are read into shared memory before any destination is written.
constexpr int MC = 32;
__global__ void __launch_bounds__(256) row_move_kernel(double* M, int64_t ld, int64_t strideM, int np, int off, int w,
                                                       const int2* moves, const int* moves_n, const int* failed) {
  __shared__ double buf[2 * PW][MC + 1];
  __shared__ int2 mv[2 * PW];
  const int z = blockIdx.y;
  if (failed[z]) return;
  const int cnt = moves_n[z];
  if (cnt == 0) return;
  const int c0 = blockIdx.x * MC;
  if (c0 >= off && c0 + MC <= off + w) return;  // entirely inside the panel (already in order)
  double* a = M + (int64_t)z * strideM;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) mv[i] = moves[(int64_t)z * 2 * PW + i];
  __syncthreads();
  const int cc = threadIdx.x & (MC - 1), r0 = threadIdx.x / MC;
  const int c = c0 + cc;
  const bool live = c < np && (c < off || c >= off + w);
  for (int i = r0; i < cnt; i += 256 / MC)
    if (live) buf[i][cc] = a[(int64_t)mv[i].y * ld + c];
  __syncthreads();
  for (int i = r0; i < cnt; i += 256 / MC)
    if (live) a[(int64_t)mv[i].x * ld + c] = buf[i][cc];
}

cudaError_t launch_panel_lu(double* M, int64_t ld, int64_t strideM, int np, int off, int w, int nsys, int* piv,
                            int npiv, const double* tol, const int* zorig, int* failed, DevStatus* status,
                            int* first_error, int2* moves, int* moves_n, cudaStream_t stream,
                            cudaEvent_t panel_done) {
  const int rows = np - off;
  static const bool no_reg = std::getenv("PF_PANEL_SMEM") != nullptr;  // A/B: the shared-memory panel
  if (w == PW && rows <= 16 * RT && !no_reg) {
    int Cr = 1;
    while (Cr * RT < rows) Cr *= 2;
    static const bool csync = std::getenv("PF_PANEL_CLUSTER_SYNC") != nullptr;  // A/B: one cluster barrier per column
    auto kern = csync ? panel_lu_reg_kernel<false> : panel_lu_reg_kernel<true>;
    static bool attr_r = false;
    if (!attr_r) {
      cudaFuncSetAttribute(panel_lu_reg_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(panel_lu_reg_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      attr_r = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(Cr, nsys);
    cfg.blockDim = dim3(RT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Cr;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t er = cudaLaunchKernelEx(&cfg, kern, M, ld, strideM, np, off, piv, npiv, tol, zorig,
                                        failed, status, first_error, moves, moves_n);
    if (er == cudaSuccess) {
      if (panel_done) cudaEventRecord(panel_done, stream);
      row_move_kernel<<<dim3((np + MC - 1) / MC, nsys), 256, 0, stream>>>(M, ld, strideM, np, off, w, moves,
                                                                          moves_n, failed);
      return cudaGetLastError();
    }
    cudaGetLastError();
  }
  // smallest cluster whose CTAs hold <= 384 rows each (<= 210 KB of shared memory), up to 16 CTAs
  int C = 1;
  while (C < 16 && (rows + C - 1) / C > MAX_ROWS_PER_CTA) C *= 2;
  const int R = (rows + C - 1) / C;
  static const bool no_cluster = std::getenv("PF_PANEL_GLOBAL") != nullptr;
  cudaError_t e = cudaSuccess;
  if (R <= MAX_ROWS_PER_CTA && !no_cluster) {
    static bool attrs = false;
    if (!attrs) {
      cudaFuncSetAttribute(panel_lu_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      attrs = true;
    }
    e = set_smem_attr_once(reinterpret_cast<const void*>(panel_lu_cluster_kernel),
                           (int)panel_lu_smem_bytes(MAX_ROWS_PER_CTA));
    if (e == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C, nsys);
      cfg.blockDim = dim3(PT);
      cfg.dynamicSmemBytes = panel_lu_smem_bytes(R);
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e = cudaLaunchKernelEx(&cfg, panel_lu_cluster_kernel, M, ld, strideM, np, off, w, R, piv, npiv, tol, zorig,
                             failed, status, first_error, moves, moves_n);
    }
    if (e != cudaSuccess) cudaGetLastError();  // no cluster launch: the global-memory panel below
  }
  if (no_cluster || R > MAX_ROWS_PER_CTA || e != cudaSuccess)
    panel_lu_global_kernel<<<nsys, 1024, 0, stream>>>(M, ld, strideM, np, off, w, piv, npiv, tol, zorig, failed,
                                                      status, first_error, moves, moves_n);
  if (panel_done) cudaEventRecord(panel_done, stream);
  row_move_kernel<<<dim3((np + MC - 1) / MC, nsys), 256, 0, stream>>>(M, ld, strideM, np, off, w, moves, moves_n,
                                                                      failed);
  return cudaGetLastError();
}

}  // namespace pf
