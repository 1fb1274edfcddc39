// Host orchestration of the large-n path (n > 128, and the DenseLu / action entry points):
// recursive LU and triangular solves over batches of identity-padded systems, every off-diagonal
// update on the DMMA GEMM (gemm.cu), 64 x 64 diagonal blocks on large.cu's base kernels.
//
//   LU(A)        = LU(A11); A12 <- L11^-1 A12; A21 <- A21 U11^-1; A22 -= A21 A12; LU(A22)
//   L^-1 B       = [L11^-1 B1; L22^-1 (B2 - L21 B1)]
//   U^-1 B       = [U11^-1 (B1 - U12 B2); U22^-1 B2]
//   B U^-1       = [B1 U11^-1, (B2 - B1 U12) U22^-1]
// The same arithmetic as dense.cpp's right-looking LU / substitution (dense.cpp:102-163), blocked.
#include <algorithm>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pf_host.h"

namespace pf {

__global__ void lu_base64_kernel(double* M, int64_t ld, int64_t strideM, int off, double* inv, int64_t inv_stride, int factor,
                                 const int* zlist);
__global__ void apply_inv64_kernel(const double* inv, int64_t inv_stride, int blk, int upper, int right, double* Bm,
                                   int64_t ld, int64_t strideB, int extent);
__global__ void lu_pivot_kernel(double* M, int64_t ld, int64_t strideM, int n, int* piv, const double* tol,
                                DevStatus* status, int* first_error, const int* zlist);
__global__ void form_shifted_kernel(const double* A, int64_t lda, int64_t strideA, int n, int np, int batch,
                                    const double* shifts, const int* j, double* M, unsigned long long* mx);
__global__ void certificate_partial_kernel(const double* M, int np, int n, int chunk, double* part);
__global__ void colstat_partial_kernel(const double* B, int64_t ld, int64_t strideB, int n, int chunk, double* part,
                                       unsigned long long* bmax);
__global__ void pair_certificate_kernel(const double* B, int64_t ld, int64_t strideB, int n, int nchunks,
                                        const double* part, const unsigned long long* bmax, const double* c, int npairs,
                                        double rel, int* ok);
__global__ void certificate_kernel(const double* M, int np, int n, int nchunks, const double* part,
                                   const unsigned long long* mx, double rel_tol, int* ok);
__global__ void form_rhs_kernel(const double* src, int64_t lds, int64_t strideS, int n, int np, int cols,
                                int ncols_true, int batch, const double* shifts, const int* j, int residual,
                                const int* perm, double* R, int64_t strideR);
__global__ void accumulate_sets_kernel(const double* X, int64_t xld, int64_t strideX, int n, int cols, int batch,
                                       int n_terms, const int* term_z, AccSets sets, const double* Bsrc, int64_t bld,
                                       int64_t strideBs, const int* j, const double* B2, int64_t b2ld,
                                       int64_t strideB2);
__global__ void accumulate_kernel(const double* X, int64_t xld, int64_t strideX, int n, int cols, int batch,
                                  int n_terms, const int* term_z, const double* w, int add_poly, double constant,
                                  double d1, double d2, const double* Bsrc, int64_t bld, int64_t strideBs,
                                  const int* j, const double* B2, int64_t b2ld, int64_t strideB2, double* out,
                                  int64_t ldo, int64_t strideOut);
__global__ void action_accumulate_kernel(const double* R, int64_t rld, int64_t strideR, const double* X, int64_t xld,
                                         int n, int k, int n_terms, const int* term_z, const double* w, int add_poly,
                                         double constant, int hybrid, double d1, double d2, const double* BX,
                                         const double* B2X, double* out, int64_t ldo);
__global__ void perm_from_piv_kernel(const int* piv, int n, int* perm, const int* zlist);
__global__ void copy2d_kernel(int rows, int cols, double s, const double* X, int64_t ldx, int64_t strideX, double* Y,
                              int64_t ldy, int64_t strideY);
__global__ void scale_pad_kernel(const double* A, int64_t lda, int n, int np, double s, double* B);
__global__ void fill_int_kernel(int* p, int count, int v);
__global__ void load_padded_kernel(const double* A, int64_t lda, int64_t strideA, int n, int np, double* M,
                                   unsigned long long* mx);
__global__ void iota_kernel(int* p, int n);
__global__ void lincomb2_kernel(int n, int k, double d1, const double* X, double d2, const double* Y, int64_t ld,
                                double* out, int64_t ldo);
size_t apply_inv64_smem_bytes();
size_t lu_base64_smem_bytes();
__global__ void lu_base128_kernel(double* M, int64_t ld, int64_t strideM, int off, double* inv, int64_t inv_stride);
__global__ void lu_dag_kernel(double* M, int np, int64_t strideM, double* inv, int64_t inv_stride, const int4* tasks,
                              int ntasks, int* next, int* state, int nt, int* err, const __grid_constant__ DagMaps maps,
                              int use_tma);
size_t lu_dag_smem_bytes();
void set_dag_trace(long long* p);
size_t lu_base128_smem_bytes();
__global__ void trsm128_kernel(const double* M, int64_t ld, int64_t strideM, int off, const double* inv,
                               int64_t inv_stride, int mode, double* Bm, int64_t ldb, int64_t strideB, int extent);
size_t trsm128_smem_bytes();

namespace host {
namespace {

constexpr int kB = 64;

int round64(int n) { return ((n + kB - 1) / kB) * kB; }
unsigned grid_for(int64_t elems) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((elems + 255) / 256, 1184)); }
// blocks per matrix for an elementwise kernel over `count` matrices (grid.y): about 2 x 1184 CTAs in
// total (one block per matrix for big batches: cfg5 forms 1024 systems, and 1024 blocks per system
// issued 8M atomics on 1024 addresses -- 5.6 ms for a 2.5 GB pass)
unsigned grid2(int64_t elems, int count) {
  const int64_t per = std::max<int64_t>(1, (2368 + count - 1) / std::max(count, 1));
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((elems + 255) / 256, std::min<int64_t>(per, 1184)));
}

// A batch of nsys systems of order np (row-major, stride np^2) plus their diagonal-block inverses.
struct Sys {
  double* M;
  int np;
  int nsys;
  double* inv;
  int64_t inv_stride;
  int64_t stride() const { return (int64_t)np * np; }
};

void apply_inv(pf_context* ctx, const Sys& s, int blk, bool upper, bool right, double* B, int64_t ldb, int64_t sb,
               int extent) {
  set_smem_attr_once(reinterpret_cast<const void*>(apply_inv64_kernel), (int)apply_inv64_smem_bytes());
  dim3 grid((extent + kB - 1) / kB, s.nsys);
  apply_inv64_kernel<<<grid, 256, apply_inv64_smem_bytes(), ctx->stream>>>(s.inv, s.inv_stride, blk, upper ? 1 : 0, right ? 1 : 0, B, ldb, sb,
                                                    extent);
  ctx->launches++;
}

// 64 x 64 diagonal block: LU in place (factor) and the explicit inverses of its L and U
void lu_base(pf_context* ctx, const Sys& s, int nblocks, int off, int factor, const int* zlist) {
  set_smem_attr_once(reinterpret_cast<const void*>(lu_base64_kernel), (int)lu_base64_smem_bytes());
  lu_base64_kernel<<<nblocks, 256, lu_base64_smem_bytes(), ctx->stream>>>(s.M, s.np, s.stride(), off, s.inv,
                                                                          s.inv_stride, factor, zlist);
  ctx->launches++;
}

int half64(int n) { return std::max(kB, ((n / kB) / 2) * kB); }

// the three solve levels of a 128 diagonal block in one launch (large.cu trsm128_kernel); mode 0
// L^-1 B, 1 U^-1 B, 2 B U^-1. PF_NO_LEAF128 keeps the 64-block recursion.
bool trsm128(pf_context* ctx, const Sys& s, int off, int mode, double* B, int64_t ldb, int64_t sb, int extent) {
  static const bool leaf128 = std::getenv("PF_NO_LEAF128") == nullptr;
  if (!leaf128) return false;
  dim3 grid((extent + kB - 1) / kB, s.nsys);
  // only where the three separate launches are latency-bound: the fused kernel runs one CTA per SM
  // (174 KB smem), the separate ones overlap better on big grids (cfg5's 256 systems: +3 ms fused)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  static const bool force = std::getenv("PF_TRSM128_FORCE") != nullptr;  // A/B on big grids
  if (!force && (int64_t)grid.x * grid.y > 2 * (int64_t)sms) return false;
  set_smem_attr_once(reinterpret_cast<const void*>(trsm128_kernel), (int)trsm128_smem_bytes());
  trsm128_kernel<<<grid, 256, trsm128_smem_bytes(), ctx->stream>>>(s.M, s.np, s.stride(), off, s.inv, s.inv_stride,
                                                                   mode, B, ldb, sb, extent);
  ctx->launches++;
  return true;
}

// B (n x cols) <- L^-1 B, L = unit-lower diagonal block [off, off + n) of s.M
void trsm_left_lower(pf_context* ctx, const Sys& s, int off, int n, double* B, int64_t ldb, int64_t sb, int cols) {
  if (n == 2 * kB && trsm128(ctx, s, off, 0, B, ldb, sb, cols)) return;
  if (n == kB) {
    apply_inv(ctx, s, off / kB, false, false, B, ldb, sb, cols);
    return;
  }
  const int n1 = half64(n), n2 = n - n1;
  trsm_left_lower(ctx, s, off, n1, B, ldb, sb, cols);
  const double* L21 = s.M + (int64_t)(off + n1) * s.np + off;
  gemm(ctx, n2, cols, n1, s.nsys, -1.0, L21, s.np, s.stride(), B, ldb, sb, 1.0, B + (int64_t)n1 * ldb, ldb, sb, 0.0);
  trsm_left_lower(ctx, s, off + n1, n2, B + (int64_t)n1 * ldb, ldb, sb, cols);
}

// B (n x cols) <- U^-1 B
void trsm_left_upper(pf_context* ctx, const Sys& s, int off, int n, double* B, int64_t ldb, int64_t sb, int cols) {
  if (n == 2 * kB && trsm128(ctx, s, off, 1, B, ldb, sb, cols)) return;
  if (n == kB) {
    apply_inv(ctx, s, off / kB, true, false, B, ldb, sb, cols);
    return;
  }
  const int n1 = half64(n), n2 = n - n1;
  trsm_left_upper(ctx, s, off + n1, n2, B + (int64_t)n1 * ldb, ldb, sb, cols);
  const double* U12 = s.M + (int64_t)off * s.np + off + n1;
  gemm(ctx, n1, cols, n2, s.nsys, -1.0, U12, s.np, s.stride(), B + (int64_t)n1 * ldb, ldb, sb, 1.0, B, ldb, sb, 0.0);
  trsm_left_upper(ctx, s, off, n1, B, ldb, sb, cols);
}

// B (rows x n) <- B U^-1
void trsm_right_upper(pf_context* ctx, const Sys& s, int off, int n, double* B, int64_t ldb, int64_t sb, int rows) {
  if (n == 2 * kB && trsm128(ctx, s, off, 2, B, ldb, sb, rows)) return;
  if (n == kB) {
    apply_inv(ctx, s, off / kB, true, true, B, ldb, sb, rows);
    return;
  }
  const int n1 = half64(n), n2 = n - n1;
  trsm_right_upper(ctx, s, off, n1, B, ldb, sb, rows);
  const double* U12 = s.M + (int64_t)off * s.np + off + n1;
  gemm(ctx, rows, n2, n1, s.nsys, -1.0, B, ldb, sb, U12, s.np, s.stride(), 1.0, B + n1, ldb, sb, 0.0);
  trsm_right_upper(ctx, s, off + n1, n2, B + n1, ldb, sb, rows);
}

// Runs `branch` on the context's side stream, concurrently with what the caller enqueues next on
// the main stream until join(): fork / join through two reused events (forks never nest: the
// branch itself enqueues on one stream only).
bool fork_side(pf_context* ctx) {
  if (!ctx->side) {
    if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      ctx->side = nullptr;
      return false;
    }
  }
  cudaEventRecord(ctx->ev_fork, ctx->stream);
  cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
  return true;
}

// stream and events of look-ahead depth d (created on first use); false if unavailable
bool aux_for(pf_context* ctx, int d) {
  while ((int)ctx->aux.size() <= d) {
    cudaStream_t st = nullptr;
    cudaEvent_t r = nullptr, e = nullptr;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&r, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      if (st) cudaStreamDestroy(st);
      if (r) cudaEventDestroy(r);
      return false;
    }
    ctx->aux.push_back(st);
    ctx->aux_ready.push_back(r);
    ctx->aux_done.push_back(e);
  }
  return true;
}

// LU of the diagonal block [off, off + n). `pending`: an event that must complete before this
// call touches its own trailing block A22 = [off + n1, off + n)^2 (the caller's look-ahead GEMM
// still updating it); everything before the trailing update (LU(A11), the panel solves) only
// touches A11 / A12 / A21 and runs concurrently with it.
//
// Look-ahead: of the trailing update A22 -= A21 A12, the rows [0, h) of A22 (all columns) and the
// block [h, n2) x [0, h) are updated on the main stream -- exactly what LU(A22)'s own A11 / A12 /
// A21 need -- and the bottom-right quadrant [h, n2)^2, the largest piece, on the depth's aux
// stream, where it overlaps the latency-bound recursion of LU(A22)'s first half. The child waits
// for it right before its own trailing update.
void lu_rec(pf_context* ctx, const Sys& s, int off, int n, cudaEvent_t pending = nullptr, int depth = 0) {
  if (n == kB) {
    lu_base(ctx, s, s.nsys, off, 1, nullptr);
    return;
  }
  // a 128 block in one launch (LU of both halves, the panels and the update between them) instead
  // of five dependent ones; PF_NO_LEAF128 keeps the 64 leaves
  static const bool leaf128 = std::getenv("PF_NO_LEAF128") == nullptr;
  if (n == 2 * kB && leaf128 && pending == nullptr) {
    set_smem_attr_once(reinterpret_cast<const void*>(lu_base128_kernel), (int)lu_base128_smem_bytes());
    lu_base128_kernel<<<s.nsys, 256, lu_base128_smem_bytes(), ctx->stream>>>(s.M, s.np, s.stride(), off, s.inv,
                                                                             s.inv_stride);
    ctx->launches++;
    return;
  }
  const int n1 = half64(n), n2 = n - n1;
  lu_rec(ctx, s, off, n1, nullptr, depth + 1);
  double* A12 = s.M + (int64_t)off * s.np + off + n1;
  double* A21 = s.M + (int64_t)(off + n1) * s.np + off;
  double* A22 = s.M + (int64_t)(off + n1) * s.np + off + n1;
  // the two panel solves are independent: A21 U11^-1 on the side stream, L11^-1 A12 on the main
  // one (their chains of small launches overlap deep in the recursion)
  if (fork_side(ctx)) {
    cudaStream_t main = ctx->stream;
    ctx->stream = ctx->side;
    trsm_right_upper(ctx, s, off, n1, A21, s.np, s.stride(), n2);
    cudaEventRecord(ctx->ev_join, ctx->side);
    ctx->stream = main;
    trsm_left_lower(ctx, s, off, n1, A12, s.np, s.stride(), n2);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
  } else {
    trsm_left_lower(ctx, s, off, n1, A12, s.np, s.stride(), n2);
    trsm_right_upper(ctx, s, off, n1, A21, s.np, s.stride(), n2);
  }
  if (pending) cudaStreamWaitEvent(ctx->stream, pending, 0);
  // opt-in (PF_LOOKAHEAD=1): measured 1-10 % slower at n = 1024-8192 (tools/lu_timing.py) -- the
  // quadrant GEMM's 212 KB-smem CTAs hold every SM for hundreds of microseconds, so the
  // recursion's small launches queue behind them instead of overlapping (needs an SM-capped GEMM)
  static const bool lookahead = std::getenv("PF_LOOKAHEAD") != nullptr;
  if (lookahead && n2 >= 2 * kB && aux_for(ctx, depth)) {
    const int h = half64(n2);  // = the child's own split
    const int64_t ld = s.np, st = s.stride();
    cudaStream_t main = ctx->stream, ax = ctx->aux[(size_t)depth];
    cudaEventRecord(ctx->aux_ready[(size_t)depth], main);
    cudaStreamWaitEvent(ax, ctx->aux_ready[(size_t)depth], 0);
    ctx->stream = ax;
    // capped: the quadrant leaves SMs to the recursion it overlaps (PF_LOOKAHEAD_RESERVE SMs, 24)
    static const int reserve = std::getenv("PF_LOOKAHEAD_RESERVE") ? std::atoi(std::getenv("PF_LOOKAHEAD_RESERVE")) : 24;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    ctx->gemm_cap = std::max(1, sms - reserve);
    gemm(ctx, n2 - h, n2 - h, n1, s.nsys, -1.0, A21 + (int64_t)h * ld, ld, st, A12 + h, ld, st, 1.0,
         A22 + (int64_t)h * ld + h, ld, st, 0.0);
    ctx->gemm_cap = 0;
    cudaEventRecord(ctx->aux_done[(size_t)depth], ax);
    ctx->stream = main;
    gemm(ctx, h, n2, n1, s.nsys, -1.0, A21, ld, st, A12, ld, st, 1.0, A22, ld, st, 0.0);
    gemm(ctx, n2 - h, h, n1, s.nsys, -1.0, A21 + (int64_t)h * ld, ld, st, A12, ld, st, 1.0, A22 + (int64_t)h * ld, ld,
         st, 0.0);
    lu_rec(ctx, s, off + n1, n2, ctx->aux_done[(size_t)depth], depth + 1);
    return;
  }
  gemm(ctx, n2, n2, n1, s.nsys, -1.0, A21, s.np, s.stride(), A12, s.np, s.stride(), 1.0, A22, s.np, s.stride(), 0.0);
  lu_rec(ctx, s, off + n1, n2, nullptr, depth + 1);
}

// lu_rec(0, np) through a CUDA graph: the recursion is a fixed chain of several hundred small
// launches on the same buffers, so it is captured once (on the second call with a given
// (M, inv, np, nsys); the first runs directly) and replayed, which removes the per-launch gaps.
// Capture and replay run on the context's private stream, fenced to the caller's stream by two
// events (the caller's may be the legacy default stream, which cannot be captured).
// Opt-in (PF_LU_GRAPH=1; not with the opt-in look-ahead, whose aux streams are not captured).
bool graph_stream(pf_context* ctx) {
  if (ctx->gstream) return true;
  if (cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_g0, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_g1, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    ctx->gstream = nullptr;
    return false;
  }
  return true;
}

void run_lu_graph(pf_context* ctx, const Sys& s) {  // on ctx->stream == ctx->gstream
  pf_context::LuGraph* hit = nullptr;
  for (auto& g : ctx->lu_graphs)
    if (g.M == s.M && g.inv == s.inv && g.inv_stride == s.inv_stride && g.np == s.np && g.nsys == s.nsys) hit = &g;
  if (hit && hit->exec) {
    if (cudaGraphLaunch(hit->exec, ctx->stream) == cudaSuccess) {
      ctx->launches += hit->launches;
      return;
    }
    cudaGetLastError();
    cudaGraphExecDestroy(hit->exec);  // stale: drop it and run directly from now on
    hit->exec = nullptr;
    hit->M = nullptr;
    lu_rec(ctx, s, 0, s.np);
    return;
  }
  if (!hit) {  // first sighting: run directly, capture next time
    if (ctx->lu_graphs.size() >= 8) {
      if (ctx->lu_graphs.front().exec) cudaGraphExecDestroy(ctx->lu_graphs.front().exec);
      ctx->lu_graphs.erase(ctx->lu_graphs.begin());
    }
    pf_context::LuGraph g;
    g.M = s.M;
    g.inv = s.inv;
    g.inv_stride = s.inv_stride;
    g.np = s.np;
    g.nsys = s.nsys;
    ctx->lu_graphs.push_back(g);
    lu_rec(ctx, s, 0, s.np);
    return;
  }
  const int64_t l0 = ctx->launches;
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    lu_rec(ctx, s, 0, s.np);
    return;
  }
  lu_rec(ctx, s, 0, s.np);
  const cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  cudaGraphExec_t exec = nullptr;
  if (e != cudaSuccess || !graph || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    ctx->launches = l0;
    lu_rec(ctx, s, 0, s.np);  // the captured launches never ran
    return;
  }
  cudaGraphDestroy(graph);
  hit->exec = exec;
  hit->launches = ctx->launches - l0;
  if (cudaGraphLaunch(exec, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    ctx->launches = l0;
    lu_rec(ctx, s, 0, s.np);
  }
}

// The device-scheduled tile-DAG LU (large.cu lu_dag_kernel): one persistent launch for the whole
// factorisation of every system. Task list (type F 0 / R 1 / C 2 / G 3, system, tile, step) in a
// topological order with one step of look-ahead; built once per (tiles, systems) and cached.
const std::vector<int4>& dag_tasks(int nt, int nsys) {
  static std::map<std::pair<int, int>, std::vector<int4>> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(nt, nsys);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<int4> t;
  // x = part (bits 28-29) | type (24-27) | first step k0 of a G task (8-23) | system (0-7); w = step
  auto add = [&](int type, int i, int j, int k, int k0 = 0) {
    // R / C: one task per 64-wide chunk; type 4: the look-ahead G of the next diagonal tile in quarters
    const int parts = (type == 1 || type == 2 || type == 5) ? 2 : (type == 4 ? 4 : 1);
    for (int z = 0; z < nsys; ++z)
      for (int h = 0; h < parts; ++h) t.push_back(make_int4((h << 28) | (type << 24) | (k0 << 8) | z, i, j, k));
  };
  auto panel = [&](int k) {  // F(k) and its two inverse tasks, then R(k, j) / C(j, k), nearest first
    add(0, k, k, k);
    add(5, k, k, k);
    for (int j = k + 1; j < nt; ++j) {
      add(1, k, j, k);
      add(2, j, k, k);
    }
  };
  // tiles off the look-ahead row / column take their updates in batches of kBatch steps (one task,
  // K = 128 kBatch: C read and written once per batch instead of once per step); a tile's batch
  // closes early at step min(i, j) - 2, before its look-ahead step. PF_DAG_BATCH=1: per step.
  // (8 systems, profiles/r02_lu_timing.jsonl: n = 1024 best per step, 2048 with 4, 4096 with 8)
  static const int forced = std::getenv("PF_DAG_BATCH") ? std::max(1, std::atoi(std::getenv("PF_DAG_BATCH"))) : 0;
  const int kBatch = forced ? forced : (nt <= 8 ? 1 : (nt <= 16 ? 4 : 8));
  // PF_DAG_DEFER=d: d of step k's far trailing updates are listed between F(k + 1) and its R / C
  // tasks, so CTAs that would spin on F(k + 1) take trailing work meanwhile
  static const int defer = std::getenv("PF_DAG_DEFER") ? std::max(0, std::atoi(std::getenv("PF_DAG_DEFER"))) : 0;
  panel(0);
  for (int k = 0; k + 1 < nt; ++k) {
    const int n1 = k + 1;
    add(4, n1, n1, k);  // the tiles of row / column k + 1 first: F(k + 1)'s look-ahead (quartered)
    for (int j = n1 + 1; j < nt; ++j) {
      add(3, n1, j, k, k);
      add(3, j, n1, k, k);
    }
    // the rest of step k: first the row / column k + 2 (the next step's look-ahead reads them), then
    // the others
    std::vector<int2> near, far;
    auto rest = [&](std::vector<int2>& into, int i, int j) {
      const int m = std::min(i, j);
      if ((k + 1) % kBatch == 0 || k == m - 2) into.push_back(make_int2(i, j));
    };
    const int n2 = n1 + 1;
    if (n2 < nt) {
      rest(near, n2, n2);
      for (int j = n2 + 1; j < nt; ++j) {
        rest(near, n2, j);
        rest(near, j, n2);
      }
    }
    for (int i = n2 + 1; i < nt; ++i)
      for (int j = n2 + 1; j < nt; ++j) rest(far, i, j);
    const int d = std::min<int>(defer / std::max(nsys, 1), (int)far.size());  // tiles (x nsys tasks)
    const int kb = (k / kBatch) * kBatch;
    add(0, n1, n1, n1);  // F(k + 1) and its inverses
    add(5, n1, n1, n1);
    for (int q = 0; q < d; ++q) add(3, far[q].x, far[q].y, k, kb);
    for (int j = n1 + 1; j < nt; ++j) {  // R(k + 1, j) / C(j, k + 1)
      add(1, n1, j, n1);
      add(2, j, n1, n1);
    }
    for (const int2& q : near) add(3, q.x, q.y, k, kb);
    for (size_t q = d; q < far.size(); ++q) add(3, far[q].x, far[q].y, k, kb);
  }
  return cache.emplace(key, std::move(t)).first->second;
}

// 1: factored, 0: not applicable (use the recursion), -1: the DAG reported a scheduling failure
int run_lu_dag(pf_context* ctx, const Sys& s) {
  // PF_LU_DAG=0 keeps the recursion; =1 forces the DAG wherever it applies (np a multiple of 128)
  static const int mode = std::getenv("PF_LU_DAG") ? std::atoi(std::getenv("PF_LU_DAG")) : -1;
  if (mode == 0 || s.np % 128 != 0 || s.np < 256 || s.nsys > 255) return 0;  // (8-bit system field)
  // measured (profiles/r02_lu_timing.jsonl, 8 systems, both on TMA operand staging): DAG 0.75 / 3.43 /
  // 22.9 ms vs recursion 1.04 / 3.47 / 16.2 at n = 1024 / 2048 / 4096 -- from 4096 on the DAG's
  // k = 128 tile updates re-read and re-write C once per step (memory), the recursion's long-k GEMMs
  // do not
  if (mode < 0 && (s.np < 1024 || s.np > 2048 || s.nsys > 64)) return 0;
  const int nt = s.np / 128;
  const std::vector<int4>& tasks = dag_tasks(nt, s.nsys);
  int4* d_tasks = static_cast<int4*>(workspace(ctx, kWsSmallArrays + 28, sizeof(int4) * tasks.size()));
  int* d_state = static_cast<int*>(workspace(ctx, kWsSmallArrays + 29, sizeof(int) * ((size_t)s.nsys * nt * nt + 2)));
  if (!d_tasks || !d_state) return 0;
  int* d_next = d_state + (size_t)s.nsys * nt * nt;
  int* d_err = d_next + 1;
  cudaMemcpyAsync(d_tasks, tasks.data(), sizeof(int4) * tasks.size(), cudaMemcpyHostToDevice, ctx->stream);
  cudaMemsetAsync(d_state, 0, sizeof(int) * ((size_t)s.nsys * nt * nt + 2), ctx->stream);
  const int smem = (int)lu_dag_smem_bytes();
  if (set_smem_attr_once(reinterpret_cast<const void*>(lu_dag_kernel), smem) != cudaSuccess) return 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  // G tasks on TMA when the tensor maps can be built (PF_DAG_TMA=0: the cp.async tile)
  static const bool no_tma = std::getenv("PF_DAG_TMA") != nullptr && std::atoi(std::getenv("PF_DAG_TMA")) == 0;
  DagMaps maps{};
  const bool tma = !no_tma && (reinterpret_cast<uintptr_t>(s.M) & 15) == 0 &&
                   make_tma_map(&maps.a, s.M, (uint64_t)s.np, (uint64_t)s.np, (uint64_t)s.nsys, s.np, s.stride(), 16,
                                128) &&
                   make_tma_map(&maps.b, s.M, (uint64_t)s.np, (uint64_t)s.np, (uint64_t)s.nsys, s.np, s.stride(), 16, 16);
  static const bool trace_on = std::getenv("PF_DAG_TRACE") != nullptr;  // diagnostics: per-task timeline
  long long* d_trace = nullptr;
  if (trace_on) {
    d_trace = static_cast<long long*>(workspace(ctx, kWsSmallArrays + 30, sizeof(long long) * 3 * tasks.size()));
    if (d_trace) cudaMemsetAsync(d_trace, 0, sizeof(long long) * 3 * tasks.size(), ctx->stream);
    set_dag_trace(d_trace);
  }
  lu_dag_kernel<<<sms, 256, smem, ctx->stream>>>(s.M, s.np, s.stride(), s.inv, s.inv_stride, d_tasks,
                                                 (int)tasks.size(), d_next, d_state, nt, d_err, maps, tma ? 1 : 0);
  if (trace_on && d_trace) {
    std::vector<long long> h(3 * tasks.size());
    cudaMemcpyAsync(h.data(), d_trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    set_dag_trace(nullptr);
    long long t0 = h[0];
    for (size_t q = 0; q < tasks.size(); ++q) t0 = std::min(t0, h[3 * q]);
    for (size_t q = 0; q < tasks.size(); ++q) {
      const int4 tk = tasks[q];
      std::fprintf(stderr, "dagtrace %d %d %d %d %d %d %lld %lld %lld\n", (tk.x >> 24) & 15, (tk.x >> 28) & 3,
                   tk.x & 0xff, tk.y, tk.z, tk.w, h[3 * q] - t0, h[3 * q + 1] - t0, h[3 * q + 2] - t0);
    }
  }
  ctx->launches++;
  if (cudaGetLastError() != cudaSuccess) return -1;
  // the spin-limit flag (a scheduling bug must not pass as a factorisation)
  if (cudaMemcpyAsync(ctx->h_first_error, d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return -1;
  return *ctx->h_first_error == 0 ? 1 : -1;
}

// false only when the device-scheduled LU failed (the factors are then unusable)
bool run_lu(pf_context* ctx, const Sys& s) {
  const int dag = run_lu_dag(ctx, s);
  if (dag != 0) return dag > 0;
  // opt-in (PF_LU_GRAPH=1): instantiating the captured recursion costs ~6 ms (128 leaves) to
  // ~40 ms (64 leaves) once per buffer set, so it pays off only over many repeated factorisations
  // of the same shape and buffers (-3 % per call at n = 4096); one-shot calls lose (cfg3 +5 ms)
  static const bool graphs = std::getenv("PF_LU_GRAPH") != nullptr && std::getenv("PF_LOOKAHEAD") == nullptr;
  if (!graphs || !graph_stream(ctx) || !fork_side(ctx)) {  // fork_side: the side stream exists
    lu_rec(ctx, s, 0, s.np);
    return true;
  }
  cudaStream_t main = ctx->stream;
  cudaEventRecord(ctx->ev_g0, main);
  cudaStreamWaitEvent(ctx->gstream, ctx->ev_g0, 0);
  ctx->stream = ctx->gstream;
  run_lu_graph(ctx, s);
  ctx->stream = main;
  cudaEventRecord(ctx->ev_g1, ctx->gstream);
  cudaStreamWaitEvent(main, ctx->ev_g1, 0);
  return true;
}

void diag_inverses(pf_context* ctx, const Sys& s) {
  for (int off = 0; off < s.np; off += kB) {
    lu_base(ctx, s, s.nsys, off, 0, nullptr);
  }
}

template <typename T>
T* upload(pf_context* ctx, int slot, const std::vector<T>& v) {
  T* d = static_cast<T*>(workspace(ctx, slot, sizeof(T) * std::max<size_t>(v.size(), 1)));
  if (d && !v.empty()) cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, ctx->stream);
  return d;
}

// Factor the nsys systems already formed in s.M (true order n, padded np). Certified systems
// (strict column diagonal dominance with margin) take the recursive no-exchange LU; otherwise every
// system runs the genuine partial-pivoting kernel. On return perm (nsys x n) is the row order of
// the RHS (nullptr when no system was pivoted). Failures are reported for system z.
struct FactorResult {
  int rc = PF_OK;
  int z = -1;
  pf::DevStatus st{};
  bool pivoted = false;
  std::vector<double> scale;
};

constexpr int kDeclined = -1000;  // pair mode declined: the caller takes the per-shift path

// ---- blocked partial pivoting (DenseLu, dense.cpp:102-133) for the systems the certificate rejects
// Recursive column split (rows always to the bottom): LU(left half) with pivoting over all rows below,
// U12 = L11^-1 A12 (DMMA TRSM with 64-block inverses), A22 -= A21 U12 (DMMA GEMM), LU(right half).
// Each 64-wide leaf is factored by pivot_lu.cu's cluster kernel (pivot search and rank-1 updates in
// distributed shared memory) and its row exchanges are applied to the whole rows right after, so the
// matrix always has the reference's row order. Pivots follow the reference's rule on the blocked
// values: equal to dense.cpp's wherever pivots are well separated (the blocked updates round differently).
struct PivotScratch {
  int* piv;
  const double* tol;
  const int* zorig;
  int* failed;
  int2* moves;
  int* moves_n;
};

void rlu_pivot(pf_context* ctx, const Sys& sp, int off, int w, const PivotScratch& ps) {
  if (w <= kB) {
    // the leaf's L and U block inverses (for the TRSMs) only need the panel: on the side stream,
    // concurrently with the panel's row moves over the other columns
    const bool side = fork_side(ctx);
    pf::launch_panel_lu(sp.M, sp.np, sp.stride(), sp.np, off, w, sp.nsys, ps.piv, sp.np, ps.tol, ps.zorig, ps.failed,
                        ctx->status, ctx->first_error, ps.moves, ps.moves_n, ctx->stream,
                        side ? ctx->ev_fork : nullptr);
    ctx->launches += 2;
    if (side) {
      cudaStream_t main = ctx->stream;
      cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
      ctx->stream = ctx->side;
      lu_base(ctx, sp, sp.nsys, off, 0, nullptr);
      cudaEventRecord(ctx->ev_join, ctx->side);
      ctx->stream = main;
      cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
    } else {
      lu_base(ctx, sp, sp.nsys, off, 0, nullptr);
    }
    return;
  }
  const int w1 = half64(w), w2 = w - w1;
  const int64_t ld = sp.np, st = sp.stride();
  rlu_pivot(ctx, sp, off, w1, ps);
  double* A12 = sp.M + (int64_t)off * ld + off + w1;
  double* A21 = sp.M + (int64_t)(off + w1) * ld + off;
  double* A22 = sp.M + (int64_t)(off + w1) * ld + off + w1;
  trsm_left_lower(ctx, sp, off, w1, A12, ld, st, w2);
  gemm(ctx, sp.np - off - w1, w2, w1, sp.nsys, -1.0, A21, ld, st, A12, ld, st, 1.0, A22, ld, st, 0.0);
  rlu_pivot(ctx, sp, off + w1, w2, ps);
}

// the nf = fails.size() failing systems: gathered into `side` when they are a subset (the caller
// already parked their matrices there), factored, scattered back with their swap sequences
int pivoted_blocked_lu(pf_context* ctx, const Sys& s, int n, const std::vector<int>& fails, double* side,
                       const std::vector<double>& tol_all, const int* d_fail, int* d_piv) {
  const int nf = (int)fails.size();
  Sys sp = s;
  sp.nsys = nf;
  if (side) sp.M = side;
  double* inv_g = side ? static_cast<double*>(workspace(ctx, kWsLargeX2 + 2, sizeof(double) * s.inv_stride * nf))
                       : s.inv;
  int* piv_g = static_cast<int*>(workspace(ctx, kWsSmallArrays + 24, sizeof(int) * ((size_t)s.np + 1) * nf));
  int2* moves = static_cast<int2*>(workspace(ctx, kWsSmallArrays + 26, sizeof(int2) * 2 * kB * (size_t)nf));
  if (!inv_g || !piv_g || !moves) return PF_ERR_CUDA;
  sp.inv = inv_g;
  int* failed = piv_g + (size_t)s.np * nf;
  int* moves_n = static_cast<int*>(workspace(ctx, kWsSmallArrays + 27, sizeof(int) * (size_t)nf));
  if (!moves_n) return PF_ERR_CUDA;
  cudaMemsetAsync(failed, 0, sizeof(int) * nf, ctx->stream);
  std::vector<double> tol(nf);
  for (int q = 0; q < nf; ++q) tol[q] = tol_all[fails[q]];
  double* d_tol = upload(ctx, kWsSmallArrays + 25, tol);
  rlu_pivot(ctx, sp, 0, s.np, PivotScratch{piv_g, d_tol, d_fail, failed, moves, moves_n});
  for (int q = 0; q < nf; ++q) {
    if (side) {  // the factors and the leaves' block inverses back to their systems' slots
      cudaMemcpyAsync(s.M + fails[q] * s.stride(), side + q * s.stride(), sizeof(double) * s.stride(),
                      cudaMemcpyDeviceToDevice, ctx->stream);
      cudaMemcpyAsync(s.inv + fails[q] * s.inv_stride, inv_g + q * s.inv_stride, sizeof(double) * s.inv_stride,
                      cudaMemcpyDeviceToDevice, ctx->stream);
    }
    cudaMemcpyAsync(d_piv + (size_t)fails[q] * n, piv_g + (size_t)q * s.np, sizeof(int) * n, cudaMemcpyDeviceToDevice,
                    ctx->stream);
  }
  return cuda_fail(cudaGetLastError());
}

FactorResult factor_systems(pf_context* ctx, const Sys& s, int n, unsigned long long* d_mx, int flags,
                            int* d_piv, int* d_perm, double pivot_rel_tol, bool decline = false) {
  FactorResult fr;
  int* d_ok = static_cast<int*>(workspace(ctx, kWsSmallArrays + 20, sizeof(int) * s.nsys));
  fill_int_kernel<<<(s.nsys + 255) / 256, 256, 0, ctx->stream>>>(d_ok, s.nsys, 1);
  const int nchunks = std::max(1, std::min(64, n / 64));
  const int chunk = (n + nchunks - 1) / nchunks;
  double* d_part = static_cast<double*>(workspace(ctx, kWsSmallArrays + 23, sizeof(double) * (size_t)s.nsys * nchunks * n));
  if (!d_part) {
    fr.rc = PF_ERR_CUDA;
    return fr;
  }
  certificate_partial_kernel<<<dim3((n + 255) / 256, nchunks, s.nsys), 256, 0, ctx->stream>>>(s.M, s.np, n, chunk,
                                                                                             d_part);
  certificate_kernel<<<dim3((n + 255) / 256, s.nsys), 256, 0, ctx->stream>>>(s.M, s.np, n, nchunks, d_part, d_mx,
                                                                             pivot_rel_tol, d_ok);
  ctx->launches += 3;
  if (cudaGetLastError() != cudaSuccess) {  // a certificate that never ran must not read as "certified"
    fr.rc = PF_ERR_CUDA;
    return fr;
  }
  std::vector<int> ok(s.nsys);
  std::vector<unsigned long long> mxbits(s.nsys);
  cudaMemcpyAsync(ok.data(), d_ok, sizeof(int) * s.nsys, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(mxbits.data(), d_mx, sizeof(unsigned long long) * s.nsys, cudaMemcpyDeviceToHost, ctx->stream);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    fr.rc = PF_ERR_CUDA;
    return fr;
  }
  fr.scale.resize(s.nsys);
  const bool force = (flags & PF_FLAG_FORCE_PIVOT) != 0;
  std::vector<int> fails;  // the pivot decision is per system: results never depend on the batch
  for (int z = 0; z < s.nsys; ++z) {
    double mx;
    std::memcpy(&mx, &mxbits[z], sizeof(double));
    fr.scale[z] = std::max(mx, 1e-300);
    if (force || !ok[z]) fails.push_back(z);
  }
  const int nf = (int)fails.size();
  if (decline && nf > 0) {  // pair mode only runs the exchange-free LU
    fr.rc = kDeclined;
    return fr;
  }
  if (nf == 0) {
    if (!run_lu(ctx, s)) fr.rc = PF_ERR_CUDA;
    return fr;
  }
  fr.pivoted = true;
  // keep the failing systems' M aside, run the blocked LU on the batch, restore them, pivot them
  double* side = nullptr;
  if (nf < s.nsys) {
    side = static_cast<double*>(workspace(ctx, kWsLargeX2 + 1, sizeof(double) * s.stride() * nf));
    if (!side) {
      fr.rc = PF_ERR_CUDA;
      return fr;
    }
    for (int q = 0; q < nf; ++q)
      cudaMemcpyAsync(side + q * s.stride(), s.M + fails[q] * s.stride(), sizeof(double) * s.stride(),
                      cudaMemcpyDeviceToDevice, ctx->stream);
    if (!run_lu(ctx, s)) {
      fr.rc = PF_ERR_CUDA;
      return fr;
    }
    for (int q = 0; q < nf; ++q)
      cudaMemcpyAsync(s.M + fails[q] * s.stride(), side + q * s.stride(), sizeof(double) * s.stride(),
                      cudaMemcpyDeviceToDevice, ctx->stream);
  }
  std::vector<double> tol(s.nsys);
  for (int z = 0; z < s.nsys; ++z) tol[z] = pivot_rel_tol * fr.scale[z];
  double* d_tol = upload(ctx, kWsSmallArrays + 21, tol);
  int* d_fail = upload(ctx, kWsSmallArrays + 22, fails);
  // certified systems keep the identity row order and swap sequence
  iota_kernel<<<dim3((n + 255) / 256, s.nsys), 256, 0, ctx->stream>>>(d_perm, n);
  iota_kernel<<<dim3((n + 255) / 256, s.nsys), 256, 0, ctx->stream>>>(d_piv, n);
  ctx->launches += 2;
  int rc = ensure_status(ctx, s.nsys);
  if (rc) {
    fr.rc = rc;
    return fr;
  }
  static const bool unblocked = std::getenv("PF_PIVOT_UNBLOCKED") != nullptr;  // A/B: the old fallback
  if (unblocked) {
    lu_pivot_kernel<<<nf, 1024, 0, ctx->stream>>>(s.M, s.np, s.stride(), n, d_piv, d_tol, ctx->status,
                                                  ctx->first_error, d_fail);
    ctx->launches++;
  } else {
    rc = pivoted_blocked_lu(ctx, s, n, fails, side, tol, d_fail, d_piv);
    if (rc) {
      fr.rc = rc;
      return fr;
    }
  }
  pf_status ps;
  rc = collect_status(ctx, s.nsys, 0, &ps);
  if (rc) {
    fr.rc = rc;
    fr.z = ps.batch_index;
    fr.st.code = ps.code;
    fr.st.column = ps.column;
    fr.st.pivot_magnitude = ps.pivot_magnitude;
    return fr;
  }
  perm_from_piv_kernel<<<nf, 32, 0, ctx->stream>>>(d_piv, n, d_perm, d_fail);
  ctx->launches++;
  if (unblocked)  // the blocked LU formed every diagonal block's inverses after its panel
    for (int off = 0; off < s.np; off += kB) lu_base(ctx, s, nf, off, 0, d_fail);
  return fr;
}

// ---- explicit inverses of large diagonal blocks (thin right-hand sides: the action operator)
// A solve with k = 64 columns through the 64-leaf recursion is a chain of ~512 dependent small
// launches per triangle (cfg4: 1026 launches, 25 ms per substep). The operator is factored once and
// applied many times, so the inverses of its nbig x nbig diagonal blocks are formed once here
// (recursive block inversion on DMMA GEMMs from the 64 x 64 leaf inverses):
//   [L11 0; L21 L22]^-1 = [X11 0; -X22 L21 X11  X22],  [U11 U12; 0 U22]^-1 = [Y11 -Y11 U12 Y22; 0 Y22]
// and every apply is a left-looking blocked substitution with two GEMMs per block.
// dst (b x b, leading dimension ldd, batch stride sd) = inverse of the unit-lower / upper diagonal
// block [off, off + b) of every system; tmp holds (b/2)^2 per system.
void tri_inv(pf_context* ctx, const Sys& s, bool upper, int off, int b, double* dst, int64_t ldd, int64_t sd,
             double* tmp, int64_t st) {
  if (b == kB) {
    const double* src = s.inv + (int64_t)(off / kB) * 2 * kB * kB + (upper ? kB * kB : 0);
    copy2d_kernel<<<dim3(grid2((int64_t)kB * kB, s.nsys), s.nsys), 256, 0, ctx->stream>>>(kB, kB, 1.0, src, kB,
                                                                                      s.inv_stride, dst, ldd, sd);
    ctx->launches++;
    return;
  }
  const int b1 = half64(b), b2 = b - b1;
  double* X11 = dst;
  double* X22 = dst + (int64_t)b1 * ldd + b1;
  tri_inv(ctx, s, upper, off, b1, X11, ldd, sd, tmp, st);
  tri_inv(ctx, s, upper, off + b1, b2, X22, ldd, sd, tmp, st);
  if (!upper) {
    // T = L21 X11 (b2 x b1); X21 = -X22 T
    const double* L21 = s.M + (int64_t)(off + b1) * s.np + off;
    gemm(ctx, b2, b1, b1, s.nsys, 1.0, L21, s.np, s.stride(), X11, ldd, sd, 0.0, tmp, b1, st, 0.0);
    gemm(ctx, b2, b1, b2, s.nsys, -1.0, X22, ldd, sd, tmp, b1, st, 0.0, dst + (int64_t)b1 * ldd, ldd, sd, 0.0);
  } else {
    // T = U12 X22 (b1 x b2); X12 = -X11 T
    const double* U12 = s.M + (int64_t)off * s.np + off + b1;
    gemm(ctx, b1, b2, b2, s.nsys, 1.0, U12, s.np, s.stride(), X22, ldd, sd, 0.0, tmp, b2, st, 0.0);
    gemm(ctx, b1, b2, b1, s.nsys, -1.0, X11, ldd, sd, tmp, b2, st, 0.0, dst + b1, ldd, sd, 0.0);
  }
}

int big_block(int np) {
  if (np >= 4096) return 1024;
  if (np >= 2048) return 512;
  if (np >= 1024) return 256;
  return 0;  // small systems keep the 64-leaf recursion
}

int64_t big_inverse_stride(int np, int nb) { return (int64_t)((np + nb - 1) / nb) * 2 * nb * nb; }

// binv (per system big_inverse_stride doubles) <- block q: Linv at 2q nb^2, Uinv at (2q + 1) nb^2
bool build_big_inverses(pf_context* ctx, const Sys& s, int nb, double* binv) {
  const int nblk = (s.np + nb - 1) / nb;
  const int64_t bstride = big_inverse_stride(s.np, nb);
  double* tmp = static_cast<double*>(workspace(ctx, kWsTriTmp, sizeof(double) * (size_t)(nb / 2) * (nb / 2) * s.nsys));
  if (!tmp) return false;
  cudaMemsetAsync(binv, 0, sizeof(double) * bstride * s.nsys, ctx->stream);
  for (int q = 0; q < nblk; ++q) {
    const int off = q * nb, b = std::min(nb, s.np - off);
    for (int u = 0; u < 2; ++u)
      tri_inv(ctx, s, u == 1, off, b, binv + (int64_t)(2 * q + u) * nb * nb, b, bstride, tmp,
              (int64_t)(nb / 2) * (nb / 2));
  }
  return true;
}

// R (np x k per system, batch stride rs) <- U^-1 L^-1 R: left-looking blocked substitution with the
// explicit block inverses (forward into Y, backward back into R; two GEMMs per block) when binv is
// given, else the 64-leaf recursion.
int solve_lu(pf_context* ctx, const Sys& s, const double* binv, int nb, double* R, int k, int64_t rs) {
  if (!binv) {
    trsm_left_lower(ctx, s, 0, s.np, R, k, rs, k);
    trsm_left_upper(ctx, s, 0, s.np, R, k, rs, k);
    return PF_OK;
  }
  const int np = s.np, P = s.nsys, nblk = (np + nb - 1) / nb;
  const int64_t bstride = big_inverse_stride(np, nb), st = s.stride();
  double* Y = static_cast<double*>(workspace(ctx, kWsLargeX2, sizeof(double) * rs * P));
  if (!Y) return PF_ERR_CUDA;
  static const bool left_looking = std::getenv("PF_LEFT_LOOKING") != nullptr;
  if (!left_looking) {
    // right-looking: after each block, one GEMM updates every remaining row (np - end rows: many
    // CTAs, K = nb) instead of a K = q nb reduction over few CTAs per block
    for (int q = 0; q < nblk; ++q) {
      const int off = q * nb, b = std::min(nb, np - off), end = off + b;
      gemm(ctx, b, k, b, P, 1.0, binv + (int64_t)(2 * q) * nb * nb, b, bstride, R + (int64_t)off * k, k, rs, 0.0,
           Y + (int64_t)off * k, k, rs, 0.0);
      if (end < np)  // R[>q] -= L[>q, q] Y_q
        gemm(ctx, np - end, k, b, P, -1.0, s.M + (int64_t)end * np + off, np, st, Y + (int64_t)off * k, k, rs, 1.0,
             R + (int64_t)end * k, k, rs, 0.0);
    }
    for (int q = nblk - 1; q >= 0; --q) {
      const int off = q * nb, b = std::min(nb, np - off);
      gemm(ctx, b, k, b, P, 1.0, binv + (int64_t)(2 * q + 1) * nb * nb, b, bstride, Y + (int64_t)off * k, k, rs,
           0.0, R + (int64_t)off * k, k, rs, 0.0);
      if (off > 0)  // Y[<q] -= U[<q, q] X_q
        gemm(ctx, off, k, b, P, -1.0, s.M + off, np, st, R + (int64_t)off * k, k, rs, 1.0, Y, k, rs, 0.0);
    }
    return PF_OK;
  }
  for (int q = 0; q < nblk; ++q) {
    const int off = q * nb, b = std::min(nb, np - off);
    double* Rq = R + (int64_t)off * k;
    if (off > 0)  // R_q -= L[q, <q] Y[<q]
      gemm(ctx, b, k, off, P, -1.0, s.M + (int64_t)off * np, np, st, Y, k, rs, 1.0, Rq, k, rs, 0.0);
    gemm(ctx, b, k, b, P, 1.0, binv + (int64_t)(2 * q) * nb * nb, b, bstride, Rq, k, rs, 0.0, Y + (int64_t)off * k, k,
         rs, 0.0);
  }
  for (int q = nblk - 1; q >= 0; --q) {
    const int off = q * nb, b = std::min(nb, np - off), end = off + b;
    double* Yq = Y + (int64_t)off * k;
    if (end < np)  // Y_q -= U[q, >q] X[>q]
      gemm(ctx, b, k, np - end, P, -1.0, s.M + (int64_t)off * np + end, np, st, R + (int64_t)end * k, k, rs, 1.0,
           Yq, k, rs, 0.0);
    gemm(ctx, b, k, b, P, 1.0, binv + (int64_t)(2 * q + 1) * nb * nb, b, bstride, Yq, k, rs, 0.0,
         R + (int64_t)off * k, k, rs, 0.0);
  }
  return PF_OK;
}

bool make_sys(pf_context* ctx, Sys& s, int n, int nsys, int slotM) {
  s.np = round64(n);
  s.nsys = nsys;
  s.M = static_cast<double*>(workspace(ctx, slotM, sizeof(double) * s.stride() * std::max(nsys, 1)));
  s.inv_stride = (int64_t)(s.np / kB) * 2 * kB * kB;
  s.inv = static_cast<double*>(workspace(ctx, kWsLargeInv, sizeof(double) * s.inv_stride * std::max(nsys, 1)));
  return s.M && s.inv;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Pair mode (residual form, every nonzero shift in a pair c, -c; small_eval.cu does the same per
// matrix). With Z_p = (I - c_p^2 B^2)^-1 c_p^2 B^2 (the residual term of shift c_p^2 on B^2):
//   w+ X+ + w- X- = (w+ - w-) c (I + Z) B + (w+ + w-) Z,
// so for every weight set  f = a0 I + E_A B + E_B,  E_A = sum_p cm_p c_p (I + Z_p),  E_B = sum_p cp_p Z_p:
// half the LUs and solves of the per-shift path, plus B^2 and one product per weight set. Taken only
// when the reference's own systems I -/+ c B are certified for every pair (the reference would not
// pivot and raises nothing) and every I - c^2 B^2 passes the certificate; otherwise kDeclined.
// Pairs (c, -c) of a residual-form method without poly part: c of the first, indices of both;
// false when pair mode does not apply (or PF_NO_PAIRS / PF_FLAG_PER_SHIFT / PF_FLAG_FORCE_PIVOT).
bool plan_pairs(const pf_method* m, int flags, std::vector<double>& c, std::vector<int>& ip, std::vector<int>& im) {
  static const bool no_pairs = std::getenv("PF_NO_PAIRS") != nullptr;
  if (no_pairs || m->form != PF_FORM_RESIDUAL || m->has_poly || (flags & (PF_FLAG_FORCE_PIVOT | PF_FLAG_PER_SHIFT)))
    return false;
  std::vector<char> used(m->n_terms, 0);
  for (int i = 0; i < m->n_terms; ++i) {
    if (used[i] || m->shifts[i] == 0.0) continue;
    int jp = -1;
    for (int j = i + 1; j < m->n_terms; ++j)
      if (!used[j] && m->shifts[j] == -m->shifts[i]) {
        jp = j;
        break;
      }
    if (jp < 0) return false;
    used[i] = used[jp] = 1;
    c.push_back(m->shifts[i]);
    ip.push_back(i);
    im.push_back(jp);
  }
  return !c.empty();
}

// ok[b] = every I -/+ c_p B_b certified (B_b = B + b * strideB, n x n of leading dimension ld)
int pair_certificates(pf_context* ctx, const double* B, int64_t ld, int64_t strideB, int n, int batch,
                      const std::vector<double>& c, std::vector<int>& ok) {
  const int nchunks = std::max(1, std::min(64, n / 64));
  const int chunk = (n + nchunks - 1) / nchunks;
  double* d_part = static_cast<double*>(workspace(ctx, kWsSmallArrays + 24, sizeof(double) * (size_t)batch * nchunks * n));
  auto* d_bmax = static_cast<unsigned long long*>(workspace(ctx, kWsSmallArrays + 25, sizeof(unsigned long long) * batch));
  int* d_ok = static_cast<int*>(workspace(ctx, kWsSmallArrays + 26, sizeof(int) * batch));
  double* d_c = upload(ctx, kWsSmallArrays + 27, c);
  if (!d_part || !d_bmax || !d_ok || !d_c) return PF_ERR_CUDA;
  cudaMemsetAsync(d_bmax, 0, sizeof(unsigned long long) * batch, ctx->stream);
  fill_int_kernel<<<(batch + 255) / 256, 256, 0, ctx->stream>>>(d_ok, batch, 1);
  colstat_partial_kernel<<<dim3((n + 255) / 256, nchunks, batch), 256, 0, ctx->stream>>>(B, ld, strideB, n, chunk,
                                                                                        d_part, d_bmax);
  pair_certificate_kernel<<<dim3((n + 255) / 256, batch), 256, 0, ctx->stream>>>(
      B, ld, strideB, n, nchunks, d_part, d_bmax, d_c, (int)c.size(), 1e-14, d_ok);
  ctx->launches += 3;
  ok.assign(batch, 0);
  cudaMemcpyAsync(ok.data(), d_ok, sizeof(int) * batch, cudaMemcpyDeviceToHost, ctx->stream);
  return cudaStreamSynchronize(ctx->stream) == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

int large_eval_pairs(pf_context* ctx, const pf_method* m, int n, int batch, const double* A, int64_t lda,
                     int64_t strideA, const int* dJ, double* const* outs, int64_t ldo, int64_t strideOut, int flags,
                     pf_status* status) {
  std::vector<double> c;
  std::vector<int> ip, im;
  if (!plan_pairs(m, flags, c, ip, im)) return kDeclined;
  const int npairs = (int)c.size();
  const int64_t nn = (int64_t)n * n;
  double* Bs = static_cast<double*>(workspace(ctx, kWsPairB, sizeof(double) * nn * batch));
  double* B2 = static_cast<double*>(workspace(ctx, kWsPairB2, sizeof(double) * nn * batch));
  double* T = static_cast<double*>(workspace(ctx, kWsPairT, sizeof(double) * nn * batch));
  if (!Bs || !B2 || !T) return PF_ERR_CUDA;
  launch_ldexp_batched(n, batch, A, lda, strideA, dJ, Bs, n, nn, ctx->stream);
  ctx->launches++;
  std::vector<int> ok;
  {
    const int rc = pair_certificates(ctx, Bs, n, nn, n, batch, c, ok);
    if (rc) return rc;
  }
  int nok = 0;
  for (int v : ok) nok += v ? 1 : 0;
  if (nok == 0) return kDeclined;
  if (nok < batch) {  // mixed batch: every matrix decides for itself
    for (int b = 0; b < batch; ++b) {
      double* ob[2] = {outs[0] + b * strideOut, m->n_sets > 1 ? outs[1] + b * strideOut : nullptr};
      const int rc = large_eval(ctx, m, n, 1, A + b * strideA, lda, 0, dJ ? dJ + b : nullptr, ob, ldo, 0, flags,
                                status);
      if (rc) {
        if (status) status->batch_index = b;
        return rc;
      }
    }
    return PF_OK;
  }
  gemm(ctx, n, n, n, batch, 1.0, Bs, n, nn, Bs, n, nn, 0.0, B2, n, nn, 0.0);
  Sys s;
  const int nsys = npairs * batch;
  if (!make_sys(ctx, s, n, nsys, kWsLargeM)) return PF_ERR_CUDA;
  double* R = static_cast<double*>(workspace(ctx, kWsLargeR, sizeof(double) * s.stride() * nsys));
  auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * nsys));
  int* d_piv = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * nsys * 2));
  if (!R || !d_mx || !d_piv) return PF_ERR_CUDA;
  std::vector<double> c2(npairs);
  for (int q = 0; q < npairs; ++q) c2[q] = c[q] * c[q];
  double* d_c2 = upload(ctx, kWsSmallArrays + 1, c2);
  cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long) * nsys, ctx->stream);
  form_shifted_kernel<<<dim3(grid2(s.stride(), nsys), nsys), 256, 0, ctx->stream>>>(B2, n, nn, n, s.np, batch, d_c2,
                                                                                 nullptr, s.M, d_mx);
  ctx->launches++;
  FactorResult fr = factor_systems(ctx, s, n, d_mx, flags, d_piv, d_piv + (size_t)n * nsys, 1e-14, true);
  if (fr.rc) return fr.rc;  // kDeclined (an I - c^2 B^2 failed the certificate) or a CUDA error
  form_rhs_kernel<<<dim3(grid2(s.stride(), nsys), nsys), 256, 0, ctx->stream>>>(B2, n, nn, n, s.np, s.np, n, batch, d_c2,
                                                                             nullptr, 1, nullptr, R, s.stride());
  ctx->launches++;
  trsm_left_lower(ctx, s, 0, s.np, R, s.np, s.stride(), s.np);
  trsm_left_upper(ctx, s, 0, s.np, R, s.np, s.stride(), s.np);
  std::vector<int> tz(npairs);
  for (int q = 0; q < npairs; ++q) tz[q] = q;
  int* d_tz = upload(ctx, kWsSmallArrays + 2, tz);
  // E_B of every weight set into its output, E_A into T / T2: one pass over the solutions
  double* T2 = m->n_sets > 1 ? static_cast<double*>(workspace(ctx, kWsPairT2, sizeof(double) * nn * batch)) : nullptr;
  if (m->n_sets > 1 && !T2) return PF_ERR_CUDA;
  std::vector<double> wall(4 * (size_t)npairs);
  AccSets sets{};
  sets.n = 2 * m->n_sets;
  for (int q = 0; q < m->n_sets; ++q) {
    double consta = 0.0;
    for (int t = 0; t < npairs; ++t) {
      const double wp = m->weights[q * m->n_terms + ip[t]], wm = m->weights[q * m->n_terms + im[t]];
      wall[(2 * q + 1) * npairs + t] = (wp - wm) * c[t];  // E_A
      wall[(2 * q) * npairs + t] = wp + wm;              // E_B
      consta += wall[(2 * q + 1) * npairs + t];
    }
    sets.s[2 * q] = AccSet{nullptr, 0.0, 0.0, 0.0, 0, outs[q], ldo, strideOut};
    sets.s[2 * q + 1] = AccSet{nullptr, consta, 0.0, 0.0, 1, q == 0 ? T : T2, n, nn};
  }
  double* d_wall = upload(ctx, kWsSmallArrays + 3, wall);
  for (int o = 0; o < sets.n; ++o) sets.s[o].w = d_wall + (size_t)o * npairs;
  accumulate_sets_kernel<<<dim3(grid2(nn, batch), batch), 256, 0, ctx->stream>>>(
      R, s.np, s.stride(), n, n, batch, npairs, d_tz, sets, nullptr, 0, 0, nullptr, nullptr, 0, 0);
  ctx->launches++;
  for (int q = 0; q < m->n_sets; ++q) {
    gemm(ctx, n, n, n, batch, 1.0, q == 0 ? T : T2, n, nn, Bs, n, nn, 1.0, outs[q], ldo, strideOut, m->constant[q]);
  }
  return cuda_fail(cudaGetLastError());
}

static int large_eval_chunk(pf_context* ctx, const pf_method* m, int n, int batch, const double* A, int64_t lda,
                            int64_t strideA, const int* dJ, double* const* outs, int64_t ldo, int64_t strideOut,
                            int flags, pf_status* status) {
  if (status) std::memset(status, 0, sizeof(*status));
  if (batch == 0 || n == 0) return PF_OK;
  {
    const int rc = large_eval_pairs(ctx, m, n, batch, A, lda, strideA, dJ, outs, ldo, strideOut, flags, status);
    if (rc != kDeclined) return rc;
    if (status) std::memset(status, 0, sizeof(*status));
  }
  std::vector<int> nz;
  for (int i = 0; i < m->n_terms; ++i)
    if (m->shifts[i] != 0.0) nz.push_back(i);
  const int P = (int)nz.size();
  const bool residual = m->form == PF_FORM_RESIDUAL;
  Sys s;
  const int nsys = P * batch;
  if (!make_sys(ctx, s, n, nsys, kWsLargeM)) return PF_ERR_CUDA;
  double* R = static_cast<double*>(workspace(ctx, kWsLargeR, sizeof(double) * s.stride() * std::max(nsys, 1)));
  auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * std::max(nsys, 1)));
  int* d_piv = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * std::max(nsys, 1) * 2));
  if (!R || !d_mx || !d_piv) return PF_ERR_CUDA;
  int* d_perm = d_piv + (size_t)n * std::max(nsys, 1);
  std::vector<double> sh(P);
  for (int q = 0; q < P; ++q) sh[q] = m->shifts[nz[q]];
  double* d_sh = upload(ctx, kWsSmallArrays + 1, sh);
  bool pivoted = false;
  if (nsys > 0) {
    cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long) * nsys, ctx->stream);
    form_shifted_kernel<<<dim3(grid2(s.stride(), nsys), nsys), 256, 0, ctx->stream>>>(A, lda, strideA, n, s.np, batch,
                                                                                   d_sh, dJ, s.M, d_mx);
    ctx->launches++;
    FactorResult fr = factor_systems(ctx, s, n, d_mx, flags, d_piv, d_perm, 1e-14);
    if (fr.rc) {
      if (status) {
        status->code = fr.rc;
        if (fr.z >= 0) {
          status->batch_index = fr.z % batch;
          status->shift_index = nz[fr.z / batch] + 1;
          status->column = fr.st.column;
          status->pivot_magnitude = fr.st.pivot_magnitude;
          status->scale = fr.scale.empty() ? 0.0 : fr.scale[fr.z];
        }
      }
      return fr.rc;
    }
    pivoted = fr.pivoted;
    form_rhs_kernel<<<dim3(grid2(s.stride(), nsys), nsys), 256, 0, ctx->stream>>>(
        A, lda, strideA, n, s.np, s.np, n, batch, d_sh, dJ, residual ? 1 : 0, pivoted ? d_perm : nullptr, R,
        s.stride());
    ctx->launches++;
    trsm_left_lower(ctx, s, 0, s.np, R, s.np, s.stride(), s.np);
    trsm_left_upper(ctx, s, 0, s.np, R, s.np, s.stride(), s.np);
  }
  // poly part needs B^2 when any d2 != 0
  double* B2 = nullptr;
  bool need_b2 = false;
  for (int q = 0; q < m->n_sets && m->has_poly; ++q) need_b2 |= m->poly[3 * q + 2] != 0.0;
  if (need_b2) {
    double* Bs = static_cast<double*>(workspace(ctx, kWsLargeB, sizeof(double) * (size_t)n * n * batch));
    B2 = static_cast<double*>(workspace(ctx, kWsLargeX2, sizeof(double) * (size_t)n * n * batch));
    if (!Bs || !B2) return PF_ERR_CUDA;
    launch_ldexp_batched(n, batch, A, lda, strideA, dJ, Bs, n, (int64_t)n * n, ctx->stream);
    ctx->launches++;
    gemm(ctx, n, n, n, batch, 1.0, Bs, n, (int64_t)n * n, Bs, n, (int64_t)n * n, 0.0, B2, n, (int64_t)n * n, 0.0);
  }
  // every weight set's sum in one pass over the solutions (the term list is the same for all sets)
  std::vector<int> tz;
  int slot = 0;
  for (int i = 0; i < m->n_terms; ++i) {
    if (m->shifts[i] != 0.0)
      tz.push_back(slot++);
    else if (!residual)
      tz.push_back(-1);
  }
  const int nt = (int)tz.size();
  std::vector<double> wall((size_t)m->n_sets * nt);
  AccSets sets{};
  sets.n = m->n_sets;
  const bool add_poly = residual || m->has_poly;
  for (int q = 0; q < m->n_sets; ++q) {
    int t = 0;
    for (int i = 0; i < m->n_terms; ++i)
      if (m->shifts[i] != 0.0 || !residual) wall[(size_t)q * nt + t++] = m->weights[q * m->n_terms + i];
    const double constant = residual ? m->constant[q] : (m->has_poly ? m->poly[3 * q] : 0.0);
    const double d1 = m->has_poly ? m->poly[3 * q + 1] : 0.0, d2 = m->has_poly ? m->poly[3 * q + 2] : 0.0;
    sets.s[q] = AccSet{nullptr, constant, d1, d2, add_poly ? 1 : 0, outs[q], ldo, strideOut};
  }
  int* d_tz = upload(ctx, kWsSmallArrays + 2, tz);
  double* d_wall = upload(ctx, kWsSmallArrays + 3, wall);
  for (int q = 0; q < m->n_sets; ++q) sets.s[q].w = d_wall + (size_t)q * nt;
  accumulate_sets_kernel<<<dim3(grid2((int64_t)n * n, batch), batch), 256, 0, ctx->stream>>>(
      R, s.np, s.stride(), n, n, batch, nt, d_tz, sets, A, lda, strideA, dJ, B2, n, (int64_t)n * n);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------------
// Block action in pair mode (see large_eval_pairs): B = A / N; every pair's system I - c^2 B^2 is
// factored once; per substep Y_p = (I - c_p^2 B^2)^-1 (c_p B X) for all pairs in one batched solve,
// U = a0 X + sum_p cm_p Y_p, V = sum_p cp_p c_p Y_p, and X <- U + B V (one extra n^2 k product per
// substep instead of the second solve of every pair).
int large_action_pairs(pf_context* ctx, const pf_method* m, int n, int k, const double* A, int64_t lda,
                       const double* V, int64_t ldv, int substeps, double* out, int64_t ldo, int flags) {
  std::vector<double> c;
  std::vector<int> ip, im;
  if (!plan_pairs(m, flags, c, ip, im)) return kDeclined;
  const int npairs = (int)c.size();
  const int np = round64(n);
  const int64_t st = (int64_t)np * np;
  double* Bp = static_cast<double*>(workspace(ctx, kWsLargeB, sizeof(double) * st));
  if (!Bp) return PF_ERR_CUDA;
  scale_pad_kernel<<<grid_for(st), 256, 0, ctx->stream>>>(A, lda, n, np, 1.0 / substeps, Bp);
  ctx->launches++;
  std::vector<int> ok;
  {
    const int rc = pair_certificates(ctx, Bp, np, 0, n, 1, c, ok);
    if (rc) return rc;
    if (!ok[0]) return kDeclined;
  }
  double* B2 = static_cast<double*>(workspace(ctx, kWsPairB2, sizeof(double) * st));
  if (!B2) return PF_ERR_CUDA;
  gemm(ctx, np, np, np, 1, 1.0, Bp, np, 0, Bp, np, 0, 0.0, B2, np, 0, 0.0);
  Sys s;
  if (!make_sys(ctx, s, n, npairs, kWsLargeM)) return PF_ERR_CUDA;
  const size_t blk = (size_t)np * k;
  double* R = static_cast<double*>(workspace(ctx, kWsLargeR, sizeof(double) * blk * npairs));
  double* X = static_cast<double*>(workspace(ctx, kWsT1, sizeof(double) * blk * 4));
  auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * npairs));
  int* d_piv = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * npairs * 2));
  if (!R || !X || !d_mx || !d_piv) return PF_ERR_CUDA;
  std::vector<double> c2(npairs);
  for (int q = 0; q < npairs; ++q) c2[q] = c[q] * c[q];
  double* d_c2 = upload(ctx, kWsSmallArrays + 1, c2);
  double* d_c = upload(ctx, kWsSmallArrays + 4, c);
  cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long) * npairs, ctx->stream);
  form_shifted_kernel<<<dim3(grid2(st, npairs), npairs), 256, 0, ctx->stream>>>(B2, np, 0, n, np, 1, d_c2, nullptr, s.M,
                                                                           d_mx);
  ctx->launches++;
  FactorResult fr = factor_systems(ctx, s, n, d_mx, flags, d_piv, d_piv + (size_t)n * npairs, 1e-14, true);
  if (fr.rc) return fr.rc;  // kDeclined or a CUDA error
  const int nb = big_block(np);
  double* binv = nullptr;
  if (nb) {
    binv = static_cast<double*>(workspace(ctx, kWsLargeBinv, sizeof(double) * big_inverse_stride(np, nb) * npairs));
    if (!binv || !build_big_inverses(ctx, s, nb, binv)) return PF_ERR_CUDA;
  }
  double* BX = X + blk;
  double* Vs = X + 2 * blk;
  double* Xn = X + 3 * blk;
  cudaMemsetAsync(X, 0, sizeof(double) * blk * 4, ctx->stream);  // padding rows stay zero
  copy2d_kernel<<<dim3(grid_for((int64_t)n * k), 1), 256, 0, ctx->stream>>>(n, k, 1.0, V, ldv, 0, X, k, 0);
  ctx->launches++;
  std::vector<int> tz(npairs);
  std::vector<double> wu(npairs), wv(npairs);
  for (int q = 0; q < npairs; ++q) {
    tz[q] = q;
    const double wp = m->weights[ip[q]], wm = m->weights[im[q]];
    wu[q] = wp - wm;
    wv[q] = (wp + wm) * c[q];
  }
  int* d_tz = upload(ctx, kWsSmallArrays + 2, tz);
  double* d_wu = upload(ctx, kWsSmallArrays + 3, wu);
  double* d_wv = upload(ctx, kWsSmallArrays + 5, wv);
  for (int step = 0; step < substeps; ++step) {
    gemm(ctx, np, k, np, 1, 1.0, Bp, np, 0, X, k, 0, 0.0, BX, k, 0, 0.0);
    form_rhs_kernel<<<dim3(grid2((int64_t)blk, npairs), npairs), 256, 0, ctx->stream>>>(BX, k, 0, n, np, k, k, 1, d_c, nullptr,
                                                                                  1, nullptr, R, (int64_t)blk);
    ctx->launches++;
    const int rc = solve_lu(ctx, s, binv, nb, R, k, (int64_t)blk);
    if (rc) return rc;
    action_accumulate_kernel<<<grid_for((int64_t)n * k), 256, 0, ctx->stream>>>(
        R, k, (int64_t)blk, X, k, n, k, npairs, d_tz, d_wu, 1, m->constant[0], 0, 0.0, 0.0, nullptr, nullptr, Xn, k);
    action_accumulate_kernel<<<grid_for((int64_t)n * k), 256, 0, ctx->stream>>>(
        R, k, (int64_t)blk, X, k, n, k, npairs, d_tz, d_wv, 0, 0.0, 0, 0.0, 0.0, nullptr, nullptr, Vs, k);
    ctx->launches += 2;
    gemm(ctx, np, k, np, 1, 1.0, Bp, np, 0, Vs, k, 0, 1.0, Xn, k, 0, 0.0);  // X <- a0 X + U + B V
    std::swap(X, Xn);
  }
  copy2d_kernel<<<dim3(grid_for((int64_t)n * k), 1), 256, 0, ctx->stream>>>(n, k, 1.0, X, k, 0, out, ldo, 0);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

int large_action(pf_context* ctx, const pf_method* m, int n, int k, const double* A, int64_t lda, const double* V,
                 int64_t ldv, int substeps, double* out, int64_t ldo, int flags, pf_status* status) {
  if (status) std::memset(status, 0, sizeof(*status));
  {
    const int rc = large_action_pairs(ctx, m, n, k, A, lda, V, ldv, substeps, out, ldo, flags);
    if (rc != kDeclined) return rc;
  }
  std::vector<int> nz;
  for (int i = 0; i < m->n_terms; ++i)
    if (m->shifts[i] != 0.0) nz.push_back(i);
  const int P = (int)nz.size();
  const bool residual = m->form == PF_FORM_RESIDUAL;
  const bool hybrid = m->has_poly != 0;
  Sys s;
  if (!make_sys(ctx, s, n, P, kWsLargeM)) return PF_ERR_CUDA;
  const int np = s.np;
  double* Bp = static_cast<double*>(workspace(ctx, kWsLargeB, sizeof(double) * s.stride()));
  const size_t blk = (size_t)np * k;
  double* R = static_cast<double*>(workspace(ctx, kWsLargeR, sizeof(double) * blk * std::max(P, 1)));
  double* X = static_cast<double*>(workspace(ctx, kWsT1, sizeof(double) * blk * 4));
  auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * std::max(P, 1)));
  int* d_piv = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * std::max(P, 1) * 2));
  if (!Bp || !R || !X || !d_mx || !d_piv) return PF_ERR_CUDA;
  int* d_perm = d_piv + (size_t)n * std::max(P, 1);
  double* BX = X + blk;
  double* B2X = X + 2 * blk;
  double* Xn = X + 3 * blk;
  // B = A * (1.0 / N) (action.cpp:330-334), zero padded
  const double inv = 1.0 / substeps;
  scale_pad_kernel<<<grid_for(s.stride()), 256, 0, ctx->stream>>>(A, lda, n, np, inv, Bp);
  ctx->launches++;
  std::vector<double> sh(P);
  for (int q = 0; q < P; ++q) sh[q] = m->shifts[nz[q]];
  double* d_sh = upload(ctx, kWsSmallArrays + 1, sh);
  bool pivoted = false;
  if (P > 0) {
    cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long) * P, ctx->stream);
    form_shifted_kernel<<<dim3(grid2(s.stride(), P), P), 256, 0, ctx->stream>>>(Bp, np, 0, n, np, 1, d_sh, nullptr,
                                                                               s.M, d_mx);
    ctx->launches++;
    FactorResult fr = factor_systems(ctx, s, n, d_mx, flags, d_piv, d_perm, 1e-14);
    if (fr.rc) {
      if (status) {
        status->code = fr.rc;
        if (fr.z >= 0) {
          status->shift_index = nz[fr.z] + 1;
          status->column = fr.st.column;
          status->pivot_magnitude = fr.st.pivot_magnitude;
          status->scale = fr.scale[fr.z];
        }
      }
      return fr.rc;
    }
    pivoted = fr.pivoted;
  }
  // factored once, solved `substeps` times: explicit inverses of the big diagonal blocks
  const int nb = P > 0 ? big_block(np) : 0;
  double* binv = nullptr;
  if (nb) {
    binv = static_cast<double*>(workspace(ctx, kWsLargeBinv, sizeof(double) * big_inverse_stride(np, nb) * P));
    if (!binv || !build_big_inverses(ctx, s, nb, binv)) return PF_ERR_CUDA;
  }
  // X = V (padded rows are zero, in both iterate buffers)
  cudaMemsetAsync(X, 0, sizeof(double) * blk, ctx->stream);
  cudaMemsetAsync(Xn, 0, sizeof(double) * blk, ctx->stream);
  copy2d_kernel<<<dim3(grid_for((int64_t)n * k), 1), 256, 0, ctx->stream>>>(n, k, 1.0, V, ldv, 0, X, k, 0);
  ctx->launches++;
  std::vector<int> tz;
  std::vector<double> w;
  {
    int slot = 0;
    for (int i = 0; i < m->n_terms; ++i) {
      if (m->shifts[i] != 0.0) {
        tz.push_back(slot++);
        w.push_back(m->weights[i]);
      } else if (!residual) {
        tz.push_back(-1);
        w.push_back(m->weights[i]);
      }
    }
  }
  int* d_tz = upload(ctx, kWsSmallArrays + 2, tz);
  double* d_w = upload(ctx, kWsSmallArrays + 3, w);
  std::vector<double> ones(std::max(P, 1), 1.0);
  double* d_one = upload(ctx, kWsSmallArrays + 9, ones);
  const double constant = residual ? m->constant[0] : (hybrid ? m->poly[0] : 0.0);
  const double d1 = hybrid ? m->poly[1] : 0.0, d2 = hybrid ? m->poly[2] : 0.0;
  for (int step = 0; step < substeps; ++step) {
    if (residual || hybrid) gemm(ctx, np, k, np, 1, 1.0, Bp, np, 0, X, k, 0, 0.0, BX, k, 0, 0.0);
    if (hybrid) gemm(ctx, np, k, np, 1, 1.0, Bp, np, 0, BX, k, 0, 0.0, B2X, k, 0, 0.0);
    if (P > 0) {
      // R_i = c_i B X (residual, action.cpp:252-258) or X (plain), rows permuted when pivoted
      // R_i = c_i (B X) (residual) or 1 * X (plain; unit "shift" table), rows permuted when pivoted
      form_rhs_kernel<<<dim3(grid2((int64_t)blk, P), P), 256, 0, ctx->stream>>>(
          residual ? BX : X, k, 0, n, np, k, k, 1, residual ? d_sh : d_one, nullptr, 1, pivoted ? d_perm : nullptr, R,
          (int64_t)blk);
      ctx->launches++;
      const int rc = solve_lu(ctx, s, binv, nb, R, k, (int64_t)blk);
      if (rc) return rc;
    }
    action_accumulate_kernel<<<grid_for((int64_t)n * k), 256, 0, ctx->stream>>>(
        R, k, (int64_t)blk, X, k, n, k, (int)tz.size(), d_tz, d_w, (residual || hybrid) ? 1 : 0, constant,
        hybrid ? 1 : 0, d1, d2, BX, B2X, Xn, k);
    ctx->launches++;
    std::swap(X, Xn);
  }
  copy2d_kernel<<<dim3(grid_for((int64_t)n * k), 1), 256, 0, ctx->stream>>>(n, k, 1.0, X, k, 0, out, ldo, 0);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------------
static int large_lu_factor_chunk(pf_context* ctx, int n, int batch, double* A, int64_t lda, int64_t strideA,
                                 int* piv, double pivot_rel_tol, int flags, pf_status* status) {
  if (status) std::memset(status, 0, sizeof(*status));
  if (batch == 0 || n == 0) return PF_OK;
  Sys s;
  if (!make_sys(ctx, s, n, batch, kWsLargeM)) return PF_ERR_CUDA;
  auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * batch));
  int* d_piv = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * batch * 2));
  if (!d_mx || !d_piv) return PF_ERR_CUDA;
  int* d_perm = d_piv + (size_t)n * batch;
  cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long) * batch, ctx->stream);
  // n a multiple of 64 and a packed batch: factor in the caller's buffer (no padded copy in and out)
  const bool in_place = s.np == n && lda == n && strideA == (int64_t)n * n;
  load_padded_kernel<<<dim3(grid2(s.stride(), batch), batch), 256, 0, ctx->stream>>>(A, lda, strideA, n, s.np,
                                                                                      in_place ? nullptr : s.M, d_mx);
  ctx->launches++;
  if (in_place) s.M = A;
  FactorResult fr = factor_systems(ctx, s, n, d_mx, flags, d_piv, d_perm, pivot_rel_tol);
  if (fr.rc) {
    if (status) {
      status->code = fr.rc;
      status->batch_index = std::max(fr.z, 0);
      status->column = fr.st.column;
      status->pivot_magnitude = fr.st.pivot_magnitude;
      status->scale = fr.z >= 0 ? fr.scale[fr.z] : 0.0;
    }
    return fr.rc;
  }
  if (!in_place) {
    copy2d_kernel<<<dim3(grid2((int64_t)n * n, batch), batch), 256, 0, ctx->stream>>>(n, n, 1.0, s.M, s.np, s.stride(),
                                                                                 A, lda, strideA);
    ctx->launches++;
  }
  if (piv) {
    if (fr.pivoted) {  // every system's swap sequence (identity for the certified ones)
      cudaMemcpyAsync(piv, d_piv, sizeof(int) * (size_t)n * batch, cudaMemcpyDeviceToDevice, ctx->stream);
    } else {
      iota_kernel<<<dim3((n + 255) / 256, batch), 256, 0, ctx->stream>>>(piv, n);
      ctx->launches++;
    }
  }
  return cuda_fail(cudaGetLastError());
}

int large_lu_solve(pf_context* ctx, int n, int k, int batch, const double* LU, int64_t lda, int64_t strideLU,
                   const int* piv, double* R, int64_t ldr, int64_t strideR) {
  if (batch == 0 || n == 0 || k == 0) return PF_OK;
  Sys s;
  if (!make_sys(ctx, s, n, batch, kWsLargeM)) return PF_ERR_CUDA;
  auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * batch));
  int* d_perm = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * batch * 2));
  const size_t blk = (size_t)s.np * k;
  double* X = static_cast<double*>(workspace(ctx, kWsLargeR, sizeof(double) * blk * batch));
  if (!d_mx || !d_perm || !X) return PF_ERR_CUDA;
  load_padded_kernel<<<dim3(grid2(s.stride(), batch), batch), 256, 0, ctx->stream>>>(LU, lda, strideLU, n, s.np, s.M, d_mx);
  perm_from_piv_kernel<<<batch, 32, 0, ctx->stream>>>(piv, n, d_perm, nullptr);
  ctx->launches += 2;
  diag_inverses(ctx, s);
  std::vector<double> ones(batch, 1.0);
  double* d_one = upload(ctx, kWsSmallArrays + 9, ones);
  // X = P R (padded zeros): form_rhs with c = 1, batch 1 per system via z = b (one shift slot)
  form_rhs_kernel<<<dim3(grid2((int64_t)blk, batch), batch), 256, 0, ctx->stream>>>(R, ldr, strideR, n, s.np, k, k, batch,
                                                                               d_one, nullptr, 1, d_perm, X,
                                                                               (int64_t)blk);
  ctx->launches++;
  trsm_left_lower(ctx, s, 0, s.np, X, k, (int64_t)blk, k);
  trsm_left_upper(ctx, s, 0, s.np, X, k, (int64_t)blk, k);
  copy2d_kernel<<<dim3(grid2((int64_t)n * k, batch), batch), 256, 0, ctx->stream>>>(n, k, 1.0, X, k, (int64_t)blk, R, ldr,
                                                                               strideR);
  ctx->launches++;
  return cuda_fail(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------------
// ActionOperator on a dense A (action.hpp:68-82, action.cpp:300-325): B = A * (1/N) and the LU
// factors of the owned shifts persist; apply() performs one substep r(B) V restricted to the owned
// terms (a shift subset per rank for the multi-GPU partition), optionally with the poly part.
int action_op_create(pf_context* ctx, const pf_method* m, int n, const double* A, int64_t lda, int substeps,
                     const int* owned, int flags, pf_status* status, pf_action_op** out) {
  if (status) std::memset(status, 0, sizeof(*status));
  auto* op = new pf_action_op();
  op->ctx = ctx;
  op->n = n;
  op->np = round64(n);
  op->substeps = substeps;
  op->form = m->form;
  op->hybrid = m->has_poly ? 1 : 0;
  const bool residual = m->form == PF_FORM_RESIDUAL;
  op->constant = residual ? m->constant[0] : (op->hybrid ? m->poly[0] : 0.0);
  op->d1 = op->hybrid ? m->poly[1] : 0.0;
  op->d2 = op->hybrid ? m->poly[2] : 0.0;
  for (int i = 0; i < m->n_terms; ++i) {
    const bool nonzero = m->shifts[i] != 0.0;
    if (!nonzero && residual) continue;  // residual zero shifts fold into a_0
    if (owned && !owned[i]) continue;
    op->term_index.push_back(i);
    op->term_weight.push_back(m->weights[i]);
    if (nonzero) {
      op->term_slot.push_back((int)op->shifts.size());
      op->shifts.push_back(m->shifts[i]);
    } else {
      op->term_slot.push_back(-1);
    }
  }
  const int P = (int)op->shifts.size();
  const int64_t st = (int64_t)op->np * op->np;
  const int64_t inv_stride = (int64_t)(op->np / kB) * 2 * kB * kB;
  bool okalloc = cudaMalloc(&op->B, sizeof(double) * st) == cudaSuccess;
  if (P > 0) {
    okalloc = okalloc && cudaMalloc(&op->M, sizeof(double) * st * P) == cudaSuccess;
    okalloc = okalloc && cudaMalloc(&op->inv, sizeof(double) * inv_stride * P) == cudaSuccess;
    okalloc = okalloc && cudaMalloc(&op->perm, sizeof(int) * (size_t)n * P) == cudaSuccess;
    okalloc = okalloc && cudaMalloc(&op->d_shifts, sizeof(double) * P) == cudaSuccess;
    okalloc = okalloc && cudaMalloc(&op->d_ones, sizeof(double) * P) == cudaSuccess;
  }
  if (!okalloc) {
    action_op_destroy(op);
    return PF_ERR_CUDA;
  }
  scale_pad_kernel<<<grid_for(st), 256, 0, ctx->stream>>>(A, lda, n, op->np, 1.0 / substeps, op->B);
  ctx->launches++;
  if (P > 0) {
    std::vector<double> ones(P, 1.0);
    cudaMemcpyAsync(op->d_shifts, op->shifts.data(), sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(op->d_ones, ones.data(), sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream);
    auto* d_mx = static_cast<unsigned long long*>(workspace(ctx, kWsLargeAux, sizeof(unsigned long long) * P));
    int* d_piv = static_cast<int*>(workspace(ctx, kWsLargePiv, sizeof(int) * (size_t)n * P));
    if (!d_mx || !d_piv) {
      action_op_destroy(op);
      return PF_ERR_CUDA;
    }
    cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long) * P, ctx->stream);
    form_shifted_kernel<<<dim3(grid2(st, P), P), 256, 0, ctx->stream>>>(op->B, op->np, 0, n, op->np, 1, op->d_shifts,
                                                                       nullptr, op->M, d_mx);
    ctx->launches++;
    Sys s{op->M, op->np, P, op->inv, inv_stride};
    FactorResult fr = factor_systems(ctx, s, n, d_mx, flags, d_piv, op->perm, 1e-14);
    if (fr.rc) {
      if (status) {
        status->code = fr.rc;
        if (fr.z >= 0) {
          int q = 0;
          for (size_t t = 0; t < op->term_slot.size(); ++t)
            if (op->term_slot[t] == fr.z) q = op->term_index[t];
          status->shift_index = q + 1;
          status->column = fr.st.column;
          status->pivot_magnitude = fr.st.pivot_magnitude;
          status->scale = fr.scale[fr.z];
        }
      }
      const int rc = fr.rc;
      action_op_destroy(op);
      return rc;
    }
    op->pivoted = fr.pivoted;
    op->nbig = big_block(op->np);
    if (op->nbig) {
      if (cudaMalloc(&op->binv, sizeof(double) * big_inverse_stride(op->np, op->nbig) * P) != cudaSuccess ||
          !build_big_inverses(ctx, s, op->nbig, op->binv)) {
        action_op_destroy(op);
        return PF_ERR_CUDA;
      }
    }
  }
  *out = op;
  return cuda_fail(cudaGetLastError());
}

int action_op_apply(pf_action_op* op, const double* V, int64_t ldv, int k, double* out, int64_t ldo,
                    int include_poly, double* terms) {
  pf_context* ctx = op->ctx;
  const int n = op->n, np = op->np, P = (int)op->shifts.size();
  const size_t blk = (size_t)np * k;
  const bool residual = op->form == PF_FORM_RESIDUAL;
  double* X = static_cast<double*>(workspace(ctx, kWsT1, sizeof(double) * blk * 3));
  double* R = static_cast<double*>(workspace(ctx, kWsLargeR, sizeof(double) * blk * std::max(P, 1)));
  if (!X || !R) return PF_ERR_CUDA;
  double* BX = X + blk;
  double* B2X = X + 2 * blk;
  cudaMemsetAsync(X, 0, sizeof(double) * blk, ctx->stream);
  copy2d_kernel<<<dim3(grid_for((int64_t)n * k), 1), 256, 0, ctx->stream>>>(n, k, 1.0, V, ldv, 0, X, k, 0);
  ctx->launches++;
  if (residual || op->hybrid) gemm(ctx, np, k, np, 1, 1.0, op->B, np, 0, X, k, 0, 0.0, BX, k, 0, 0.0);
  if (op->hybrid) gemm(ctx, np, k, np, 1, 1.0, op->B, np, 0, BX, k, 0, 0.0, B2X, k, 0, 0.0);
  if (P > 0) {
    // R_i = c_i (B X) (residual, action.cpp:252-258) or X (plain), rows permuted when pivoted
    form_rhs_kernel<<<dim3(grid2((int64_t)blk, P), P), 256, 0, ctx->stream>>>(
        residual ? BX : X, k, 0, n, np, k, k, 1, residual ? op->d_shifts : op->d_ones, nullptr, 1,
        op->pivoted ? op->perm : nullptr, R, (int64_t)blk);
    ctx->launches++;
    Sys s{op->M, np, P, op->inv, (int64_t)(np / kB) * 2 * kB * kB};
    const int rc = solve_lu(ctx, s, op->binv, op->nbig, R, k, (int64_t)blk);
    if (rc) return rc;
  }
  const int nt = (int)op->term_slot.size();
  int* d_tz = upload(ctx, kWsSmallArrays + 12, op->term_slot);
  double* d_w = upload(ctx, kWsSmallArrays + 13, op->term_weight);
  const bool add_poly = include_poly && (residual || op->hybrid);
  action_accumulate_kernel<<<grid_for((int64_t)n * k), 256, 0, ctx->stream>>>(
      R, k, (int64_t)blk, X, k, n, k, nt, d_tz, d_w, add_poly ? 1 : 0, op->constant, op->hybrid, op->d1, op->d2, BX,
      B2X, out, ldo);
  ctx->launches++;
  if (terms) {
    // the same products the accumulation adds, one n x k block per owned term (ascending shift
    // index), then c X and d1 BX + d2 B^2 X: an ordered sum of these reproduces `out` bit for bit
    const size_t nk = (size_t)n * k;
    for (int t = 0; t < nt; ++t) {
      const int slot = op->term_slot[t];
      const double* src = slot >= 0 ? R + (size_t)slot * blk : X;
      copy2d_kernel<<<dim3(grid_for((int64_t)nk), 1), 256, 0, ctx->stream>>>(n, k, op->term_weight[t], src, k, 0,
                                                                             terms + t * nk, k, 0);
      ctx->launches++;
    }
    if (add_poly) {
      copy2d_kernel<<<dim3(grid_for((int64_t)nk), 1), 256, 0, ctx->stream>>>(n, k, op->constant, X, k, 0,
                                                                             terms + nt * nk, k, 0);
      ctx->launches++;
      if (op->hybrid) {
        lincomb2_kernel<<<grid_for((int64_t)nk), 256, 0, ctx->stream>>>(n, k, op->d1, BX, op->d2, B2X, k,
                                                                        terms + (nt + 1) * nk, k);
        ctx->launches++;
      }
    }
  }
  return cuda_fail(cudaGetLastError());
}

void action_op_destroy(pf_action_op* op) {
  if (!op) return;
  if (op->ctx) cudaStreamSynchronize(op->ctx->stream);
  cudaFree(op->B);
  cudaFree(op->M);
  cudaFree(op->inv);
  cudaFree(op->perm);
  cudaFree(op->d_shifts);
  cudaFree(op->d_ones);
  cudaFree(op->binv);
  delete op;
}

}  // namespace host
}  // namespace pf

namespace pf {
namespace host {

// The large-path kernels put the system index (shift x matrix) in gridDim.y / gridDim.z, at most
// 65535: batches are processed in slices of at most 65535 / PF_MAX_TERMS matrices (status batch
// indices are rebased to the caller's batch).
constexpr int kLargeBatchChunk = 65535 / PF_MAX_TERMS;

int large_eval(pf_context* ctx, const pf_method* m, int n, int batch, const double* A, int64_t lda, int64_t strideA,
               const int* dJ, double* const* outs, int64_t ldo, int64_t strideOut, int flags, pf_status* status) {
  if (batch <= kLargeBatchChunk)
    return large_eval_chunk(ctx, m, n, batch, A, lda, strideA, dJ, outs, ldo, strideOut, flags, status);
  for (int b0 = 0; b0 < batch; b0 += kLargeBatchChunk) {
    const int nb = std::min(kLargeBatchChunk, batch - b0);
    double* o[2] = {outs[0] + (int64_t)b0 * strideOut, m->n_sets > 1 ? outs[1] + (int64_t)b0 * strideOut : nullptr};
    const int rc = large_eval_chunk(ctx, m, n, nb, A + (int64_t)b0 * strideA, lda, strideA, dJ ? dJ + b0 : nullptr, o,
                                    ldo, strideOut, flags, status);
    if (rc) {
      if (status) status->batch_index += b0;
      return rc;
    }
  }
  return PF_OK;
}

int large_lu_factor(pf_context* ctx, int n, int batch, double* A, int64_t lda, int64_t strideA, int* piv,
                    double pivot_rel_tol, int flags, pf_status* status) {
  if (batch <= kLargeBatchChunk)
    return large_lu_factor_chunk(ctx, n, batch, A, lda, strideA, piv, pivot_rel_tol, flags, status);
  for (int b0 = 0; b0 < batch; b0 += kLargeBatchChunk) {
    const int nb = std::min(kLargeBatchChunk, batch - b0);
    const int rc = large_lu_factor_chunk(ctx, n, nb, A + (int64_t)b0 * strideA, lda, strideA,
                                         piv ? piv + (int64_t)b0 * n : nullptr, pivot_rel_tol, flags, status);
    if (rc) {
      if (status) status->batch_index += b0;
      return rc;
    }
  }
  return PF_OK;
}

}  // namespace host
}  // namespace pf
