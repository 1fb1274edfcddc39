// Internal host-side declarations shared by the C-ABI translation units (not part of the ABI).
#pragma once
#include <cstdint>
#include <vector>

#include "pf_common.cuh"
#include "pf_kernels.h"

struct pf_group;  // multi-device contexts (pf_multi.cu)

struct pf_context {
  int device = 0;
  pf_group* group = nullptr;  // set on the root of pf_context_create_multi
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  pf::DevStatus* status = nullptr;
  int status_cap = 0;
  int* first_error = nullptr;
  int* h_first_error = nullptr;
  std::vector<void*> ws;
  std::vector<size_t> ws_bytes;
  unsigned long long* prof = nullptr;
  bool sticky = false;  // keep first_error across launches (pipelined async use)
  // side stream for independent branches of the large LU (created on first use)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // look-ahead streams of the large LU, one per recursion depth (created on first use): the
  // bottom-right quadrant of each trailing update runs there while the recursion factors the rest
  std::vector<cudaStream_t> aux;
  std::vector<cudaEvent_t> aux_ready, aux_done;
  bool l2_persisting = false;  // the small kernel left persisting L2 lines (reset before large GEMMs)
  int gemm_cap = 0;  // > 0: host gemm() launches persistent GEMMs on at most this many SMs
  // replayable launch graphs of the large LU recursion, keyed by its buffers and shape
  struct LuGraph {
    const double* M = nullptr;
    const double* inv = nullptr;
    int64_t inv_stride = 0;
    int np = 0, nsys = 0;
    cudaGraphExec_t exec = nullptr;  // nullptr: seen once (the next call captures)
    int64_t launches = 0;
  };
  std::vector<LuGraph> lu_graphs;
  cudaStream_t gstream = nullptr;  // private capture / replay stream (the caller's may be the legacy one)
  cudaEvent_t ev_g0 = nullptr, ev_g1 = nullptr;
};

// Dense ActionOperator (action.hpp:68-82): B = A * (1/N) and the LU factors of the owned shifts,
// persistent across applies (own allocations, not the context workspace).
struct pf_action_op {
  pf_context* ctx = nullptr;
  int n = 0, np = 0, substeps = 1;
  int form = PF_FORM_RESIDUAL, hybrid = 0;
  double constant = 0.0, d1 = 0.0, d2 = 0.0;
  std::vector<double> shifts;      // owned nonzero shifts, ascending shift index
  std::vector<int> term_index;     // shift index of every owned term (nonzero shifts + plain zero shift)
  std::vector<double> term_weight;
  std::vector<int> term_slot;      // factor slot of the term (-1: plain zero shift, term = w X)
  double* B = nullptr;             // np x np, zero padded
  double* M = nullptr;             // P_owned x np x np LU factors
  double* inv = nullptr;           // diagonal-block inverses
  int* perm = nullptr;             // P_owned x n row order (pivoted systems)
  bool pivoted = false;
  double* d_shifts = nullptr;      // device copy of `shifts`
  double* d_ones = nullptr;
  // explicit inverses of the nbig x nbig diagonal blocks of L and U (per system: for block q,
  // Linv at q * 2 * nbig^2, Uinv at (2q + 1) * nbig^2), for the blocked thin-RHS solves
  int nbig = 0;
  double* binv = nullptr;
};

namespace pf {
namespace host {

// Every ABI entry point runs on its context's device and restores the caller's current device
// afterwards: one process may drive several GPUs through several contexts, and the caller's
// current device may be any of them.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const pf_context* ctx) {
    if (!ctx || cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      return;
    }
    if (prev == ctx->device)
      prev = -1;
    else
      cudaSetDevice(ctx->device);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

void group_destroy(pf_context* root);  // members, streams and NCCL communicators of a multi context

int action_op_create(pf_context* ctx, const pf_method* m, int n, const double* A, int64_t lda, int substeps,
                     const int* owned, int flags, pf_status* status, pf_action_op** out);
int action_op_apply(pf_action_op* op, const double* V, int64_t ldv, int k, double* out, int64_t ldo,
                    int include_poly, double* terms);
void action_op_destroy(pf_action_op* op);

int cuda_fail(cudaError_t e);
void* workspace(pf_context* ctx, int slot, size_t bytes);
int ensure_status(pf_context* ctx, int batch);
int collect_status(pf_context* ctx, int batch, int flags, pf_status* out);
int bad(pf_status* st);
bool fill_method(const pf_method* m, SmallParams& p);
int launch_small(pf_context* ctx, SmallParams& p);
// PF_FLAG_REFERENCE_ORDER (n <= 128): ref_order.cu, dense.cpp's exact operation order
int launch_small_reference_order(pf_context* ctx, SmallParams& p);
void gemm(pf_context* ctx, int m, int n, int k, int batch, double alpha, const double* A, int64_t lda, int64_t sA,
          const double* B, int64_t ldb, int64_t sB, double beta, double* C, int64_t ldc, int64_t sC, double gamma,
          const int* jmask = nullptr, int step = 0, const double* pass = nullptr, const double* sd_ref = nullptr,
          double* sd_d = nullptr, double* sd_e = nullptr);
int max_j(pf_context* ctx, const int* dJ, int batch, int* out);

// workspace slots (each slot is an independently grown device buffer)
enum Slot {
  kWsJ = 0,
  kWsT1 = 1,
  kWsT2 = 2,
  kWsT3 = 3,
  kWsT4 = 4,
  kWsNorm = 5,
  kWsLargeM = 10,
  kWsLargeR = 11,
  kWsLargeInv = 12,
  kWsLargeAux = 13,
  kWsLargePiv = 14,
  kWsLargeB = 15,
  kWsLargeX2 = 16,
  kWsLargeBinv = 18,    // explicit inverses of the big diagonal blocks (thin-RHS solves)
  kWsPairB = 19,        // large pair mode: B = 2^-j A, B^2, E_A
  kWsPairB2 = 21,
  kWsPairT = 22,
  kWsPairT2 = 23,       // large pair mode: E_A of the second weight set
  kWsGemmSplit = 24,    // split-K partial products of thin GEMMs
  kWsTriTmp = 26,       // triangular block inversion temporaries
  kWsBandA = 27,        // banded action: scaled band, factors, per-shift solutions, iterates
  kWsBandF = 28,
  kWsBandY = 29,
  kWsBandX = 30,
  kWsBandRec = 31,      // banded action: per-row coefficient records of the bulk-copy kernel
  kWsScratch = 20,      // per-SM accumulator slots of the small kernel
  kWsRefX = 32,         // reference-order evaluator: per-matrix solve / product scratch
  kWsSmallArrays = 64,  // small uploaded tables: kWsSmallArrays + i (slots grow on demand)
};

// Large-n evaluation (pf_large.cu): outs[s] = r_s(2^-j A_b) for every weight set, any n.
// dJ: per-matrix squaring counts (device) or nullptr for j = 0.
int large_eval(pf_context* ctx, const pf_method* m, int n, int batch, const double* A, int64_t lda, int64_t strideA,
               const int* dJ, double* const* outs, int64_t ldo, int64_t strideOut, int flags, pf_status* status);

// n x k block action (pf_large.cu)
int large_action(pf_context* ctx, const pf_method* m, int n, int k, const double* A, int64_t lda, const double* V,
                 int64_t ldv, int substeps, double* out, int64_t ldo, int flags, pf_status* status);

// DenseLu on any n (pf_large.cu)
int large_lu_factor(pf_context* ctx, int n, int batch, double* A, int64_t lda, int64_t strideA, int* piv,
                    double pivot_rel_tol, int flags, pf_status* status);
int large_lu_solve(pf_context* ctx, int n, int k, int batch, const double* LU, int64_t lda, int64_t strideLU,
                   const int* piv, double* R, int64_t ldr, int64_t strideR);

}  // namespace host
}  // namespace pf
