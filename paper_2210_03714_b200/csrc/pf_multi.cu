// Multi-device evaluation of ONE matrix through the C ABI (SURVEY §8(b) pf_eval_multi_gpu, §8(e)):
// the s resolvents of eval_dense are independent (dense.cpp:202, one worker per shift,
// worker_pool.hpp:16-44), so the shifts are partitioned over the context's devices, every device
// evaluates its share on its own stream from its own host thread, and ONE exchange over NCCL
// brings the weighted terms to the root before the squaring / doubling recurrence.
//
// Partition. Units are the (c, -c) pairs of a residual-form method (merged into one solve of
// I - c^2 B^2 on a device) when there are at least as many pairs as devices, else single shifts
// (R8 on 8 GPUs: one shift per GPU). Unit u goes to device u mod G; zero shifts (the plain form's
// w I term) and a_0 / the polynomial part go to the root.
//
// Exchange.
//   fast:          every device sums its own terms (pair merging allowed); ncclReduce(sum) to the
//                  root. The sum order over devices is NCCL's: results agree to rounding for any G.
//   deterministic: every device evaluates each owned shift on its own (PF_FLAG_PER_SHIFT); the
//                  root receives every weighted term (grouped ncclSend / ncclRecv, n^2 doubles per
//                  shift and weight set, root only -- no all-gather), sums them in ascending shift
//                  index (pf_ordered_sum: acc = ((T_0 + T_1) + T_2) + ..., dense.cpp:245-246), then
//                  adds the polynomial part as poly_part does (:176-189). Bit-identical for any G
//                  and any device order: the reference's bit-identical-workers contract.
// NCCL is resolved from libnccl.so.2 at run time (dlopen), so the engine has no link-time NCCL
// dependency. A device list with repeated ids (several ranks on one GPU: tests) uses peer copies
// instead of NCCL with the same partition, terms and reduction order.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "pf_host.h"

namespace pf {

__global__ void add_poly_kernel(double* E, int64_t lde, int n, double constant, double d1, const double* B,
                                double d2, const double* B2) {
  // E = E + poly, poly = (0 + constant) I [+ d1 B] [+ d2 B^2]: poly_part's operation order
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx % n);
    double pv = (r == c) ? __dadd_rn(0.0, constant) : 0.0;
    if (B) pv = __dadd_rn(pv, __dmul_rn(d1, B[idx]));
    if (B2) pv = __dadd_rn(pv, __dmul_rn(d2, B2[idx]));
    double* e = E + (int64_t)r * lde + c;
    *e = __dadd_rn(*e, pv);
  }
}

__global__ void scale_pow2_kernel(const double* A, int64_t lda, int n, const int* dJ, double* B) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx % n);
    B[idx] = ldexp(A[(int64_t)r * lda + c], -(dJ ? *dJ : 0));
  }
}

namespace host {
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.Reduce = reinterpret_cast<decltype(api.Reduce)>(dlsym(h, "ncclReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
    api.ok = api.CommInitAll && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Broadcast && api.Reduce &&
             api.Send && api.Recv;
  });
  return api;
}

constexpr int kWsMultiA = 40;      // member copy of A (n x n)
constexpr int kWsMultiOut = 41;    // member partial / per-shift terms
constexpr int kWsMultiJ = 42;      // member j
constexpr int kWsMultiRecv = 43;   // root: received partials / terms
constexpr int kWsMultiB = 44;      // root: B and B^2 for the hybrid polynomial part
constexpr int kWsMultiE = 45;      // root: reduced E (and Phi) before the recurrence

struct Unit {
  std::vector<int> shifts;  // global shift indices, ascending
};

// pairs (residual form, adjacent c, -c) or single nonzero shifts; zero shifts separately
std::vector<Unit> make_units(const pf_method* m, int G, bool per_shift) {
  std::vector<Unit> pairs, singles;
  for (int i = 0; i < m->n_terms; ++i) {
    const double c = m->shifts[i];
    if (c == 0.0) continue;
    if (m->form == PF_FORM_RESIDUAL && !m->has_poly && i + 1 < m->n_terms && m->shifts[i + 1] == -c) {
      pairs.push_back(Unit{{i, i + 1}});
      singles.push_back(Unit{{i}});
      singles.push_back(Unit{{i + 1}});
      ++i;
    } else {
      pairs.push_back(Unit{{i}});
      singles.push_back(Unit{{i}});
    }
  }
  if (per_shift || (int)pairs.size() < G) return singles;
  return pairs;
}

struct MemberWork {
  pf_context* ctx = nullptr;
  std::vector<int> owned;  // global shift indices owned (ascending), zero shifts included on root
  bool root = false;
  int rc = PF_OK;
  pf_status st{};
  double* A = nullptr;     // member copy of A (n x n, ld n)
  double* out = nullptr;   // fast: partial (n_sets x n^2); deterministic: one slot per owned shift
  int* dJ = nullptr;
};

// sub-method of the owned shifts: weights per set, a_0 / poly on the root only
struct SubMethod {
  std::vector<double> shifts, weights, poly, constant;
  pf_method m{};
  SubMethod(const pf_method* base, const std::vector<int>& idx, bool root) {
    const int ns = base->n_sets;
    for (int i : idx) shifts.push_back(base->shifts[i]);
    for (int s = 0; s < ns; ++s)
      for (int i : idx) weights.push_back(base->weights[s * base->n_terms + i]);
    for (int s = 0; s < ns; ++s) {
      for (int k = 0; k < 3; ++k) poly.push_back(root && base->has_poly ? base->poly[3 * s + k] : 0.0);
      constant.push_back(root && base->constant ? base->constant[s] : 0.0);
    }
    m.n_terms = (int)shifts.size();
    m.shifts = shifts.data();
    m.n_sets = ns;
    m.weights = weights.data();
    m.has_poly = root && base->has_poly ? 1 : 0;
    m.poly = poly.data();
    m.constant = constant.data();
    m.form = base->form;
  }
};

int eval_member(MemberWork& w, const pf_method* m, double theta, int recurrence, int n, bool deterministic,
                int flags) {
  pf_context* ctx = w.ctx;
  DeviceGuard guard(ctx);
  const int64_t nn = (int64_t)n * n;
  const int ns = m->n_sets;
  const int f = flags & ~(PF_FLAG_ASYNC | PF_FLAG_REFERENCE_ORDER);
  const int* dJin = recurrence == PF_REC_NONE ? nullptr : w.dJ;
  auto run = [&](const pf_method* sub, double* out0, pf_status* st, int ff) {
    double* outs[2] = {out0, ns > 1 ? out0 + nn : nullptr};
    if (recurrence == PF_REC_NONE) return pf_eval_dense_batched(ctx, sub, n, 1, w.A, n, nn, outs, n, nn, ff, st);
    return pf_eval_scaled_batched(ctx, sub, theta, n, 1, w.A, n, nn, dJin, nullptr, outs, n, nn, ff, st);
  };
  if (!deterministic) {
    if (w.owned.empty() && !w.root) {
      cudaMemsetAsync(w.out, 0, sizeof(double) * nn * ns, ctx->stream);
      return cuda_fail(cudaStreamSynchronize(ctx->stream));
    }
    SubMethod sub(m, w.owned, w.root);
    const int rc = run(&sub.m, w.out, &w.st, f);
    if (rc && w.st.shift_index > 0) w.st.shift_index = w.owned[w.st.shift_index - 1] + 1;
    return rc;
  }
  // one weighted term per owned shift: T_i = 0 + w_i X_i (a one-term method, no constant)
  for (size_t q = 0; q < w.owned.size(); ++q) {
    SubMethod sub(m, {w.owned[q]}, false);
    const int rc = run(&sub.m, w.out + (int64_t)q * ns * nn, &w.st, f | PF_FLAG_PER_SHIFT);
    if (rc) {
      w.st.shift_index = w.owned[q] + 1;
      return rc;
    }
  }
  return PF_OK;
}

}  // namespace
}  // namespace host
}  // namespace pf

struct pf_group {
  std::vector<pf_context*> members;  // members[0] is the root context itself
  std::vector<cudaStream_t> own_streams;
  std::vector<ncclComm_t> comms;     // empty: peer-copy exchange (repeated devices)
};

using namespace pf::host;

extern "C" {

int pf_context_create_multi(int n_devices, const int* device_ids, pf_context** out) {
  if (!out || n_devices < 1 || !device_ids) return PF_ERR_BAD_ARGUMENT;
  *out = nullptr;
  pf_context* root = nullptr;
  int rc = pf_context_create(device_ids[0], &root);
  if (rc) return rc;
  auto* g = new pf_group();
  g->members.push_back(root);
  for (int i = 1; i < n_devices && !rc; ++i) {
    pf_context* c = nullptr;
    rc = pf_context_create(device_ids[i], &c);
    if (!rc) g->members.push_back(c);
  }
  // one non-blocking stream per member: the members run concurrently (own host threads)
  for (pf_context* c : g->members) {
    if (rc) break;
    DeviceGuard guard(c);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      rc = PF_ERR_CUDA;
      break;
    }
    g->own_streams.push_back(s);
    c->stream = s;
  }
  std::vector<int> ids(device_ids, device_ids + n_devices);
  std::vector<int> sorted = ids;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (!rc && distinct && nccl().ok) {
    g->comms.resize(n_devices);
    DeviceGuard guard(root);
    if (nccl().CommInitAll(g->comms.data(), n_devices, ids.data()) != ncclSuccess) {
      g->comms.clear();
      rc = distinct && n_devices > 1 ? PF_ERR_CUDA : PF_OK;
    }
  }
  root->group = g;
  if (rc) {
    pf_context_destroy(root);
    return rc;
  }
  *out = root;
  return PF_OK;
}

int pf_context_device_count(pf_context* ctx) {
  if (!ctx) return 0;
  return ctx->group ? (int)ctx->group->members.size() : 1;
}

int pf_context_uses_nccl(pf_context* ctx) { return ctx && ctx->group && !ctx->group->comms.empty() ? 1 : 0; }

int pf_eval_multi_gpu(pf_context* ctx, const pf_method* m, double theta, int recurrence, int n, const double* dA,
                      int64_t lda, double* dOut0, double* dOut1, int64_t ldo, int deterministic, int flags,
                      int* j_out, pf_status* status) {
  DeviceGuard device_guard(ctx);
  if (status) std::memset(status, 0, sizeof(*status));
  pf::SmallParams probe{};
  if (!ctx || !fill_method(m, probe) || n < 1 || lda < n || ldo < n || !dA || !dOut0 ||
      (m->n_sets > 1 && !dOut1) || recurrence < PF_REC_NONE || recurrence > PF_REC_EXP_PHI1 ||
      (recurrence != PF_REC_NONE && !(theta > 0)) || (recurrence == PF_REC_EXP_PHI1 && m->n_sets < 2) ||
      (flags & PF_FLAG_REFERENCE_ORDER))
    return bad(status);
  std::vector<pf_context*> members = ctx->group ? ctx->group->members : std::vector<pf_context*>{ctx};
  const int G = (int)members.size();
  const bool use_nccl = ctx->group && !ctx->group->comms.empty();
  const int64_t nn = (int64_t)n * n;
  const int ns = recurrence == PF_REC_EXP ? 1 : m->n_sets;
  pf_method mm = *m;
  mm.n_sets = ns;
  const bool det = deterministic != 0;

  // ---- partition
  std::vector<MemberWork> work(G);
  const std::vector<Unit> units = make_units(&mm, G, det || (flags & PF_FLAG_PER_SHIFT));
  for (int gi = 0; gi < G; ++gi) {
    work[gi].ctx = members[gi];
    work[gi].root = gi == 0;
  }
  for (size_t u = 0; u < units.size(); ++u)
    for (int i : units[u].shifts) work[u % G].owned.push_back(i);
  if (mm.form == PF_FORM_PLAIN)
    for (int i = 0; i < mm.n_terms; ++i)
      if (mm.shifts[i] == 0.0) work[0].owned.push_back(i);  // the w I term
  for (auto& w : work) std::sort(w.owned.begin(), w.owned.end());

  // ---- buffers, A on every member, j on the root
  for (int gi = 0; gi < G; ++gi) {
    MemberWork& w = work[gi];
    DeviceGuard guard(w.ctx);
    const size_t slots = det ? std::max<size_t>(w.owned.size(), 1) : 1;
    w.A = static_cast<double*>(workspace(w.ctx, kWsMultiA, sizeof(double) * nn));
    w.out = static_cast<double*>(workspace(w.ctx, kWsMultiOut, sizeof(double) * nn * ns * slots));
    w.dJ = static_cast<int*>(workspace(w.ctx, kWsMultiJ, sizeof(int)));
    if (!w.A || !w.out || !w.dJ) return PF_ERR_CUDA;
  }
  pf_context* root = members[0];
  cudaMemcpy2DAsync(work[0].A, sizeof(double) * n, dA, sizeof(double) * lda, sizeof(double) * n, n,
                    cudaMemcpyDeviceToDevice, root->stream);
  int j = 0;
  if (recurrence != PF_REC_NONE) {
    int rc = pf_squarings_batched(root, n, 1, work[0].A, n, nn, theta, work[0].dJ);
    if (rc) return rc;
    if (cudaMemcpyAsync(&j, work[0].dJ, sizeof(int), cudaMemcpyDeviceToHost, root->stream) != cudaSuccess ||
        cudaStreamSynchronize(root->stream) != cudaSuccess)
      return PF_ERR_CUDA;
  }
  if (cudaStreamSynchronize(root->stream) != cudaSuccess) return PF_ERR_CUDA;
  if (G > 1) {
    if (use_nccl) {
      nccl().GroupStart();
      for (int gi = 0; gi < G; ++gi)
        nccl().Broadcast(work[0].A, work[gi].A, (size_t)nn, ncclDouble, 0, ctx->group->comms[gi], members[gi]->stream);
      if (nccl().GroupEnd() != ncclSuccess) return PF_ERR_CUDA;
    } else {
      for (int gi = 1; gi < G; ++gi)
        cudaMemcpyPeerAsync(work[gi].A, members[gi]->device, work[0].A, root->device, sizeof(double) * nn,
                            members[gi]->stream);
    }
    for (int gi = 1; gi < G; ++gi) {
      DeviceGuard guard(members[gi]);
      cudaMemcpyAsync(work[gi].dJ, &j, sizeof(int), cudaMemcpyHostToDevice, members[gi]->stream);
      if (cudaStreamSynchronize(members[gi]->stream) != cudaSuccess) return PF_ERR_CUDA;
    }
  }

  // ---- the s resolvents, one host thread per device
  {
    std::vector<std::thread> th;
    for (int gi = 1; gi < G; ++gi)
      th.emplace_back([&, gi] { work[gi].rc = eval_member(work[gi], &mm, theta, recurrence, n, det, flags); });
    work[0].rc = eval_member(work[0], &mm, theta, recurrence, n, det, flags);
    for (auto& t : th) t.join();
  }
  int first = -1;
  for (int gi = 0; gi < G; ++gi)
    if (work[gi].rc && (first < 0 || work[gi].st.shift_index < work[first].st.shift_index)) first = gi;
  if (first >= 0) {
    if (status) {
      *status = work[first].st;
      status->code = work[first].rc;
      status->batch_index = 0;
    }
    return work[first].rc;
  }

  // ---- the one exchange
  double* outs[2] = {dOut0, ns > 1 ? dOut1 : nullptr};
  double* E = static_cast<double*>(workspace(root, kWsMultiE, sizeof(double) * nn * 2));
  if (!E) return PF_ERR_CUDA;
  double* P = ns > 1 ? E + nn : nullptr;
  double* res[2] = {E, P};
  if (!det) {
    double* red = G > 1 ? static_cast<double*>(workspace(root, kWsMultiRecv, sizeof(double) * nn * ns * G)) : nullptr;
    if (G > 1 && !red) return PF_ERR_CUDA;
    if (G == 1) {
      for (int s = 0; s < ns; ++s)
        cudaMemcpyAsync(res[s], work[0].out + s * nn, sizeof(double) * nn, cudaMemcpyDeviceToDevice, root->stream);
    } else if (use_nccl) {
      nccl().GroupStart();
      for (int gi = 0; gi < G; ++gi)
        nccl().Reduce(work[gi].out, gi == 0 ? red : nullptr, (size_t)(nn * ns), ncclDouble, ncclSum, 0,
                      ctx->group->comms[gi], members[gi]->stream);
      if (nccl().GroupEnd() != ncclSuccess) return PF_ERR_CUDA;
      for (int s = 0; s < ns; ++s)
        cudaMemcpyAsync(res[s], red + s * nn, sizeof(double) * nn, cudaMemcpyDeviceToDevice, root->stream);
    } else {  // peer copies, summed in device order
      for (int gi = 0; gi < G; ++gi)
        cudaMemcpyPeerAsync(red + (int64_t)gi * ns * nn, root->device, work[gi].out, members[gi]->device,
                            sizeof(double) * nn * ns, root->stream);
      for (int s = 0; s < ns; ++s) {
        std::vector<const double*> t(G);
        for (int gi = 0; gi < G; ++gi) t[gi] = red + (int64_t)gi * ns * nn + s * nn;
        const int rc = pf_ordered_sum(root, G, t.data(), nn, res[s]);
        if (rc) return rc;
      }
    }
  } else {
    // every weighted term to the root, ascending shift index
    std::vector<int> owner(mm.n_terms, -1), slot(mm.n_terms, -1);
    for (int gi = 0; gi < G; ++gi)
      for (size_t q = 0; q < work[gi].owned.size(); ++q) {
        owner[work[gi].owned[q]] = gi;
        slot[work[gi].owned[q]] = (int)q;
      }
    std::vector<int> order;
    for (int i = 0; i < mm.n_terms; ++i)
      if (owner[i] >= 0) order.push_back(i);
    const int T = (int)order.size();
    double* recv = static_cast<double*>(workspace(root, kWsMultiRecv, sizeof(double) * nn * ns * std::max(T, 1)));
    if (!recv) return PF_ERR_CUDA;
    if (use_nccl && G > 1) {
      nccl().GroupStart();
      for (int t = 0; t < T; ++t) {
        const int i = order[t], gi = owner[i];
        const double* src = work[gi].out + (int64_t)slot[i] * ns * nn;
        if (gi == 0) {
          cudaMemcpyAsync(recv + (int64_t)t * ns * nn, src, sizeof(double) * nn * ns, cudaMemcpyDeviceToDevice,
                          root->stream);
        } else {
          nccl().Send(src, (size_t)(nn * ns), ncclDouble, 0, ctx->group->comms[gi], members[gi]->stream);
          nccl().Recv(recv + (int64_t)t * ns * nn, (size_t)(nn * ns), ncclDouble, gi, ctx->group->comms[0],
                      root->stream);
        }
      }
      if (nccl().GroupEnd() != ncclSuccess) return PF_ERR_CUDA;
    } else {
      for (int t = 0; t < T; ++t) {
        const int i = order[t], gi = owner[i];
        cudaMemcpyPeerAsync(recv + (int64_t)t * ns * nn, root->device, work[gi].out + (int64_t)slot[i] * ns * nn,
                            members[gi]->device, sizeof(double) * nn * ns, root->stream);
      }
    }
    for (int s = 0; s < ns; ++s) {
      if (T == 0) {
        cudaMemsetAsync(res[s], 0, sizeof(double) * nn, root->stream);
        continue;
      }
      std::vector<const double*> t(T);
      for (int q = 0; q < T; ++q) t[q] = recv + (int64_t)q * ns * nn + s * nn;
      const int rc = pf_ordered_sum(root, T, t.data(), nn, res[s]);
      if (rc) return rc;
    }
    // poly_part: residual a_0 I (+ hybrid d1 B + d2 B^2), or the plain hybrid's d0 I + d1 B + d2 B^2
    const bool need_poly = mm.form == PF_FORM_RESIDUAL || mm.has_poly;
    if (need_poly) {
      double* B = nullptr;
      double* B2 = nullptr;
      if (mm.has_poly) {
        B = static_cast<double*>(workspace(root, kWsMultiB, sizeof(double) * nn * 2));
        if (!B) return PF_ERR_CUDA;
        B2 = B + nn;
        pf::scale_pow2_kernel<<<(unsigned)std::min<int64_t>((nn + 255) / 256, 4736), 256, 0, root->stream>>>(
            work[0].A, n, n, recurrence == PF_REC_NONE ? nullptr : work[0].dJ, B);
        gemm(root, n, n, n, 1, 1.0, B, n, nn, B, n, nn, 0.0, B2, n, nn, 0.0);
        root->launches++;
      }
      for (int s = 0; s < ns; ++s) {
        const double constant = mm.form == PF_FORM_RESIDUAL ? mm.constant[s] : mm.poly[3 * s];
        const double d1 = mm.has_poly ? mm.poly[3 * s + 1] : 0.0, d2 = mm.has_poly ? mm.poly[3 * s + 2] : 0.0;
        pf::add_poly_kernel<<<(unsigned)std::min<int64_t>((nn + 255) / 256, 4736), 256, 0, root->stream>>>(
            res[s], n, n, constant, d1, mm.has_poly ? B : nullptr, d2, (mm.has_poly && d2 != 0.0) ? B2 : nullptr);
        root->launches++;
      }
    }
  }
  // every member's stream must be done before its buffers are reused
  for (int gi = 0; gi < G; ++gi) {
    DeviceGuard guard(members[gi]);
    if (cudaStreamSynchronize(members[gi]->stream) != cudaSuccess) return PF_ERR_CUDA;
  }

  // ---- the recurrence on the root
  int rc = PF_OK;
  if (recurrence == PF_REC_EXP)
    rc = pf_square_chain(root, n, 1, work[0].dJ, E);
  else if (recurrence == PF_REC_EXP_PHI1)
    rc = pf_phi1_doubling(root, n, 1, work[0].dJ, E, P);
  if (rc) return rc;
  for (int s = 0; s < ns; ++s)
    cudaMemcpy2DAsync(outs[s], sizeof(double) * ldo, res[s], sizeof(double) * n, sizeof(double) * n, n,
                      cudaMemcpyDeviceToDevice, root->stream);
  if (j_out) *j_out = j;
  return collect_status(root, 0, flags & ~PF_FLAG_ASYNC, nullptr);
}

}  // extern "C"

namespace pf {
namespace host {

void group_destroy(pf_context* root) {
  pf_group* g = root->group;
  if (!g) return;
  root->group = nullptr;
  for (size_t i = 0; i < g->comms.size(); ++i)
    if (g->comms[i]) nccl().CommDestroy(g->comms[i]);
  for (size_t i = 0; i < g->members.size(); ++i) {
    pf_context* c = g->members[i];
    {
      DeviceGuard guard(c);
      if (i < g->own_streams.size()) {
        cudaStreamSynchronize(g->own_streams[i]);
        cudaStreamDestroy(g->own_streams[i]);
      }
    }
    c->stream = nullptr;
    if (i > 0) pf_context_destroy(c);
  }
  delete g;
}

}  // namespace host
}  // namespace pf
