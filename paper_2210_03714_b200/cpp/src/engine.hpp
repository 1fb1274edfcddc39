#pragma once
// Internal to the C++ host layer (not installed): the process-wide B200 context, device buffers,
// and the mapping of ABI status codes back to parfrac::Error with the reference's messages.
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "parfrac/error.hpp"
#include "parfrac/methods.hpp"
#include "pf_b200.h"

namespace parfrac {
namespace engine {

// Process-wide device context; the ABI context is used by one host thread at a time.
struct Device {
  std::mutex mu;
  pf_context* ctx = nullptr;
  // device buffers are recycled (size classes of powers of two): a call does not pay cudaMalloc
  std::multimap<size_t, void*> pool;
  Device() {
    if (pf_context_create(0, &ctx) != PF_OK)
      raise(Errc::BadArgument, "parfrac: no CUDA device (the B200 engine has no CPU fallback)");
  }
  ~Device() {
    for (auto& kv : pool) pf_device_free(ctx, kv.second);
    pf_context_destroy(ctx);
  }
};

inline Device& device() {
  static Device d;
  return d;
}

// Multi-device contexts for EvalOptions::devices / device_ids, one per device list, process-wide.
struct MultiDevices {
  std::mutex mu;
  std::map<std::vector<int>, pf_context*> ctxs;
  ~MultiDevices() {
    for (auto& kv : ctxs) pf_context_destroy(kv.second);
  }
  pf_context* get(const std::vector<int>& ids) {
    auto it = ctxs.find(ids);
    if (it != ctxs.end()) return it->second;
    pf_context* c = nullptr;
    if (pf_context_create_multi(int(ids.size()), ids.data(), &c) != PF_OK)
      raise(Errc::BadArgument, "parfrac: cannot create a context over the requested devices");
    ctxs[ids] = c;
    return c;
  }
};

inline MultiDevices& multi_devices() {
  static MultiDevices m;
  return m;
}

// A device buffer of `count` doubles from the pool of `dev` (caller holds dev.mu for its lifetime).
class Buf {
 public:
  Buf(Device& dev, size_t count) : dev_(&dev), ctx_(dev.ctx) {
    size_t bytes = 256;
    while (bytes < count * sizeof(double)) bytes <<= 1;
    bytes_ = bytes;
    auto it = dev.pool.find(bytes);
    if (it != dev.pool.end()) {
      p_ = it->second;
      dev.pool.erase(it);
    } else if (pf_device_alloc(ctx_, bytes, &p_) != PF_OK) {
      raise(Errc::BadArgument, "device allocation failed");
    }
  }
  // a buffer owned outside the pool (long-lived objects: DenseLu factors, operators)
  Buf(pf_context* ctx, size_t count) : ctx_(ctx) {
    if (pf_device_alloc(ctx, std::max<size_t>(count, 1) * sizeof(double), &p_) != PF_OK)
      raise(Errc::BadArgument, "device allocation failed");
  }
  ~Buf() {
    if (!p_) return;
    if (dev_)
      dev_->pool.emplace(bytes_, p_);
    else
      pf_device_free(ctx_, p_);
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  double* d() const { return static_cast<double*>(p_); }
  int* i() const { return static_cast<int*>(p_); }
  void put(const double* h, size_t count) { check(pf_copy_to_device(ctx_, p_, h, count * sizeof(double))); }
  void get(double* h, size_t count) const { check(pf_copy_to_host(ctx_, h, p_, count * sizeof(double))); }
  static void check(int rc) {
    if (rc) raise(Errc::BadArgument, std::string("device transfer failed: ") + pf_error_string(rc));
  }

 private:
  Device* dev_ = nullptr;
  pf_context* ctx_;
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

inline Errc errc_of(int rc) { return rc >= 1 && rc <= 10 ? static_cast<Errc>(rc - 1) : Errc::BadArgument; }

[[noreturn]] inline void rethrow(int rc, const pf_status& st, bool with_shift) {
  const Errc code = errc_of(rc);
  if (code == Errc::ZeroPivot) {  // thomas_solve / pentadiag_solve (action.cpp:104,113,185, :291)
    std::string msg = "zero pivot at row " + std::to_string(st.column);
    if (with_shift && st.shift_index > 0) msg = "shift " + std::to_string(st.shift_index) + ": " + msg;
    raise(code, msg);
  }
  if (code == Errc::SingularShift) {
    std::string msg = "singular system: pivot magnitude " + format_sig17(st.pivot_magnitude) + " at column " +
                      std::to_string(st.column) + " (scale " + format_sig17(st.scale) + ")";
    if (with_shift && st.shift_index > 0) msg = "shift " + std::to_string(st.shift_index) + ": " + msg;
    raise(code, msg);
  }
  raise(code, std::string("B200 engine: ") + pf_error_string(rc));
}

struct Packed {
  std::vector<double> shifts, weights, poly, constant;
  pf_method m{};
  Packed(const std::vector<const FractionMethod*>& sets, EvalForm form) {
    const FractionMethod& base = *sets[0];
    for (const auto& c : base.shifts) shifts.push_back(to_double_nearest(c));
    bool has_poly = false;
    for (auto* s : sets) {
      for (const auto& w : s->weights) weights.push_back(to_double_nearest(w));
      has_poly |= s->poly.size() == 3;
    }
    for (auto* s : sets) {
      for (int k = 0; k < 3; ++k) poly.push_back(s->poly.size() == 3 ? to_double_nearest(s->poly[k]) : 0.0);
      constant.push_back(to_double_nearest(s->constant_term()));
    }
    m.n_terms = int(shifts.size());
    m.shifts = shifts.data();
    m.n_sets = int(sets.size());
    m.weights = weights.data();
    m.has_poly = has_poly ? 1 : 0;
    m.poly = poly.data();
    m.constant = constant.data();
    m.form = form == EvalForm::Residual ? PF_FORM_RESIDUAL : PF_FORM_PLAIN;
  }
};

}  // namespace engine
}  // namespace parfrac
