#pragma once
// Internal to the C++ host layer (not installed): the process-wide B200 context, device buffers,
// and the mapping of ABI status codes back to parfrac::Error with the reference's messages.
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
  Device() {
    if (pf_context_create(0, &ctx) != PF_OK)
      raise(Errc::BadArgument, "parfrac: no CUDA device (the B200 engine has no CPU fallback)");
  }
  ~Device() { pf_context_destroy(ctx); }
};

inline Device& device() {
  static Device d;
  return d;
}

class Buf {
 public:
  Buf(pf_context* ctx, size_t count) : ctx_(ctx) {
    if (pf_device_alloc(ctx, count * sizeof(double), &p_) != PF_OK) raise(Errc::BadArgument, "device allocation failed");
  }
  ~Buf() { pf_device_free(ctx_, p_); }
  double* d() const { return static_cast<double*>(p_); }
  int* i() const { return static_cast<int*>(p_); }
  void put(const double* h, size_t count) { check(pf_copy_to_device(ctx_, p_, h, count * sizeof(double))); }
  void get(double* h, size_t count) const { check(pf_copy_to_host(ctx_, h, p_, count * sizeof(double))); }
  static void check(int rc) {
    if (rc) raise(Errc::BadArgument, std::string("device transfer failed: ") + pf_error_string(rc));
  }

 private:
  pf_context* ctx_;
  void* p_ = nullptr;
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
      constant.push_back(to_double_nearest(s->constant));
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
