// Shared device helpers for the parfrac B200 kernels (sm_100a).
//
// FP64 tensor work on sm_100a is warp-synchronous DMMA: `mma.sync.m8n8k4.f64` assembles to
// SASS DMMA.8x8x4 (tcgen05 has no kind::f64). Measured on this pool's B200: one DMMA per
// 16 cycles per SMSP (37.1 TFLOP/s chip-wide), 27-cycle dependent latency
// (profiles/r01_fp64_probe.jsonl).
//
// Fragment layout of m8n8k4 (row.col), g = lane >> 2, t = lane & 3:
//   A (8x4):  a = A[g][t]
//   B (4x8):  b = B[t][g]
//   C (8x8):  c0 = C[g][2t], c1 = C[g][2t+1]
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pf_b200.h"

namespace pf {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// Device-side status record, one per batch entry; mirrors pf_status (include/pf_b200.h).
struct DevStatus {
  int code;
  int shift_index;
  int column;
  int pad;
  double pivot_magnitude;
  double scale;
};

// Reference error ordinals (proj/core/include/parfrac/error.hpp:8-19), +1 so 0 = ok.
constexpr int kErrSingularShift = PF_ERR_SINGULAR_SHIFT;

}  // namespace pf
