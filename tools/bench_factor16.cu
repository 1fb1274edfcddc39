// Microbenchmark: latency of the 16x16 register LU chain (one warp) used by small_eval.cu, with
// variants that remove one ingredient at a time. Prints cycles per pivot step.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
template <int V>
__global__ void k(double* out, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  double d[16];
  for (int c = 0; c < 16; ++c) d[c] = (lane == c ? 4.0 : 0.01 * (lane + c + 1));
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const double piv = __shfl_sync(FULL, d[m], m);
      double inv;
      if (V == 1) inv = 0.25; else if (V == 3 || V == 5) inv = 1.0 / piv; else inv = fast_rcp(piv);
      double u[16];
#pragma unroll
      for (int c = m + 1; c < 16; ++c) u[c] = (V == 2) ? d[c] : __shfl_sync(FULL, d[c], m);
      const bool below = lane > m;
      const double f = d[m] * inv;
      if (V >= 4) {
        if (below) {
          d[m] = f;
#pragma unroll
          for (int c = m + 1; c < 16; ++c) d[c] = fma(-f, u[c], d[c]);
        }
      } else {
        d[m] = below ? f : d[m];
#pragma unroll
        for (int c = m + 1; c < 16; ++c) d[c] = below ? fma(-f, u[c], d[c]) : d[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) d[c] = d[c] * 0.999 + (lane == c ? 3.0 : 0.0);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < 16; ++c) s += d[c];
  out[lane] = s;
  if (lane == 0) *cyc = t1 - t0;
}

// paired pivot steps (m, m+1): one shuffle of the 2x2 pivot block, rcp(a) and rcp(det) in
// parallel, lane m+1 updates its row (pointwise U), one shuffle of that row, the other rows apply
// both multipliers with 1/e' = a rcp(det)
__global__ void k_pair(double* out, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  double d[16];
  for (int c = 0; c < 16; ++c) d[c] = (lane == c ? 4.0 : 0.01 * (lane + c + 1));
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int m = 0; m < 16; m += 2) {
      const double a = __shfl_sync(FULL, d[m], m), b = __shfl_sync(FULL, d[m + 1], m);
      const double c_ = __shfl_sync(FULL, d[m], m + 1), e = __shfl_sync(FULL, d[m + 1], m + 1);
      const double ia = fast_rcp(a);
      const double idet = fast_rcp(fma(a, e, -(b * c_)));
      double um[16];
#pragma unroll
      for (int c = m + 2; c < 16; ++c) um[c] = __shfl_sync(FULL, d[c], m);
      if (lane == m + 1) {
        const double l1 = c_ * ia;
        d[m] = l1;
        d[m + 1] = fma(-l1, b, e);
#pragma unroll
        for (int c = m + 2; c < 16; ++c) d[c] = fma(-l1, um[c], d[c]);
      }
      double wm[16];
#pragma unroll
      for (int c = m + 2; c < 16; ++c) wm[c] = __shfl_sync(FULL, d[c], m + 1);
      if (lane > m + 1 && lane < 16) {
        const double f = d[m] * ia;
        const double f2 = fma(-f, b, d[m + 1]) * (a * idet);
        d[m] = f;
        d[m + 1] = f2;
#pragma unroll
        for (int c = m + 2; c < 16; ++c) d[c] = fma(-f2, wm[c], fma(-f, um[c], d[c]));
      }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) d[c] = d[c] * 0.999 + (lane == c ? 3.0 : 0.0);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < 16; ++c) s += d[c];
  out[lane] = s;
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 8);
  const char* names[] = {"current (shfl row, fast_rcp, select)", "no reciprocal", "no row shuffles", "IEEE div", "branch instead of select", "branch + IEEE div", "paired pivots (2x2 block, parallel rcp)"};
  double ref[32], got[32];
  for (int v = 0; v < 7; ++v) {
    for (int it = 0; it < 2; ++it) {
      switch (v) {
        case 0: k<0><<<1, 32>>>(o, c, 1000); break;
        case 1: k<1><<<1, 32>>>(o, c, 1000); break;
        case 2: k<2><<<1, 32>>>(o, c, 1000); break;
        case 3: k<3><<<1, 32>>>(o, c, 1000); break;
        case 4: k<4><<<1, 32>>>(o, c, 1000); break;
        case 5: k<5><<<1, 32>>>(o, c, 1000); break;
        case 6: k_pair<<<1, 32>>>(o, c, 1000); break;
      }
      cudaDeviceSynchronize();
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.1f cycles/step\n", names[v], h / 16000.0);
    if (v == 4) cudaMemcpy(ref, o, 256, cudaMemcpyDeviceToHost);
    if (v == 6) {
      cudaMemcpy(got, o, 256, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 16; ++i) mx = fmax(mx, fabs(got[i] - ref[i]) / fabs(ref[i]));
      printf("paired vs pointwise: max rel diff of the row sums %.3e\n", mx);
    }
  }
  return 0;
}
