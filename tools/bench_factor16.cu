// Microbenchmark: latency of the 16x16 register LU chain (one warp) used by small_eval.cu, with
// variants that remove one ingredient at a time. Prints cycles per pivot step.
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
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 8);
  const char* names[] = {"current (shfl row, fast_rcp, select)", "no reciprocal", "no row shuffles", "IEEE div", "branch instead of select", "branch + IEEE div", "branch + rcp, 2 rows/lane"};
  for (int v = 0; v < 6; ++v) {
    for (int it = 0; it < 2; ++it) {
      switch (v) {
        case 0: k<0><<<1, 32>>>(o, c, 1000); break;
        case 1: k<1><<<1, 32>>>(o, c, 1000); break;
        case 2: k<2><<<1, 32>>>(o, c, 1000); break;
        case 3: k<3><<<1, 32>>>(o, c, 1000); break;
        case 4: k<4><<<1, 32>>>(o, c, 1000); break;
        case 5: k<5><<<1, 32>>>(o, c, 1000); break;
      }
      cudaDeviceSynchronize();
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.1f cycles/step\n", names[v], h / 16000.0);
  }
  return 0;
}
