// Microbenchmark: the DMMA GEMM's inner k-loop (gemm_tile.cuh, 64 x 64 x 16 tile, 4 warps of 32 x 32,
// four CTAs per SM) with the operands already in shared memory -- no global loads, no pipeline --
// against variants of the fragment loads. Prints TFLOP/s per variant.
//   V0: as gemm_tile: per k-step 4 A + 4 B LDS.64, 16 DMMA
//   V1: k-permuted A fragments: one LDS.128 gives a lane its A values for two DMMA k-sets
//       ({0,2,4,6} and {1,3,5,7} of an 8-wide k block), B from a k-pair-interleaved tile (LDS.128)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe_gemm_inner.cu -o tools/probe_gemm_inner.bin
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr int BM = 64, BN = 64, BK = 16, LA = BK + 4, LB = BN + 4, LB2 = BN + 4;  // LB2: double2 stride of the k-pair tile

template <int V>
__global__ void __launch_bounds__(128, 4) inner_kernel(double* out, int iters) {
  __shared__ __align__(16) double a[BM * LA];
  __shared__ __align__(16) double b[BK * LB2];
  for (int i = threadIdx.x; i < BM * LA; i += 128) a[i] = 1e-3 * (i % 7);
  for (int i = threadIdx.x; i < BK * LB2; i += 128) b[i] = 1e-3 * (i % 5);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = 32 * (warp >> 1), wn = 32 * (warp & 1);
  double acc[4][4][2] = {};
  for (int it = 0; it < iters; ++it) {
    if (V == 0) {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = a[(wm + 8 * mi + g) * LA + kk + t];
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) bf[nj] = b[(kk + t) * LB + wn + 8 * nj + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
      }
    } else {
      // b viewed as [BK/2][LB][2]: k-pairs interleaved
#pragma unroll
      for (int kk = 0; kk < BK; kk += 8) {
        double2 af[4], bf[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = *reinterpret_cast<const double2*>(&a[(wm + 8 * mi + g) * LA + kk + 2 * t]);
#pragma unroll
        for (int nj = 0; nj < 4; ++nj)
          bf[nj] = reinterpret_cast<const double2*>(b)[(kk / 2 + t) * LB2 + wn + 8 * nj + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma(acc[mi][nj], af[mi].x, bf[nj].x);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma(acc[mi][nj], af[mi].y, bf[nj].y);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) s += acc[mi][nj][0] + acc[mi][nj][1];
  if (s == 1234.5) out[0] = s;
}

template <int V>
double run(int sms) {
  double* d;
  cudaMalloc(&d, 64);
  const int iters = 4000, blocks = sms * 4;
  inner_kernel<V><<<blocks, 128>>>(d, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    inner_kernel<V><<<blocks, 128>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(d);
  const double flops = (double)blocks * 4 /*warps*/ * iters * (BK / 4) * 16 * 512.0;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"V0_tflops\": %.2f, \"V1_tflops\": %.2f}\n", run<0>(sms), run<1>(sms));
  return 0;
}
