// FP64 pipe probe for B200 (sm_100a): DMMA.8x8x4 and DFMA throughput/latency.
// Used once per box to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_tput(double* out, int iters) {
  double acc[CHAINS][2];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_tput(double* out, int iters) {
  double acc[CHAINS];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], b, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int blocks, int threads, int iters, double flop_per_thread_iter) {
    kern<<<blocks, threads>>>(d, 10);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double flops = double(blocks) * threads * iters * flop_per_thread_iter;
    printf("{\"probe\":\"%s\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", name, blocks, threads, best,
           flops / best / 1e9);
  };
  // DMMA: one mma = 8*8*4 FMA = 512 flop per warp -> 16 flop per thread
  for (int warps : {4, 8, 16, 32}) {
    run("dmma_c8", dmma_tput<8>, sms, warps * 32, 20000, 8 * 16.0);
    run("dmma_c4", dmma_tput<4>, sms, warps * 32, 20000, 4 * 16.0);
  }
  run("dmma_c1_latency_1warp", dmma_tput<1>, 1, 32, 20000, 16.0);
  run("dmma_c2_1warp", dmma_tput<2>, 1, 32, 20000, 2 * 16.0);
  run("dmma_c8_1warp", dmma_tput<8>, 1, 32, 20000, 8 * 16.0);
  run("dmma_c8_4warp_1sm", dmma_tput<8>, 1, 128, 20000, 8 * 16.0);
  for (int warps : {8, 16, 32}) run("dfma_c8", dfma_tput<8>, sms, warps * 32, 20000, 8 * 2.0);
  run("dfma_c1_latency_1warp", dfma_tput<1>, 1, 32, 20000, 2.0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, clk);
  return 0;
}
