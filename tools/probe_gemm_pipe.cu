// Microbenchmark: where the DMMA GEMM (gemm.cu, 64 x 64 x 16 tiles, 4 CTAs per SM) loses against the
// inner-loop rate (tools/probe_gemm_inner.cu: 37.0 TF/s = the DMMA probe). Runs the production
// kernel (the same translation unit) on m = n = k = 4096:
//   real  : distinct A, B (the batched GEMM as used)
//   hot   : lda = ldb = 0 -- every row of A / every k-row of B is the same 32 KB row, so every
//           operand copy hits L2 (pipeline + instruction overhead only, no memory-system effects)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/probe_gemm_pipe.cu -o tools/probe_gemm_pipe.bin
#include <cstdio>
#include <vector>

#include "../paper_2210_03714_b200/csrc/gemm.cu"

int main() {
  const int n = 4096;
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(double) * n * n);
  cudaMalloc(&B, sizeof(double) * n * n);
  cudaMalloc(&C, sizeof(double) * n * n);
  std::vector<double> h((size_t)n * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * (double)(i % 97);
  cudaMemcpy(A, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    pf::GemmParams p{};
    p.m = p.n = p.k = n;
    p.batch = 1;
    p.alpha = 1.0;
    p.A = A;
    p.B = B;
    p.C = C;
    p.lda = mode ? 0 : n;
    p.ldb = mode ? 0 : n;
    p.ldc = n;
    pf::launch_gemm(p, 0);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      pf::launch_gemm(p, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("{\"mode\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f, \"err\": \"%s\"}\n", mode ? "hot" : "real", best,
           2.0 * n * (double)n * n / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
