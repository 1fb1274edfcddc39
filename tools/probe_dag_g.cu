// Microbenchmark: the DAG LU's G-task tile (128 x 128 output, K = 128 * steps, TMA ring) in a
// persistent kernel, 8 warps of 32 x 64 (1 CTA per SM, as lu_dag_kernel) vs the same tile by 16
// warps of 32 x 32 (a 512-thread CTA) -- does the DAG lose G efficiency to its warp count?
// Operands stay in L2 (one 1024^2 matrix per CTA group), results discarded.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2210_03714_b200/csrc \
//        tools/probe_dag_g.cu paper_2210_03714_b200/csrc/gemm_tma.cu paper_2210_03714_b200/csrc/misc.cu -o tools/probe_dag_g.bin -lcuda
#include <cstdio>
#include <vector>

#include "pf_common.cuh"
#include "pf_kernels.h"
#include "tma_util.cuh"

namespace pf {
constexpr int A_BYTES = 128 * 16 * 8, STAGE = 2 * A_BYTES, NS = 3;

template <int NWARPS>
__global__ void __launch_bounds__(NWARPS * 32, 1) g_probe(const __grid_constant__ DagMaps maps, int tasks, int steps,
                                                           double* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) unsigned long long bars[2 * NS];
  const unsigned fullb = su32(&bars[0]), emptyb = su32(&bars[NS]);
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int g = lane >> 2, t = lane & 3;
  constexpr int WN = NWARPS == 8 ? 64 : 32;  // warp tile 32 x WN
  constexpr int NJ = WN / 8;
  const int wm = 32 * (NWARPS == 8 ? (warp >> 1) : (warp >> 2)), wn = WN * (NWARPS == 8 ? (warp & 1) : (warp & 3));
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      mb_init(fullb + 8 * q, 1);
      mb_init(emptyb + 8 * q, NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const unsigned base = su32(ring);
  unsigned fills = 0;
  unsigned offA[4], offB[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int kt_ = 2 * (s & 1) + 8 * (s >> 1) + (t & 1) + 4 * (t >> 1);
    offA[s] = (unsigned)((wm + g) * 128 + ((((kt_ >> 1) ^ g) & 7) << 4) + ((kt_ & 1) << 3));
    offB[s] = (unsigned)(A_BYTES + (wn / 16) * 2048 + kt_ * 128 + ((((g >> 1) ^ (kt_ & 7)) & 7) << 4) + ((g & 1) << 3));
  }
  double total = 0.0;
  for (int task = blockIdx.x; task < tasks; task += gridDim.x) {
    const int i = task % 8, j = (task / 8) % 8;
    const int NK = 8 * steps;
    auto issue = [&](unsigned f, int kt) {
      const unsigned s = f % NS, sa = base + s * STAGE, sb = sa + A_BYTES, bar = fullb + 8 * s;
      if (f >= NS) mb_wait(emptyb + 8 * s, ((f / NS) - 1) & 1u);
      mb_expect(bar, STAGE);
      tma3(sa, &maps.a, 16 * kt % 1024, 128 * i, 0, bar);
#pragma unroll
      for (int q = 0; q < 8; ++q) tma3(sb + q * 2048, &maps.b, 128 * j + 16 * q, 16 * kt % 1024, 0, bar);
    };
    if (tid == 0)
      for (int kt = 0; kt < NS - 1 && kt < NK; ++kt) issue(fills + kt, kt);
    double acc[4][NJ][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
    for (int kt = 0; kt < NK; ++kt) {
      const unsigned f = fills + kt;
      if (tid == 0 && kt + NS - 1 < NK) issue(f + NS - 1, kt + NS - 1);
      mb_wait(fullb + 8 * (f % NS), (f / NS) & 1u);
      const unsigned char* sp = ring + (f % NS) * STAGE;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        double af[4], bf[NJ];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = *reinterpret_cast<const double*>(sp + offA[ks] + mi * 1024);
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
          bf[nj] = *reinterpret_cast<const double*>(sp + ((offB[ks] + (nj >> 1) * 2048) ^ ((nj & 1) << 6)));
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < NJ; ++nj) dmma(acc[mi][nj], af[mi], bf[nj]);
      }
      __syncwarp();
      if (lane == 0) mb_arrive(emptyb + 8 * (f % NS));
    }
    fills += NK;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) total += acc[mi][nj][0] + acc[mi][nj][1];
    __syncthreads();
  }
  if (total == 1234.5) sink[0] = total;
}
}  // namespace pf

int main() {
  const int n = 1024;
  double *M, *sink;
  cudaMalloc(&M, sizeof(double) * n * n);
  cudaMalloc(&sink, 64);
  std::vector<double> h((size_t)n * n, 1e-3);
  cudaMemcpy(M, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  pf::DagMaps maps;
  pf::make_tma_map(&maps.a, M, n, n, 1, n, n * n, 16, 128);
  pf::make_tma_map(&maps.b, M, n, n, 1, n, n * n, 16, 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = pf::NS * pf::STAGE + 2048;
  cudaFuncSetAttribute(pf::g_probe<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pf::g_probe<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int steps : {1, 4, 8}) {
    const int tasks = sms * 8;
    for (int w = 0; w < 2; ++w) {
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        if (w == 0)
          pf::g_probe<8><<<sms, 256, smem>>>(maps, tasks, steps, sink);
        else
          pf::g_probe<16><<<sms, 512, smem>>>(maps, tasks, steps, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      const double flops = (double)tasks * 2.0 * 128 * 128 * 128 * steps;
      printf("{\"warps\": %d, \"steps\": %d, \"ms\": %.3f, \"tflops\": %.2f, \"err\": \"%s\"}\n", w ? 16 : 8, steps, best,
             flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
