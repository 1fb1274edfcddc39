// Microbenchmark: the certified block LU of the small kernel (small_eval.cu lu_block) in
// isolation, 1 CTA per SM, against ablations and the alternative schedules kept in
// tools/lu_variants.cuh. Prints SM cycles per 128x128 LU (thread 0 clock64, mean over CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/bench_lu.cu -o tools/bench_lu.bin
//
// Measured on B200 (cycles per LU): production 48.1k; its lead chain alone (8 factors + schur)
// 23.2k, substitution panels alone 15.6k, trailing alone 17.4k. Alternatives (all slower):
// DMMA panels from two-warp triangular inverses 48.1k; lead factors + inverts (column sweeps)
// 51.1k; lead factor_invert_block (row sweeps by SHFL) 57.7k; factor with the pivot row broadcast
// through shared memory 3.5k per block vs 2.5k (the per-pivot chain is latency-bound: SHFL 26,
// MUFU.RCP64H 18, DFMA 8 cycles -- tools/probe_latency.cu).
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2210_03714_b200/csrc/small_eval.cu"
#include "lu_variants.cuh"

namespace pf {
namespace {

// Production schedule with knobs. V bits: 1 = no lead factor, 2 = no trailing update,
// 4 = no panels (and no final inverses), 8 = no lead schur
template <int V>
__device__ void lu_head(Smem& sm) {
  const int warp = warp_id();
  const bool lead = warp == NW - 1;
  if (lead && !(V & 1)) factor_diag_block(sm, 0);
  __syncthreads();
  for (int k0 = 0; k0 < N; k0 += NB) {
    const int rest = N - k0 - NB;
    if (rest == 0) break;
    if (!(V & 4)) {
      if (threadIdx.x < rest) {
        const int row = k0 + NB + threadIdx.x;
        double x[NB], rinv[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          x[c] = sm.S[row * LS + k0 + c];
          rinv[c] = fast_rcp(sm.S[(k0 + c) * LS + k0 + c]);
        }
#pragma unroll
        for (int m = 0; m < NB; ++m) {
          x[m] = x[m] * rinv[m];
#pragma unroll
          for (int c = m + 1; c < NB; ++c) x[c] = fma(-x[m], sm.S[(k0 + m) * LS + k0 + c], x[c]);
        }
#pragma unroll
        for (int c = NB - 1; c > 0; --c)
#pragma unroll
          for (int m = 0; m < c; ++m) x[m] = fma(-x[c], sm.S[(k0 + c) * LS + k0 + m], x[m]);
#pragma unroll
        for (int c = 0; c < NB; c += 2)
          *reinterpret_cast<double2*>(&sm.S[row * LS + k0 + c]) = make_double2(x[c], x[c + 1]);
      }
      __syncthreads();
    }
    const int nbk = rest / NB;
    if (lead) {
      if (!(V & 8)) schur_block(sm, k0, k0 + NB, k0 + NB);
      __syncwarp();
      if (!(V & 1)) factor_diag_block(sm, k0 + NB);
    } else if (!(V & 2)) {
      if (V & 16) {  // keep the lead's SMSP (warps 3, 7, 11) free of trailing work
        if ((warp & 3) != 3) {
          const int w = (warp >> 2) * 3 + (warp & 3);
          for (int blk = w + 1; blk < nbk * nbk; blk += 12)
            schur_block(sm, k0, k0 + NB + NB * (blk / nbk), k0 + NB + NB * (blk % nbk));
        }
      } else {
        for (int blk = warp + 1; blk < nbk * nbk; blk += NW - 1)
          schur_block(sm, k0, k0 + NB + NB * (blk / nbk), k0 + NB + NB * (blk % nbk));
      }
    }
    __syncthreads();
  }
  if (!(V & 4)) {
    invert_all_diag_blocks(sm);
    diag_inverse_products(sm);
  }
}

// DMMA-panel schedules. F selects the lead's chain step: 0 = factor_diag_block then two warps
// invert in the panel phase; 1 = factor_invert_block on the lead; 2 = factor_diag_block_sm then two
// warps invert.
__device__ __forceinline__ void tri_inverse_2warps(Smem& sm, LuExtra& ex, int k0, bool upper) {
  const int lane = lane_id();
  const int l = lane & 15;
  double x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) x[i] = (i == l) ? 1.0 : 0.0;
  if (upper) {
#pragma unroll
    for (int m = NB - 1; m >= 0; --m) {
      x[m] = x[m] * fast_rcp(sm.S[(k0 + m) * LS + k0 + m]);
#pragma unroll
      for (int i = 0; i < m; ++i) x[i] = fma(-sm.S[(k0 + i) * LS + k0 + m], x[m], x[i]);
    }
  } else {
#pragma unroll
    for (int m = 0; m < NB - 1; ++m)
#pragma unroll
      for (int i = m + 1; i < NB; ++i) x[i] = fma(-sm.S[(k0 + i) * LS + k0 + m], x[m], x[i]);
  }
  if (lane < NB) {
#pragma unroll
    for (int i = 0; i < NB; ++i) ex.tinv[upper ? 0 : 1][i * TS + l] = x[i];
  }
}

template <int F>
__device__ void lu_dmma_panels(Smem& sm, LuExtra& ex) {
  const int warp = warp_id();
  const bool lead = warp == NW - 1;
  auto chain = [&](int k) {
    if (F == 1)
      factor_invert_block(sm, ex, k);
    else if (F == 2)
      factor_diag_block_sm(sm, ex, k);
    else
      factor_diag_block(sm, k);
  };
  if (lead) chain(0);
  __syncthreads();
  for (int k0 = 0; k0 < N; k0 += NB) {
    const int rest = N - k0 - NB;
    const int nbk = rest / NB;
    if (F != 1) {
      if (warp < 2) tri_inverse_2warps(sm, ex, k0, warp == 0);
      __syncthreads();
    }
    if (warp < nbk)
      panel_block(sm, ex, k0, k0 + NB + NB * warp);
    else if (warp == NW - 2)
      diag_inverse_product(sm, ex, k0);
    __syncthreads();
    if (rest == 0) break;
    if (lead) {
      schur_block(sm, k0, k0 + NB, k0 + NB);
      __syncwarp();
      chain(k0 + NB);
    } else {
      for (int blk = warp + 1; blk < nbk * nbk; blk += NW - 1)
        schur_block(sm, k0, k0 + NB + NB * (blk / nbk), k0 + NB + NB * (blk % nbk));
    }
    __syncthreads();
  }
}

__device__ void fill(Smem& sm, int b) {
  for (int idx = threadIdx.x; idx < N * N; idx += NT) {
    const int r = idx >> 7, c = idx & (N - 1);
    const unsigned h = (unsigned)(r * 131 + c * 71 + b * 17) * 2654435761u;
    const double v = 1e-3 * ((double)(h >> 8) / 16777216.0 - 0.5);
    sm.S[r * LS + c] = (r == c) ? 1.0 + v : v;
  }
  __syncthreads();
}

// K: 0..15 = lu_head<K>, 100 = lu_block, 200 + F = lu_dmma_panels<F>, -1 = nothing
template <int K>
__global__ void __launch_bounds__(NT, 1) lu_kernel(int reps, long long* cyc, double* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  LuExtra& ex = *reinterpret_cast<LuExtra*>(smem_raw + sizeof(Smem));
  long long total = 0;
  for (int r = 0; r < reps; ++r) {
    fill(sm, blockIdx.x + r);
    const long long t0 = clock64();
    if constexpr (K == 100) {
      lu_block(sm, nullptr);
    } else if constexpr (K >= 200) {
      lu_dmma_panels<K - 200>(sm, ex);
    } else if constexpr (K >= 0) {
      lu_head<K>(sm);
    }
    __syncthreads();
    total += clock64() - t0;
  }
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = total / reps;
    out[blockIdx.x] = sm.S[5 * LS + 77] + sm.S[127 * LS + 127];
  }
}

__global__ void rcp_kernel(double* err, int n) {
  double e = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = ldexp(1.0 + (double)i / n, (i % 41) - 20) * ((i & 1) ? -1.0 : 1.0);
    const double r = rcp_cubic(x), q = 1.0 / x;
    e = fmax(e, fabs(r - q) / fabs(q));
  }
  atomicMax(reinterpret_cast<unsigned long long*>(err), __double_as_longlong(e));
}

}  // namespace
}  // namespace pf

template <int K>
void run(const char* name, int ctas, long long* dc, double* dout) {
  const int smem = (int)(sizeof(pf::Smem) + sizeof(pf::LuExtra));
  cudaFuncSetAttribute(pf::lu_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pf::lu_kernel<K><<<ctas, pf::NT, smem>>>(2, dc, dout);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pf::lu_kernel<K><<<ctas, pf::NT, smem>>>(8, dc, dout);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> h(ctas);
  cudaMemcpy(h.data(), dc, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double s = 0;
  for (long long v : h) s += (double)v;
  printf("%-52s %9.0f cycles/LU   (kernel %.3f ms, %s)\n", name, s / ctas, ms,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* dc;
  double* dout;
  cudaMalloc(&dc, sizeof(long long) * sms);
  cudaMalloc(&dout, sizeof(double) * sms);
  run<-1>("empty (fill + barrier only)", sms, dc, dout);
  run<100>("lu_block (production)", sms, dc, dout);
  run<0>("production schedule, all parts", sms, dc, dout);
  run<1>("  no lead factor", sms, dc, dout);
  run<2>("  no trailing update", sms, dc, dout);
  run<4>("  no panels / final inverses", sms, dc, dout);
  run<6>("  lead chain only (factor + schur)", sms, dc, dout);
  run<3>("  panels + final inverses only", sms, dc, dout);
  run<5>("  trailing only", sms, dc, dout);
  run<7>("  barriers + lead schur only", sms, dc, dout);
  run<16>("quiet lead SMSP (trailing on 12 warps)", sms, dc, dout);
  run<20>("  quiet lead SMSP, no panels", sms, dc, dout);
  run<21>("  quiet lead SMSP, trailing only", sms, dc, dout);
  run<200>("DMMA panels, two-warp triangular inverses", sms, dc, dout);
  run<201>("DMMA panels, lead factor_invert_block", sms, dc, dout);
  run<202>("DMMA panels, smem-broadcast factor", sms, dc, dout);
  double* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  pf::rcp_kernel<<<592, 256>>>(d, 1 << 26);
  double h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("rcp_cubic max relative error over 2^26 samples: %.3e\n", h);
  return 0;
}
