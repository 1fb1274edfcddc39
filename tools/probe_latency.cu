// Dependent-chain latencies (SM cycles) of the operations on the small kernel's LU critical path,
// one warp alone on the GPU:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 4096;

template <int OP>
__global__ void chain(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = seed + lane;
  sm[lane + 32] = 0.0;
  __syncwarp();
  double x = seed + lane * 1e-3, y = 1.0 + 1e-9 * lane;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < R; ++i) {
    if (OP == 0) x = fma(x, y, 1e-300);                          // DFMA
    if (OP == 1) x = x * y;                                       // DMUL
    if (OP == 2) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);  // SHFL (64-bit = 2 x 32)
    if (OP == 3) {                                                // MUFU.RCP64H
      double r;
      asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
      x = r;
    }
    if (OP == 4) x = sm[(int)(x * 0.0) + lane];                   // LDS (address depends on x)
    if (OP == 5) {                                                // DMMA m8n8k4, C chained
      double d0 = x, d1 = y;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d0), "+d"(d1) : "d"(1e-3), "d"(1e-3));
      x = d0;
      y = d1;
    }
    if (OP == 6) x = __shfl_sync(0xffffffffu, x, 0);              // SHFL broadcast
    if (OP == 7) x = (lane & 1) ? x * y : x;                      // select path
  }
  long long t1 = clock64();
  out[lane] = x + y;
  if (lane == 0) *cyc = t1 - t0;
}

// throughput: 8 independent streams per lane
template <int OP>
__global__ void thru(double* out, long long* cyc, double seed) {
  __shared__ double sm[256];
  const int lane = threadIdx.x;
  for (int i = lane; i < 256; i += 32) sm[i] = seed + i;
  __syncwarp();
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed + lane * 1e-3 + k;
  long long t0 = clock64();
  for (int i = 0; i < R / 8; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = __shfl_sync(0xffffffffu, x[k], (lane + k + 1) & 31);
      if (OP == 1) x[k] = fma(x[k], 1.0000001, 1e-300);
      if (OP == 2) {  // LDS.128 uniform address (broadcast) of two doubles
        const double2 v = *reinterpret_cast<const double2*>(&sm[((i + k) & 63) * 2]);
        x[k] += v.x * v.y;
      }
      if (OP == 3) {  // STS.64 + LDS.64 broadcast
        sm[(k * 16 + (i & 15))] = x[k];
        x[k] = sm[(k * 16 + ((i + 1) & 15))];
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[lane] = s;
  if (lane == 0) *cyc = t1 - t0;
}

template <int OP>
void runt(const char* name, double* o, long long* c) {
  long long h = 0;
  for (int it = 0; it < 2; ++it) {
    thru<OP><<<1, 32>>>(o, c, 1.5);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  }
  printf("%-28s %6.2f cycles per op (1 warp)\n", name, (double)h / R);
}

template <int OP>
void run(const char* name, double* o, long long* c) {
  long long h = 0;
  for (int it = 0; it < 2; ++it) {
    chain<OP><<<1, 32>>>(o, c, 1.5);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  }
  printf("%-28s %6.1f cycles\n", name, (double)h / R);
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&c, 8);
  run<0>("DFMA dependent", o, c);
  run<1>("DMUL dependent", o, c);
  run<2>("SHFL.IDX f64 dependent", o, c);
  run<6>("SHFL broadcast f64 dependent", o, c);
  run<3>("MUFU.RCP64H dependent", o, c);
  run<4>("LDS.64 dependent", o, c);
  run<5>("DMMA 8x8x4 dependent (C)", o, c);
  run<7>("DMUL under select", o, c);
  runt<0>("SHFL.IDX f64 independent", o, c);
  runt<1>("DFMA independent", o, c);
  runt<2>("LDS.128 broadcast + DFMA", o, c);
  runt<3>("STS.64 + LDS.64", o, c);
  return 0;
}
