// Probe: the reciprocal-based correctly rounded division used by the fused banded step
// (band.cu div_rcp) against __ddiv_rn, on random operands over the exponent range the fast path
// accepts plus its edges. Prints the mismatch count (must be 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_div tools/probe_div.cu && /tmp/probe_div
#include <cstdint>
#include <cstdio>

#include "../paper_2210_03714_b200/csrc/band_div.cuh"

__device__ uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ double rand_double(uint64_t& s, int emin, int emax) {
  const uint64_t r = splitmix(s);
  const int e = emin + (int)(r % (uint64_t)(emax - emin + 1));
  const uint64_t mant = splitmix(s) & ((1ull << 52) - 1);
  const uint64_t sign = (r >> 63) << 63;
  return __longlong_as_double((long long)(sign | ((uint64_t)(e + 1023) << 52) | mant));
}

__global__ void probe(uint64_t seed, int iters, int ex_lo, int ex_hi, int eg_lo, int eg_hi,
                      unsigned long long* bad, unsigned long long* fast) {
  uint64_t s = seed ^ (0x1234567ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  unsigned long long nb = 0, nf = 0;
  for (int it = 0; it < iters; ++it) {
    const double x = rand_double(s, ex_lo, ex_hi);
    const double g = rand_double(s, eg_lo, eg_hi);
    const double y = pf::band_rcp(g);
    const double q = pf::div_rcp(x, g, y);
    const double ref = __ddiv_rn(x, g);
    nb += __double_as_longlong(q) != __double_as_longlong(ref);
    nf += pf::div_rcp_fast_ok(x, y);
    // also the near-quotient-boundary operands: x = g * q' for a random q' (exact ties are rare;
    // products rounded to nearby representables stress the final rounding)
    const double qq = rand_double(s, -60, 60);
    const double x2 = __dmul_rn(g, qq);
    const double q2 = pf::div_rcp(x2, g, y), r2 = __ddiv_rn(x2, g);
    nb += __double_as_longlong(q2) != __double_as_longlong(r2);
  }
  atomicAdd(bad, nb);
  atomicAdd(fast, nf);
}

int main() {
  unsigned long long *bad, *fast;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&fast, 8);
  struct Case {
    int xl, xh, gl, gh;
  } cases[] = {{-30, 30, -30, 30}, {-900, 900, -900, 900}, {-1000, 1000, -1000, 1000}, {-1022, 1023, -1022, 1023},
               {-5, 5, -990, -980}, {-5, 5, 980, 990}, {-820, -780, -110, 110}, {780, 820, -110, 110},
               {-1074, -1000, -3, 3}};
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  bool ok = true;
  for (const Case& c : cases) {
    *bad = 0;
    *fast = 0;
    probe<<<blocks, threads>>>(42 + c.xl, iters, c.xl, c.xh, c.gl, c.gh, bad, fast);
    cudaDeviceSynchronize();
    const double n = (double)blocks * threads * iters;
    std::printf("x exp [%d,%d] g exp [%d,%d]: %.3e pairs x2, mismatches %llu, fast path %.1f%%\n", c.xl, c.xh, c.gl,
                c.gh, n, *bad, 100.0 * (double)*fast / n);
    ok = ok && *bad == 0;
  }
  std::printf(ok ? "div_rcp == __ddiv_rn on every probe\n" : "MISMATCH\n");
  return ok ? 0 : 1;
}
