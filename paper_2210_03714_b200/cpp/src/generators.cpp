// Seeded input generators (not timed): SplitMix64 / NormalSampler (proj/core/include/parfrac/rng.hpp:10-39,
// proj/core/src/rng.cpp:7-19) and the matrix kinds of make_dense_matrix (proj/core/src/cli.cpp:35-56).
// Host code: glibc log/sin/cos give the identical bytes the reference's generator produces.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "parfrac/rng.hpp"

namespace parfrac {

double NormalSampler::next() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  double u1 = 1.0 - rng_.uniform();  // (0, 1], keeps the log finite
  double u2 = rng_.uniform();
  double r = std::sqrt(-2.0 * std::log(u1));
  double angle = 2.0 * 3.14159265358979323846 * u2;
  spare_ = r * std::sin(angle);
  have_spare_ = true;
  return r * std::cos(angle);
}

}  // namespace parfrac

extern "C" {

// `count` normals from NormalSampler(seed), row-major fill order.
void pf_gen_randn(uint64_t seed, int64_t count, double* out) {
  parfrac::NormalSampler s(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = s.next();
}

// `count` uniforms in [0, 1) from SplitMix64(seed).
void pf_gen_uniform(uint64_t seed, int64_t count, double* out) {
  parfrac::SplitMix64 s(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = s.uniform();
}

// batch of n x n randn matrices, matrix b from NormalSampler(seed0 + b), generated on `threads` host threads.
void pf_gen_randn_batch(uint64_t seed0, int batch, int n, double* out, int threads) {
  const int64_t nn = int64_t(n) * n;
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([=] {
      for (int b = t; b < batch; b += threads) pf_gen_randn(seed0 + uint64_t(b), nn, out + nn * b);
    });
  for (auto& th : pool) th.join();
}

}  // extern "C"
