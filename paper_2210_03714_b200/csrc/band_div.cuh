// Correctly rounded x / g from a precomputed reciprocal (band.cu's back-substitution divides every
// column by the same pivot fdiag_i, so the reciprocal is formed once per pivot, not per column).
//
//   y  = RN(1 / g)                 (__drcp_rn, once per pivot; 0 marks "no fast path")
//   q0 = RN(x y)                   faithful: |q0 - x/g| < 1 ulp
//   r  = x - g q0                  exact (one fma) when nothing underflows
//   q  = RN(q0 + r y)              = RN(x / g)   (Markstein's correction theorem)
//
// The fast path needs y != 0 -- set only for 2^-100 <= |g| <= 2^100 -- and 2^-800 <= |x| < 2^800
// (one integer test on x's exponent field). Then 2^-901 < |q0| < 2^901: the residual cannot
// underflow and the quotient cannot overflow, the theorem's hypotheses. Anything else (zeros,
// infinities, NaNs, extreme exponents, extreme pivots) goes through __ddiv_rn.
// tools/probe_div.cu checks equality with __ddiv_rn.
#pragma once

namespace pf {

__device__ __forceinline__ double band_rcp(double g) {
  const double a = fabs(g);
  return (a >= 0x1p-100 && a <= 0x1p100) ? __drcp_rn(g) : 0.0;
}

// biased exponent of x in [1023 - 800, 1023 + 800)
__device__ __forceinline__ bool div_rcp_x_ok(double x) {
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
  return e - (1023u - 800u) < 1600u;
}

// y is +0.0 (hi word 0) or a normal reciprocal (hi word != 0): an integer test
__device__ __forceinline__ bool div_rcp_fast_ok(double x, double y) { return __double2hiint(y) != 0 && div_rcp_x_ok(x); }

__device__ __forceinline__ double div_rcp(double x, double g, double y) {
  if (div_rcp_fast_ok(x, y)) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-g, q0, x);
    return __fma_rn(r, y, q0);
  }
  return __ddiv_rn(x, g);
}

}  // namespace pf
