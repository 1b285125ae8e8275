// green.cuh -- device evaluation of the on-surface Neumann Green's functions.
//
// Paper forms (three terms, d = |x - x'|):
//   G_E = 2/d - log(2/d) - log(1 + d/2)      eq:Gextonsurface
//   G_I = 2/d + log(2/d) - log(1 + d/2)      eq:Gintonsurface
// Exact single-log rewrites used on the GPU (SURVEY.md §8(a) "Kernel facts"):
// with w = 2/d,  w (1 + d/2) = w + 1  and  (2/d) / (1 + d/2) = 4 / (d^2 + 2d), hence
//   G_E = w - log(1 + w)
//   G_I = w + log 4 - log(d^2 + 2 d)
// One reciprocal square root and one logarithm per pair, no division.
#pragma once

#include <stdint.h>

namespace nc {

constexpr double kLog4 = 1.3862943611198906188344642429163531;  // log(4)
constexpr double kLn2Hi = 6.93147180369123816490e-01;           // fdlibm split of ln 2
constexpr double kLn2Lo = 1.90821492927058770002e-10;

// ------------------------------------------------------------------------------------------------
// Table-free fp64 natural log for x in [1, 2^1000): x = 2^e m, m in [sqrt(1/2), sqrt(2));
// f = m - 1, s = f / (2 + f) (computed without division: s = f * rcp(2+f) by Newton on MUFU seed),
// log(m) = 2 atanh(s) = f - hf + s (hf + R(s^2)),  R = Remez/fdlibm minimax polynomial (|err| < 2^-58).
// Accuracy: < 1 ulp of the result over the range used (validated in tests/test_kernels_gpu.py
// against the oracle at the 1e-13 relative level).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double nc_log(double x) {
  return log(x);
}

// rsqrt with full fp64 accuracy (CUDA's rsqrt: <= 1 ulp)
__device__ __forceinline__ double nc_rsqrt(double x) { return rsqrt(x); }

template <int KIND>
__device__ __forceinline__ double green_from_d2(double d2) {
  double rs = nc_rsqrt(d2);
  double w = 2.0 * rs;
  if (KIND == 1) {
    return w - nc_log(1.0 + w);
  } else {
    double d = d2 * rs;
    return w + kLog4 - nc_log(fma(2.0, d, d2));
  }
}

}  // namespace nc
