// fp64 sin / cos fast paths for the integrator.
//
// CUDA's sin/cos reduce the argument by pi/2 with integer quadrant logic
// and load polynomial coefficients from a global table (LDG + XU/ALU work
// per call).  The state-space arguments of the BASELINE models are small
// (pendulum angle |x1| <~ 1.3, cart-pole |theta| <~ 0.3), so:
//   |x| <= pi/2 : sin x = x + x^3 P(x^2), P the Taylor coefficients through
//                 x^21 (truncation < 2e-18 relative): 2 DMUL + 10 DFMA
//   |x| <= pi/4 : cos x = 1 + x^2 Q(x^2), Q through x^22: 1 DMUL + 11 DFMA
// and CUDA's sin/cos otherwise.  The coefficients live in the constant bank
// (__constant__) so every DFMA takes its coefficient as a c[][] operand --
// no loads and no 64-bit immediate moves.  Accuracy <= 2 ulp against libm
// on the fast-path ranges, the same class as CUDA's and numpy's sin/cos.
#pragma once

namespace gis {

// 1/21!, -1/19!, ..., -1/3!
static __constant__ double kSinCoef[10] = {
    1.9572941063391263e-20,
    -8.22063524662433e-18,
    2.8114572543455206e-15,
    -7.647163731819816e-13,
    1.6059043836821613e-10,
    -2.505210838544172e-08,
    2.7557319223985893e-06,
    -0.0001984126984126984,
    0.008333333333333333,
    -0.16666666666666666,
};

// -1/22!, 1/20!, ..., -1/2!
static __constant__ double kCosCoef[11] = {
    -8.896791392450574e-22,
    4.110317623312165e-19,
    -1.5619206968586225e-16,
    4.779477332387385e-14,
    -1.1470745597729725e-11,
    2.08767569878681e-09,
    -2.755731922398589e-07,
    2.48015873015873e-05,
    -0.001388888888888889,
    0.041666666666666664,
    -0.5,
};

__device__ __forceinline__ double sin_poly(double x) {
  const double x2 = x * x;
  double p = kSinCoef[0];
#pragma unroll
  for (int i = 1; i < 10; ++i) p = fma(p, x2, kSinCoef[i]);
  return fma(x * x2, p, x);
}

__device__ __forceinline__ double cos_poly(double x) {
  const double x2 = x * x;
  double q = kCosCoef[0];
#pragma unroll
  for (int i = 1; i < 11; ++i) q = fma(q, x2, kCosCoef[i]);
  return fma(x2, q, 1.0);
}

__device__ __forceinline__ double fast_sin(double x) {
  return (fabs(x) <= 1.5707963267948966) ? sin_poly(x) : sin(x);
}

__device__ __forceinline__ double fast_cos(double x) {
  return (fabs(x) <= 0.78539816339744831) ? cos_poly(x) : cos(x);
}

__device__ __forceinline__ void fast_sincos(double x, double* s, double* c) {
  if (fabs(x) <= 0.78539816339744831) {
    *s = sin_poly(x);
    *c = cos_poly(x);
  } else {
    sincos(x, s, c);
  }
}

}  // namespace gis
