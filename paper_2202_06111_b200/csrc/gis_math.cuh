// fp64 sin / cos fast paths for the integrator.
//
// CUDA's sin/cos reduce the argument by pi/2 with integer quadrant logic
// and load polynomial coefficients from a global table (LDG + XU/ALU work
// per call).  The state-space arguments of the BASELINE models are small
// (pendulum angle |x1| <~ 1.3, cart-pole |theta| <~ 0.3), so:
//   |x| <= pi/2 : sin x = x + x^3 P(x^2), P the Taylor coefficients through
//                 x^21 (truncation < 2e-18 relative), 9 DFMA + 2 DMUL + 1 DFMA
//   |x| <= pi/4 : cos x = 1 + x^2 Q(x^2), Q through x^22
// and CUDA's sin/cos otherwise.  Coefficients are compile-time constants
// (constant-bank operands, no loads).  Accuracy ~1 ulp, the same class as
// CUDA's and numpy's implementations.
#pragma once

namespace gis {

__device__ __forceinline__ double sin_poly(double x) {
  const double x2 = x * x;
  double p = 1.9572941063391263e-20;           //  1/21!
  p = fma(p, x2, -8.22063524662433e-18);     // -1/19!
  p = fma(p, x2, 2.8114572543455206e-15);      //  1/17!
  p = fma(p, x2, -7.647163731819816e-13);     // -1/15!
  p = fma(p, x2, 1.6059043836821613e-10);      //  1/13!
  p = fma(p, x2, -2.505210838544172e-08);     // -1/11!
  p = fma(p, x2, 2.7557319223985893e-06);      //  1/9!
  p = fma(p, x2, -0.0001984126984126984);     // -1/7!
  p = fma(p, x2, 0.008333333333333333);      //  1/5!
  p = fma(p, x2, -0.16666666666666666);     // -1/3!
  return fma(x * x2, p, x);
}

__device__ __forceinline__ double cos_poly(double x) {
  const double x2 = x * x;
  double q = -8.896791392450574e-22;          // -1/22!
  q = fma(q, x2, 4.110317623312165e-19);      //  1/20!
  q = fma(q, x2, -1.5619206968586225e-16);     // -1/18!
  q = fma(q, x2, 4.779477332387385e-14);      //  1/16!
  q = fma(q, x2, -1.1470745597729725e-11);     // -1/14!
  q = fma(q, x2, 2.08767569878681e-09);      //  1/12!
  q = fma(q, x2, -2.755731922398589e-07);     // -1/10!
  q = fma(q, x2, 2.48015873015873e-05);      //  1/8!
  q = fma(q, x2, -0.001388888888888889);     // -1/6!
  q = fma(q, x2, 0.041666666666666664);      //  1/4!
  q = fma(q, x2, -0.5);                        // -1/2!
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
