// sin / cos without CUDA's Payne-Hanek slow path (local-memory table walk),
// which the Weierstrass series hits for every k >= 9: its arguments
// fl(fl(2*pi*3^k) * (z + 0.5)) reach ~5e10 (kernels.py:104).
//
// One reduction by pi and ONE polynomial per call (no sin/cos pair + select):
//   n = rint(x / pi)                    (1.5*2^52 shifter, |x| < 2^40)
//   r = x - n*P1 - n*P2                 (FMA Cody-Waite, pi = P1 + P2 + O(2^-107);
//                                        |r| <= pi/2, abs. error ~ulp(r) + |n| 2^-107)
//   cos x = (-1)^n cos r,  sin x = (-1)^n sin r
//   cos r = 1 + z Q(z),    sin r = r + r z S(z),   z = r^2
// Q, S: minimax on |r| <= pi/2 for the absolute error of the whole
// (tools/trig_fit.py): double 7.7e-18 / 4.9e-19, float 4.4e-10 / 1.0e-8,
// i.e. every result is within ~1 ulp of 1 in absolute terms.  The sign flip
// is an integer xor (ALU pipe).  |x| >= 2^40 (only reachable with huge
// user inputs) takes CUDA's full-range cos/sin.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rb {

constexpr double kShifter = 6755399441055744.0;          // 1.5 * 2^52
constexpr double kInvPi = 0.31830988618379067154;
constexpr double kPi1 = 3.141592653589793116;            // RN(pi)
constexpr double kPi2 = 1.2246467991473532e-16;          // RN(pi - P1)
constexpr double kTrigBig = 1099511627776.0;             // 2^40

__device__ __forceinline__ double trig_reduce_pi(double x, int& q) {
  const double t = fma(x, kInvPi, kShifter);
  q = __double2loint(t);
  const double n = t - kShifter;
  const double r = fma(-n, kPi1, x);
  return fma(-n, kPi2, r);
}

__device__ __forceinline__ double flip_sign(double v, int q) {
  return __hiloint2double(__double2hiint(v) ^ (int)((unsigned)q << 31), __double2loint(v));
}
__device__ __forceinline__ float flip_sign(float v, int q) {
  return __int_as_float(__float_as_int(v) ^ (int)((unsigned)q << 31));
}

// cos r = 1 + z Q(z) on |r| <= pi/2, degree-7 Q (abs. error 7.7e-18)
__device__ __forceinline__ double cos_poly(double z) {
  double p = fma(z, 4.608992189914223e-14, -1.1462960932485546e-11);
  p = fma(z, p, 2.087656686900375e-09);
  p = fma(z, p, -2.7557316560884815e-07);
  p = fma(z, p, 2.4801587280266368e-05);
  p = fma(z, p, -0.0013888888888797584);
  p = fma(z, p, 0.041666666666664895);
  p = fma(z, p, -0.4999999999999999);
  return fma(z, p, 1.0);
}
// degree-6 Q (abs. error 3.9e-15): the Weierstrass series only, where 21*d
// terms of weight <= 1 sum to a value of order d and the bar is 1e-12 relative
__device__ __forceinline__ double cos_poly6(double z) {
  double p = fma(z, -1.1008014104749214e-11, 2.0858498365979955e-09);
  p = fma(z, p, -2.7556948583923867e-07);
  p = fma(z, p, 2.48015832336902e-05);
  p = fma(z, p, -0.0013888888865724836);
  p = fma(z, p, 0.0416666666660776);
  p = fma(z, p, -0.499999999999956);
  return fma(z, p, 1.0);
}
// sin r = r + r z S(z), degree-7 S (abs. error 4.9e-19)
__device__ __forceinline__ double sin_poly(double r) {
  const double z = r * r;
  double p = fma(z, 2.7215821926997076e-15, -7.643057647491696e-13);
  p = fma(z, p, 1.6058943530517797e-10);
  p = fma(z, p, -2.5052106980181033e-08);
  p = fma(z, p, 2.7557319212734233e-06);
  p = fma(z, p, -0.00019841269841221654);
  p = fma(z, p, 0.00833333333333324);
  p = fma(z, p, -0.16666666666666666);
  return fma(r * z, p, r);
}

static __device__ __noinline__ double cos_big(double x) { return ::cos(x); }
static __device__ __noinline__ double sin_big(double x) { return ::sin(x); }

__device__ __forceinline__ double fast_cos(double x) {
  if (!(fabs(x) < kTrigBig)) return cos_big(x);
  int q;
  const double r = trig_reduce_pi(x, q);
  return flip_sign(cos_poly(r * r), q);
}

__device__ __forceinline__ double fast_sin(double x) {
  if (!(fabs(x) < kTrigBig)) return sin_big(x);
  int q;
  const double r = trig_reduce_pi(x, q);
  return flip_sign(sin_poly(r), q);
}

// float32 sin/cos for the float path: the exact reduction runs in double
// (float arguments reach ~5e10 in Weierstrass), the polynomial in float on
// the FP32 pipe.  Within ~1 ulp of the correctly rounded result, like
// NumPy's own float32 SIMD sin/cos.
__device__ __forceinline__ float trig_reduce_pi_f(float x, int& q) {
  return (float)trig_reduce_pi((double)x, q);
}

__device__ __forceinline__ float cos_polyf(float z) {       // abs. error 4.4e-10
  float p = fmaf(z, -2.6051076353347883e-07f, 2.4760893012965208e-05f);
  p = fmaf(z, p, -0.0013888398239410408f);
  p = fmaf(z, p, 0.041666641979438764f);
  p = fmaf(z, p, -0.49999999641974857f);
  return fmaf(z, p, 1.0f);
}

__device__ __forceinline__ float sin_polyf(float r) {       // abs. error 1.0e-8
  const float z = r * r;
  float p = fmaf(z, 2.6051662760767676e-06f, -0.0001980995536299565f);
  p = fmaf(z, p, 0.008333084282862243f);
  p = fmaf(z, p, -0.16666661088338824f);
  return fmaf(r * z, p, r);
}

static __device__ __noinline__ float cosf_big(float x) { return (float)::cos((double)x); }
static __device__ __noinline__ float sinf_big(float x) { return (float)::sin((double)x); }

__device__ __forceinline__ float fast_cosf(float x) {
  if (!(fabsf(x) < (float)kTrigBig)) return cosf_big(x);
  int q;
  const float r = trig_reduce_pi_f(x, q);
  return flip_sign(cos_polyf(r * r), q);
}

__device__ __forceinline__ float fast_sinf(float x) {
  if (!(fabsf(x) < (float)kTrigBig)) return sinf_big(x);
  int q;
  const float r = trig_reduce_pi_f(x, q);
  return flip_sign(sin_polyf(r), q);
}

}  // namespace rb
