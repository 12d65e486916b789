// sin / cos in double for any |x| < 2^50 without CUDA's Payne-Hanek slow
// path (local-memory table walk, ~4x slower), which the Weierstrass series
// hits for every k >= 9: its arguments fl(fl(2*pi*3^k) * (z + 0.5)) reach
// ~5e10 (kernels.py:104).
//
// Reduction: n = rint(x * 2/pi) via the 1.5*2^52 shifter, then
// r = x - n*C1 - n*C2 - n*C3 with FMAs (pi/2 = C1 + C2 + C3 to ~160 bits).
// Each FMA rounds once; for |n| < 2^36 the result's absolute error is
// ~ulp(r) + |n| * 2^-160, i.e. < 2e-16 for |r| <= pi/4.
// Kernels: the classic fdlibm __kernel_sin / __kernel_cos minimax
// polynomials on [-pi/4, pi/4] (< 1 ulp), selected branch-free by quadrant.
#pragma once
#include <cuda_runtime.h>

namespace rb {

__device__ __forceinline__ void sincos_reduce(double x, double& r, int& q) {
  const double kShifter = 6755399441055744.0;          // 1.5 * 2^52
  const double t = fma(x, 0.63661977236758134308, kShifter);
  q = __double2loint(t);
  const double n = t - kShifter;
  r = fma(-n, 1.5707963267948965580e+00, x);           // C1 = RN(pi/2)
  r = fma(-n, 6.1232339957367658e-17, r);               // C2 = RN(pi/2 - C1)
  r = fma(-n, -1.4973849048591698e-33, r);              // C3 = RN(pi/2 - C1 - C2)
}

__device__ __forceinline__ double k_sin(double r) {
  const double z = r * r, v = z * r;
  double p = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
  p = fma(z, p, 2.75573137070700676789e-06);
  p = fma(z, p, -1.98412698298579493134e-04);
  p = fma(z, p, 8.33333333332248946124e-03);
  p = fma(z, p, -1.66666666666666324348e-01);
  return fma(v, p, r);
}

__device__ __forceinline__ double k_cos(double r) {
  const double z = r * r;
  double p = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
  p = fma(z, p, -2.75573143513906633035e-07);
  p = fma(z, p, 2.48015872894767294178e-05);
  p = fma(z, p, -1.38888888888741095749e-03);
  p = fma(z, p, 4.16666666666666019037e-02);
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  return w + (((1.0 - w) - hz) + z * (z * p));
}

__device__ __forceinline__ double fast_cos(double x) {
  double r;
  int q;
  sincos_reduce(x, r, q);
  const double s = k_sin(r), c = k_cos(r);
  const double v = (q & 1) ? s : c;
  return ((q + 1) & 2) ? -v : v;                        // q=1: -sin, 2: -cos, 3: sin
}

__device__ __forceinline__ double fast_sin(double x) {
  double r;
  int q;
  sincos_reduce(x, r, q);
  const double s = k_sin(r), c = k_cos(r);
  const double v = (q & 1) ? c : s;
  return (q & 2) ? -v : v;                              // q=1: cos, 2: -sin, 3: -cos
}

}  // namespace rb
