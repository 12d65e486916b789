// sin / cos in double for |x| < 2^45 without CUDA's Payne-Hanek slow path
// (local-memory table walk), which the Weierstrass series hits for every
// k >= 9: its arguments fl(fl(2*pi*3^k) * (z + 0.5)) reach ~5e10
// (kernels.py:104).
//
//   n = rint(x * 64/pi)                 (1.5*2^52 shifter; n < 2^45)
//   r = x - n*C1 - n*C2 - n*C3          (FMA Cody-Waite, pi/64 = C1+C2+C3 to
//                                        ~160 bits; |r| <= pi/128, abs. error
//                                        ~ulp(r) + |n|*2^-165)
//   cos x = cos(n pi/64) cos r - sin(n pi/64) sin r
//   sin x = sin(n pi/64) cos r + cos(n pi/64) sin r
// with a 128-entry table of correctly rounded (cos, sin)(k pi/64) and
// Taylor polynomials to r^6 / r^7 (truncation < 4e-18 on |r| <= pi/128).
// ~15 double ops and one 16-byte L1 load per call; error < 2 ulp.
#pragma once
#include <cuda_runtime.h>

namespace rb {

// (cos, sin)(k * pi / 64), k = 0..127, as IEEE double bit patterns
__device__ const unsigned long long kTrigTable[128][2] = {
    {0x3ff0000000000000ull, 0x0000000000000000ull},
    {0x3feff621e3796d7eull, 0x3fa91f65f10dd814ull},
    {0x3fefd88da3d12526ull, 0x3fb917a6bc29b42cull},
    {0x3fefa7557f08a517ull, 0x3fc2c8106e8e613aull},
    {0x3fef6297cff75cb0ull, 0x3fc8f8b83c69a60bull},
    {0x3fef0a7efb9230d7ull, 0x3fcf19f97b215f1bull},
    {0x3fee9f4156c62ddaull, 0x3fd294062ed59f06ull},
    {0x3fee212104f686e5ull, 0x3fd58f9a75ab1fddull},
    {0x3fed906bcf328d46ull, 0x3fd87de2a6aea963ull},
    {0x3feced7af43cc773ull, 0x3fdb5d1009e15cc0ull},
    {0x3fec38b2f180bdb1ull, 0x3fde2b5d3806f63bull},
    {0x3feb728345196e3eull, 0x3fe073879922ffeeull},
    {0x3fea9b66290ea1a3ull, 0x3fe1c73b39ae68c8ull},
    {0x3fe9b3e047f38741ull, 0x3fe30ff7fce17035ull},
    {0x3fe8bc806b151741ull, 0x3fe44cf325091dd6ull},
    {0x3fe7b5df226aafafull, 0x3fe57d69348ceca0ull},
    {0x3fe6a09e667f3bcdull, 0x3fe6a09e667f3bcdull},
    {0x3fe57d69348ceca0ull, 0x3fe7b5df226aafafull},
    {0x3fe44cf325091dd6ull, 0x3fe8bc806b151741ull},
    {0x3fe30ff7fce17035ull, 0x3fe9b3e047f38741ull},
    {0x3fe1c73b39ae68c8ull, 0x3fea9b66290ea1a3ull},
    {0x3fe073879922ffeeull, 0x3feb728345196e3eull},
    {0x3fde2b5d3806f63bull, 0x3fec38b2f180bdb1ull},
    {0x3fdb5d1009e15cc0ull, 0x3feced7af43cc773ull},
    {0x3fd87de2a6aea963ull, 0x3fed906bcf328d46ull},
    {0x3fd58f9a75ab1fddull, 0x3fee212104f686e5ull},
    {0x3fd294062ed59f06ull, 0x3fee9f4156c62ddaull},
    {0x3fcf19f97b215f1bull, 0x3fef0a7efb9230d7ull},
    {0x3fc8f8b83c69a60bull, 0x3fef6297cff75cb0ull},
    {0x3fc2c8106e8e613aull, 0x3fefa7557f08a517ull},
    {0x3fb917a6bc29b42cull, 0x3fefd88da3d12526ull},
    {0x3fa91f65f10dd814ull, 0x3feff621e3796d7eull},
    {0x0000000000000000ull, 0x3ff0000000000000ull},
    {0xbfa91f65f10dd814ull, 0x3feff621e3796d7eull},
    {0xbfb917a6bc29b42cull, 0x3fefd88da3d12526ull},
    {0xbfc2c8106e8e613aull, 0x3fefa7557f08a517ull},
    {0xbfc8f8b83c69a60bull, 0x3fef6297cff75cb0ull},
    {0xbfcf19f97b215f1bull, 0x3fef0a7efb9230d7ull},
    {0xbfd294062ed59f06ull, 0x3fee9f4156c62ddaull},
    {0xbfd58f9a75ab1fddull, 0x3fee212104f686e5ull},
    {0xbfd87de2a6aea963ull, 0x3fed906bcf328d46ull},
    {0xbfdb5d1009e15cc0ull, 0x3feced7af43cc773ull},
    {0xbfde2b5d3806f63bull, 0x3fec38b2f180bdb1ull},
    {0xbfe073879922ffeeull, 0x3feb728345196e3eull},
    {0xbfe1c73b39ae68c8ull, 0x3fea9b66290ea1a3ull},
    {0xbfe30ff7fce17035ull, 0x3fe9b3e047f38741ull},
    {0xbfe44cf325091dd6ull, 0x3fe8bc806b151741ull},
    {0xbfe57d69348ceca0ull, 0x3fe7b5df226aafafull},
    {0xbfe6a09e667f3bcdull, 0x3fe6a09e667f3bcdull},
    {0xbfe7b5df226aafafull, 0x3fe57d69348ceca0ull},
    {0xbfe8bc806b151741ull, 0x3fe44cf325091dd6ull},
    {0xbfe9b3e047f38741ull, 0x3fe30ff7fce17035ull},
    {0xbfea9b66290ea1a3ull, 0x3fe1c73b39ae68c8ull},
    {0xbfeb728345196e3eull, 0x3fe073879922ffeeull},
    {0xbfec38b2f180bdb1ull, 0x3fde2b5d3806f63bull},
    {0xbfeced7af43cc773ull, 0x3fdb5d1009e15cc0ull},
    {0xbfed906bcf328d46ull, 0x3fd87de2a6aea963ull},
    {0xbfee212104f686e5ull, 0x3fd58f9a75ab1fddull},
    {0xbfee9f4156c62ddaull, 0x3fd294062ed59f06ull},
    {0xbfef0a7efb9230d7ull, 0x3fcf19f97b215f1bull},
    {0xbfef6297cff75cb0ull, 0x3fc8f8b83c69a60bull},
    {0xbfefa7557f08a517ull, 0x3fc2c8106e8e613aull},
    {0xbfefd88da3d12526ull, 0x3fb917a6bc29b42cull},
    {0xbfeff621e3796d7eull, 0x3fa91f65f10dd814ull},
    {0xbff0000000000000ull, 0x0000000000000000ull},
    {0xbfeff621e3796d7eull, 0xbfa91f65f10dd814ull},
    {0xbfefd88da3d12526ull, 0xbfb917a6bc29b42cull},
    {0xbfefa7557f08a517ull, 0xbfc2c8106e8e613aull},
    {0xbfef6297cff75cb0ull, 0xbfc8f8b83c69a60bull},
    {0xbfef0a7efb9230d7ull, 0xbfcf19f97b215f1bull},
    {0xbfee9f4156c62ddaull, 0xbfd294062ed59f06ull},
    {0xbfee212104f686e5ull, 0xbfd58f9a75ab1fddull},
    {0xbfed906bcf328d46ull, 0xbfd87de2a6aea963ull},
    {0xbfeced7af43cc773ull, 0xbfdb5d1009e15cc0ull},
    {0xbfec38b2f180bdb1ull, 0xbfde2b5d3806f63bull},
    {0xbfeb728345196e3eull, 0xbfe073879922ffeeull},
    {0xbfea9b66290ea1a3ull, 0xbfe1c73b39ae68c8ull},
    {0xbfe9b3e047f38741ull, 0xbfe30ff7fce17035ull},
    {0xbfe8bc806b151741ull, 0xbfe44cf325091dd6ull},
    {0xbfe7b5df226aafafull, 0xbfe57d69348ceca0ull},
    {0xbfe6a09e667f3bcdull, 0xbfe6a09e667f3bcdull},
    {0xbfe57d69348ceca0ull, 0xbfe7b5df226aafafull},
    {0xbfe44cf325091dd6ull, 0xbfe8bc806b151741ull},
    {0xbfe30ff7fce17035ull, 0xbfe9b3e047f38741ull},
    {0xbfe1c73b39ae68c8ull, 0xbfea9b66290ea1a3ull},
    {0xbfe073879922ffeeull, 0xbfeb728345196e3eull},
    {0xbfde2b5d3806f63bull, 0xbfec38b2f180bdb1ull},
    {0xbfdb5d1009e15cc0ull, 0xbfeced7af43cc773ull},
    {0xbfd87de2a6aea963ull, 0xbfed906bcf328d46ull},
    {0xbfd58f9a75ab1fddull, 0xbfee212104f686e5ull},
    {0xbfd294062ed59f06ull, 0xbfee9f4156c62ddaull},
    {0xbfcf19f97b215f1bull, 0xbfef0a7efb9230d7ull},
    {0xbfc8f8b83c69a60bull, 0xbfef6297cff75cb0ull},
    {0xbfc2c8106e8e613aull, 0xbfefa7557f08a517ull},
    {0xbfb917a6bc29b42cull, 0xbfefd88da3d12526ull},
    {0xbfa91f65f10dd814ull, 0xbfeff621e3796d7eull},
    {0x0000000000000000ull, 0xbff0000000000000ull},
    {0x3fa91f65f10dd814ull, 0xbfeff621e3796d7eull},
    {0x3fb917a6bc29b42cull, 0xbfefd88da3d12526ull},
    {0x3fc2c8106e8e613aull, 0xbfefa7557f08a517ull},
    {0x3fc8f8b83c69a60bull, 0xbfef6297cff75cb0ull},
    {0x3fcf19f97b215f1bull, 0xbfef0a7efb9230d7ull},
    {0x3fd294062ed59f06ull, 0xbfee9f4156c62ddaull},
    {0x3fd58f9a75ab1fddull, 0xbfee212104f686e5ull},
    {0x3fd87de2a6aea963ull, 0xbfed906bcf328d46ull},
    {0x3fdb5d1009e15cc0ull, 0xbfeced7af43cc773ull},
    {0x3fde2b5d3806f63bull, 0xbfec38b2f180bdb1ull},
    {0x3fe073879922ffeeull, 0xbfeb728345196e3eull},
    {0x3fe1c73b39ae68c8ull, 0xbfea9b66290ea1a3ull},
    {0x3fe30ff7fce17035ull, 0xbfe9b3e047f38741ull},
    {0x3fe44cf325091dd6ull, 0xbfe8bc806b151741ull},
    {0x3fe57d69348ceca0ull, 0xbfe7b5df226aafafull},
    {0x3fe6a09e667f3bcdull, 0xbfe6a09e667f3bcdull},
    {0x3fe7b5df226aafafull, 0xbfe57d69348ceca0ull},
    {0x3fe8bc806b151741ull, 0xbfe44cf325091dd6ull},
    {0x3fe9b3e047f38741ull, 0xbfe30ff7fce17035ull},
    {0x3fea9b66290ea1a3ull, 0xbfe1c73b39ae68c8ull},
    {0x3feb728345196e3eull, 0xbfe073879922ffeeull},
    {0x3fec38b2f180bdb1ull, 0xbfde2b5d3806f63bull},
    {0x3feced7af43cc773ull, 0xbfdb5d1009e15cc0ull},
    {0x3fed906bcf328d46ull, 0xbfd87de2a6aea963ull},
    {0x3fee212104f686e5ull, 0xbfd58f9a75ab1fddull},
    {0x3fee9f4156c62ddaull, 0xbfd294062ed59f06ull},
    {0x3fef0a7efb9230d7ull, 0xbfcf19f97b215f1bull},
    {0x3fef6297cff75cb0ull, 0xbfc8f8b83c69a60bull},
    {0x3fefa7557f08a517ull, 0xbfc2c8106e8e613aull},
    {0x3fefd88da3d12526ull, 0xbfb917a6bc29b42cull},
    {0x3feff621e3796d7eull, 0xbfa91f65f10dd814ull},};

__device__ __forceinline__ void trig_reduce(double x, double& r, int& k) {
  const double kShifter = 6755399441055744.0;          // 1.5 * 2^52
  const double t = fma(x, 20.371832715762604, kShifter);   // 64/pi
  k = __double2loint(t) & 127;
  const double n = t - kShifter;
  r = fma(-n, 0.04908738521234052, x);                  // C1 = RN(pi/64)
  r = fma(-n, 1.9135106236677394e-18, r);               // C2 = RN(pi/64 - C1)
  r = fma(-n, -4.6793278276849057e-35, r);              // C3
}

__device__ __forceinline__ void trig_poly(double r, double& c, double& s) {
  const double z = r * r;
  c = fma(z, fma(z, fma(z, -1.3888888888888889e-03, 4.1666666666666664e-02), -0.5), 1.0);
  const double p = fma(z, fma(z, -1.9841269841269841e-04, 8.3333333333333332e-03),
                       -1.6666666666666666e-01);
  s = fma(r * z, p, r);
}

__device__ __forceinline__ double2 trig_entry(int k) {
  return __ldg(reinterpret_cast<const double2*>(kTrigTable) + k);
}

#ifndef RB_TRIG_TABLE
#define RB_TRIG_TABLE 0
#endif

#if RB_TRIG_TABLE
__device__ __forceinline__ double fast_cos(double x) {
  double r, c, s;
  int k;
  trig_reduce(x, r, k);
  const double2 t = trig_entry(k);
  trig_poly(r, c, s);
  return fma(t.x, c, -(t.y * s));
}

__device__ __forceinline__ double fast_sin(double x) {
  double r, c, s;
  int k;
  trig_reduce(x, r, k);
  const double2 t = trig_entry(k);
  trig_poly(r, c, s);
  return fma(t.y, c, t.x * s);
}

#else
// Table-free variant: reduce by pi/2 (same FMA Cody-Waite), evaluate the
// fdlibm __kernel_sin / __kernel_cos minimax polynomials on [-pi/4, pi/4]
// (< 1 ulp) as two independent chains and select by quadrant.
__device__ __forceinline__ void quad_reduce(double x, double& r, int& q) {
  const double kShifter = 6755399441055744.0;
  const double t = fma(x, 0.63661977236758134308, kShifter);   // 2/pi
  q = __double2loint(t);
  const double n = t - kShifter;
  r = fma(-n, 1.5707963267948965580e+00, x);
  r = fma(-n, 6.1232339957367658e-17, r);
  r = fma(-n, -1.4973849048591698e-33, r);
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
  quad_reduce(x, r, q);
  const double s = k_sin(r), c = k_cos(r);
  const double v = (q & 1) ? s : c;
  return ((q + 1) & 2) ? -v : v;      // q = 1: -sin, 2: -cos, 3: sin
}

__device__ __forceinline__ double fast_sin(double x) {
  double r;
  int q;
  quad_reduce(x, r, q);
  const double s = k_sin(r), c = k_cos(r);
  const double v = (q & 1) ? c : s;
  return (q & 2) ? -v : v;            // q = 1: cos, 2: -sin, 3: -cos
}
#endif


// float32 sin/cos for the float path: exact reduction in double (arguments
// reach ~5e10 in Weierstrass), then single-precision minimax polynomials on
// [-pi/4, pi/4] (cephes sinf/cosf coefficients, < 1 ulp), so most of the
// work runs on the FP32 pipe.  Result within ~1-2 ulp of the correctly
// rounded value, like NumPy's own float32 SIMD sin/cos.
#ifndef RB_F32_POLY
#define RB_F32_POLY 1
#endif

__device__ __forceinline__ void quad_reduce_f(float x, float& r, int& q) {
  const double kShifter = 6755399441055744.0;
  const double xd = (double)x;
  const double t = fma(xd, 0.63661977236758134308, kShifter);
  q = __double2loint(t);
  const double n = t - kShifter;
  double rd = fma(-n, 1.5707963267948965580e+00, xd);
  rd = fma(-n, 6.1232339957367658e-17, rd);
  r = (float)rd;
}

__device__ __forceinline__ float k_sinf(float r) {
  const float z = r * r;
  float p = fmaf(z, -1.9515295891e-4f, 8.3321608736e-3f);
  p = fmaf(z, p, -1.6666654611e-1f);
  return fmaf(z * r, p, r);
}

__device__ __forceinline__ float k_cosf(float r) {
  const float z = r * r;
  float p = fmaf(z, 2.443315711809948e-5f, -1.388731625493765e-3f);
  p = fmaf(z, p, 4.166664568298827e-2f);
  return fmaf(z * z, p, fmaf(z, -0.5f, 1.0f));
}

__device__ __forceinline__ float fast_cosf(float x) {
  float r;
  int q;
  quad_reduce_f(x, r, q);
  const float s = k_sinf(r), c = k_cosf(r);
  const float v = (q & 1) ? s : c;
  return ((q + 1) & 2) ? -v : v;
}

__device__ __forceinline__ float fast_sinf(float x) {
  float r;
  int q;
  quad_reduce_f(x, r, q);
  const float s = k_sinf(r), c = k_cosf(r);
  const float v = (q & 1) ? c : s;
  return (q & 2) ? -v : v;
}

}  // namespace rb
