// Precision-generic math and the NumPy-order reductions used by every kernel.
//
// Build flags (see build.py): -fmad=false so no a*b+c in this code is ever
// contracted into an FMA — NumPy rounds every product —
// and IEEE division / square root (no fast-math).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rb_svml_powf.cuh"
#include "rb_trig.cuh"

#define RB_FULL 0xffffffffu

namespace rb {

// ---------------------------------------------------------------- math
// float64: CUDA's double libm (<= 2 ulp), sin/cos through rb_trig.cuh (no
// Payne-Hanek slow path).  float32: evaluated in double and rounded once,
// i.e. (almost always) the correctly rounded float result; NumPy's float32
// SIMD transcendentals are within ~1-2 ulp of that (DESIGN.md "float32
// transcendentals").
template <class T> struct M;

template <> struct M<double> {
  static __device__ __forceinline__ double cos(double x) { return fast_cos(x); }
  static __device__ __forceinline__ double sin(double x) { return fast_sin(x); }
  static __device__ __forceinline__ double exp(double x) { return ::exp(x); }
  static __device__ __forceinline__ double log(double x) { return ::log(x); }
  static __device__ __forceinline__ double expm1(double x) { return ::expm1(x); }
  static __device__ __forceinline__ double pow(double x, double y) { return ::pow(x, y); }
  static __device__ __forceinline__ double sqrt(double x) { return ::sqrt(x); }
  static __device__ __forceinline__ double floor(double x) { return ::floor(x); }
  static __device__ __forceinline__ double fabs(double x) { return ::fabs(x); }
  static __device__ __forceinline__ double fmod(double x, double y) { return ::fmod(x, y); }
  static __device__ __forceinline__ double trunc(double x) { return ::trunc(x); }
  static __device__ __forceinline__ double rint(double x) { return ::rint(x); }
  static __device__ __forceinline__ double fma(double a, double b, double c) { return ::fma(a, b, c); }
  static __device__ __forceinline__ bool finite(double x) { return isfinite(x); }
};

template <> struct M<float> {
#if RB_F32_POLY
  static __device__ __forceinline__ float cos(float x) { return fast_cosf(x); }
  static __device__ __forceinline__ float sin(float x) { return fast_sinf(x); }
#else
  static __device__ __forceinline__ float cos(float x) { return (float)fast_cos((double)x); }
  static __device__ __forceinline__ float sin(float x) { return (float)fast_sin((double)x); }
#endif
  static __device__ __forceinline__ float exp(float x) { return (float)::exp((double)x); }
  static __device__ __forceinline__ float log(float x) { return (float)::log((double)x); }
  static __device__ __forceinline__ float expm1(float x) { return (float)::expm1((double)x); }
  static __device__ __forceinline__ float pow(float x, float y) {
    return (float)::pow((double)x, (double)y);
  }
  static __device__ __forceinline__ float sqrt(float x) { return ::sqrtf(x); }
  static __device__ __forceinline__ float floor(float x) { return ::floorf(x); }
  static __device__ __forceinline__ float fabs(float x) { return ::fabsf(x); }
  static __device__ __forceinline__ float fmod(float x, float y) { return ::fmodf(x, y); }
  static __device__ __forceinline__ float trunc(float x) { return ::truncf(x); }
  static __device__ __forceinline__ float rint(float x) { return ::rintf(x); }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return ::fmaf(a, b, c); }
  static __device__ __forceinline__ bool finite(float x) { return isfinite(x); }
};

// Array power ``a ** b`` on NumPy arrays: float64 -> libm-class pow;
// float32 -> the bit-exact restatement of NumPy's SVML powf
// (rb_svml_powf.cuh).  Scalar powers (np.float32 ** float) go through libm
// powf in NumPy and use M<T>::pow here.
template <class T> __device__ __forceinline__ T apow(T a, T b);
// float64 to tolerance: exp(b log a) (|b log a| <= ~20 on the paths that use
// it: powers, SchaffersF7 -> relative error ~1e-15), a = 0 -> 0 for b > 0
template <> __device__ __forceinline__ double apow<double>(double a, double b) {
  return ::exp(b * ::log(a));
}
template <> __device__ __forceinline__ float apow<float>(float a, float b) { return rb_svml::powf_np(a, b); }

// Python-double constant as NumPy casts it into the working dtype (NEP 50:
// the weak Python float is rounded once to T).
template <class T> __device__ __forceinline__ T C(double v) { return static_cast<T>(v); }

// ------------------------------------------------------- 8-lane pairwise sum
// A point is owned by 8 consecutive lanes (l8 = lane & 7).  pw8 returns, in
// all 8 lanes, NumPy's float sum of f(lo), ..., f(lo+n-1) with NumPy's exact
// association (umath pairwise sum):
//   n < 8     : ((0 + a0) + a1) + ...
//   8..128    : 8 strided accumulators r_k over a[k], a[k+8], ... below the
//               last multiple of 8, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//               then the tail added in order
//   > 128     : pw(first m) + pw(rest), m = n/2 rounded down to a multiple of 8
// Lane k is accumulator r_k; the combine is the xor butterfly 1, 2, 4.
// f is called once per element, by the lane that owns it.
#ifndef RB_LEAF_UNROLL
#define RB_LEAF_UNROLL 4               // A/B: 2 -> 4 +1-2 % on float32 basic functions (same summation order)
#endif
constexpr int kLeafUnroll = RB_LEAF_UNROLL;   // independent kernel terms in flight per lane

template <class T, class F>
__device__ __forceinline__ T pw8_leaf(int lo, int n, F& f, int l8) {
  T r = T(0);
  const int main_len = n < 8 ? 0 : n - (n & 7);
  if (main_len) {
#pragma unroll kLeafUnroll
    for (int i = l8; i < main_len; i += 8) r = r + f(lo + i);
    r = r + __shfl_xor_sync(RB_FULL, r, 1, 8);
    r = r + __shfl_xor_sync(RB_FULL, r, 2, 8);
    r = r + __shfl_xor_sync(RB_FULL, r, 4, 8);
  }
  const int tail = n - main_len;
  if (tail) {
    const T v = (l8 < tail) ? f(lo + main_len + l8) : T(0);
    for (int k = 0; k < tail; ++k) r = r + __shfl_sync(RB_FULL, v, k, 8);
  }
  return r;
}

// n > 128: NumPy splits recursively, pw(a, n) = pw(a, m) + pw(a + m, n - m)
// with m = n/2 rounded down to a multiple of 8.  Iterative post-order walk
// (no device recursion: its stack frames overflowed once the leaf loop was
// unrolled); every lane of the group walks the same tree.
template <class T, class F>
__device__ __noinline__ T pw8_tree(int lo, int n, F& f, int l8) {
  constexpr int kDepth = 24;                 // n < 128 * 2^23
  int s_lo[kDepth], s_n[kDepth], s_stage[kDepth];
  T s_left[kDepth];
  int sp = 0;
  s_lo[0] = lo;
  s_n[0] = n;
  s_stage[0] = 0;
  T val = T(0);
  bool have = false;                         // `val` holds a finished subtree
  while (sp >= 0) {
    const int cl = s_lo[sp], cn = s_n[sp];
    if (have) {                              // a child finished
      if (s_stage[sp] == 1) {                // left child: descend right
        s_left[sp] = val;
        s_stage[sp] = 2;
        int m = cn >> 1;
        m -= m & 7;
        ++sp;
        s_lo[sp] = cl + m;
        s_n[sp] = cn - m;
        s_stage[sp] = 0;
        have = false;
      } else {                               // right child: combine, pop
        val = s_left[sp] + val;
        --sp;
      }
      continue;
    }
    if (cn <= 128) {                         // leaf
      val = pw8_leaf<T>(cl, cn, f, l8);
      have = true;
      --sp;
      continue;
    }
    int m = cn >> 1;                         // descend left
    m -= m & 7;
    s_stage[sp] = 1;
    ++sp;
    s_lo[sp] = cl;
    s_n[sp] = m;
    s_stage[sp] = 0;
  }
  return val;
}

// float64 sums: the bar is 1e-12 relative, not NumPy's bits, so each lane
// keeps two independent partial sums (ILP) over its strided elements and
// the 8 lane partials meet in an xor butterfly.  The order is fixed per
// point (bit-identical across batches and tiles).
template <class F>
__device__ __forceinline__ double sum8_f64(int lo, int n, F& f, int l8) {
  double r0 = 0.0, r1 = 0.0;
  int i = l8;
#pragma unroll 2
  for (; i + 8 < n; i += 16) {
    r0 = r0 + f(lo + i);
    r1 = r1 + f(lo + i + 8);
  }
  if (i < n) r0 = r0 + f(lo + i);
  double r = r0 + r1;
  r = r + __shfl_xor_sync(RB_FULL, r, 1, 8);
  r = r + __shfl_xor_sync(RB_FULL, r, 2, 8);
  r = r + __shfl_xor_sync(RB_FULL, r, 4, 8);
  return r;
}

template <class T, class F>
__device__ __forceinline__ T pw8(int lo, int n, F&& f, int l8) {
  if constexpr (sizeof(T) == 8) {
    return sum8_f64(lo, n, f, l8);
  } else {
    if (n <= 128) return pw8_leaf<T>(lo, n, f, l8);
    return pw8_tree<T>(lo, n, f, l8);
  }
}

// NumPy's pairwise order in either precision (float64 HappyCat / HGBat:
// their sums feed a non-differentiable residual, exact64_kernel).
template <class T, class F>
__device__ __forceinline__ T pw8_np(int lo, int n, F&& f, int l8) {
  if (n <= 128) return pw8_leaf<T>(lo, n, f, l8);
  return pw8_tree<T>(lo, n, f, l8);
}

// Sequential product over i = 0..n-1 of f(i) (np.prod is a plain left fold,
// kernels.py:112); lane l8 evaluates the i = l8 (mod 8) factors.  float64
// multiplies lane partials instead (order-free to its tolerance).
// float32 np.prod without a shuffle chain: every lane writes its factors
// over its own elements of the point's z row (each element is read and
// rewritten by the same lane, and z is dead after the product), then lane 0
// folds the row left to right and broadcasts.  ``scratch`` = the z row.
template <class T, class F>
__device__ __forceinline__ T prod8_fold(int n, F&& f, int l8, T* scratch) {
  for (int i = l8; i < n; i += 8) scratch[i] = f(i);
  __syncwarp();
  T p = T(1);
  if (l8 == 0)
    for (int i = 0; i < n; ++i) p = p * scratch[i];
  return __shfl_sync(RB_FULL, p, 0, 8);
}

template <class T, class F>
__device__ __forceinline__ T prod8(int n, F&& f, int l8) {
  if constexpr (sizeof(T) == 8) {        // float64: lane partial products, butterfly
    double q = 1.0;
    for (int i = l8; i < n; i += 8) q = q * f(i);
    q = q * __shfl_xor_sync(RB_FULL, q, 1, 8);
    q = q * __shfl_xor_sync(RB_FULL, q, 2, 8);
    q = q * __shfl_xor_sync(RB_FULL, q, 4, 8);
    return q;
  }
  T p = T(1);
  for (int base = 0; base < n; base += 8) {
    const int cnt = min(8, n - base);
    const T v = (l8 < cnt) ? f(base + l8) : T(1);
    for (int k = 0; k < cnt; ++k) p = p * __shfl_sync(RB_FULL, v, k, 8);
  }
  return p;
}

}  // namespace rb
