// The 21 basic kernels, evaluated cooperatively by the 8 lanes that own one
// point.  z is that point's transformed vector (length d) in shared memory.
//
// Each body restates the reference expression (line numbers below are
// /root/reference/pkg/src/robench/kernels.py) with NumPy's evaluation order:
// left-to-right binary ops, every product/sum individually rounded, Python
// float constants rounded once into T, ``x**2`` on arrays = x*x, array
// powers through apow (NumPy's SVML powf in float32), sums in the pairwise
// order of rb::pw8, np.prod as a left fold.
//
// kernel_value_k<T, K> is the compile-time specialisation used by the
// per-function kernels; kernel_value<T>(k, ...) dispatches at run time for
// hybrids and compositions.
#pragma once
#include "rb_math.cuh"

namespace rb {

enum Kernel : int {
  K_SPHERE = 0, K_ELLIPSOID, K_ELLIPTIC, K_DISCUS, K_CIGAR, K_POWERS, K_SHARP_VALLEY,
  K_STEP, K_WEIERSTRASS, K_GRIEWANK, K_RASTRIGIN, K_SCHAFFERS_F7, K_GRIE_ROSEN,
  K_ROSENBROCK, K_SCHWEFEL, K_KATSUURA, K_LUNACEK, K_ACKLEY, K_HAPPYCAT, K_HGBAT,
  K_SCHAFFERS_F6, K_COUNT
};

constexpr double kTwoPi = 6.283185307179586;   // 2.0 * np.pi, folded by Python
constexpr double kE = 2.718281828459045;       // np.e

template <class T>
struct Pt {            // one point's view for the kernels
  const T* z;          // shared memory, length d
  int d;
  int l8;
  const T* ctab;       // per-(kernel, d) NumPy-computed constants (pack.py)
  bool* ill = nullptr; // float64 HappyCat / HGBat: set when the value needs the
                       // exact-order z (rb_device.cuh exact64_kernel)
};

// float64 HappyCat / HGBat next to the non-differentiable residual: the
// DMMA z is a few ulps (of its terms) off NumPy's, so the value keeps the
// parity bar only while the residual is not small against its terms.  Both
// values carry +100 (bar = 1e-12 of it, ~1e-10 absolute); r2's error is
// ~eps * S and the HGBat product's ~eps * U, so |r2 - d| >= S / 10 keeps
// HappyCat's pow within ~eps * S^0.25 and |r2^2 - sz^2| >= U / 10 keeps
// HGBat's sqrt within ~5 eps relative.  Random points in the search box
// have |r2 - d| ~ 17 d; points near an optimum are marked and re-evaluated
// in exact order (fixup_kernel).
template <class T> __device__ __forceinline__ void mark_ill(const Pt<T>& P, bool cond) {
  if (sizeof(T) == 8 && P.ill != nullptr) *P.ill = *P.ill || cond;
}

template <class T> __device__ __forceinline__ T sq(T a) { return a * a; }

// rosenbrock_pair (:130-132): 100*(x*x - y)**2 + (x - 1)**2
template <class T> __device__ __forceinline__ T rosen_link(T x, T y) {
  return C<T>(100.0) * sq(x * x - y) + sq(x - C<T>(1.0));
}
// griewank_1d (:135-137): x*x/4000 - cos(x) + 1
template <class T> __device__ __forceinline__ T griewank_1d(T x) {
  return (x * x / C<T>(4000.0) - M<T>::cos(x)) + C<T>(1.0);
}
// schaffer_f6_pair (:220-223)
template <class T> __device__ __forceinline__ T f6_link(T x, T y) {
  const T q = x * x + y * y;
  return (sq(M<T>::sin(M<T>::sqrt(q))) - C<T>(0.5)) / sq(C<T>(1.0) + C<T>(0.001) * q) + C<T>(0.5);
}
// np.mod(u, 500) for u > 0 (floored == truncated for positive operands):
// q = trunc(u / 500) corrected by one step, then u - 500 q is exact
// (Sterbenz: 500 q lies within [u/2, u]).  Huge u keeps libm's fmod.
template <class T> __device__ __forceinline__ T mod500(T u) {
  const T big = sizeof(T) == 8 ? T(1099511627776.0) : T(1048576.0);   // 2^40 / 2^20
  if (!(u < big)) return M<T>::fmod(u, C<T>(500.0));
  T q = M<T>::trunc(u * C<T>(0.002));
  T r = M<T>::fma(C<T>(-500.0), q, u);
  if (r < T(0)) {
    q = q - T(1);
    r = M<T>::fma(C<T>(-500.0), q, u);
  } else if (r >= C<T>(500.0)) {
    q = q + T(1);
    r = M<T>::fma(C<T>(-500.0), q, u);
  }
  return r;
}
// schwefel_g1 (:152-165): the branch np.where selects, evaluated once: every
// branch is "mult * sin(sqrt(arg)) - pen" with the reference's own operands
//   |w| <= 500: w * sin(sqrt(|w|))
//   w > 500:    top * sin(sqrt(top)) - (w - 500)**2 / (10000 d),   top = 500 - mod(w, 500)
//   w < -500:   (rem - 500) * sin(sqrt(500 - rem)) - (w + 500)**2 / (10000 d),
//               rem = mod(-w, 500)
// so a warp runs one sin and one sqrt per element whatever the branch mix.
template <class T> __device__ __forceinline__ T schwefel_g1(T w, T c10000d) {
  const T aw = M<T>::fabs(w);
  const T r = mod500(aw);                              // mod(w) or mod(-w), |w| > 500
  const bool mid = aw <= C<T>(500.0);
  const bool high = w > C<T>(500.0);
  const T arg = mid ? aw : C<T>(500.0) - r;            // top == 500 - rem
  const T mult = mid ? w : (high ? arg : r - C<T>(500.0));
  const T e = high ? w - C<T>(500.0) : w + C<T>(500.0);
  const T pen = mid ? T(0) : sq(e) / c10000d;
  const T v = mult * M<T>::sin(M<T>::sqrt(arg));
  return mid ? v : v - pen;
}
// katsuura row sum over i = 1..32 (:178-180) for one coordinate: 8
// accumulators in NumPy order (32 is a multiple of 8: no tail)
template <class T> __device__ __forceinline__ T katsuura_row(T zj) {
  T r[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) r[a] = T(0);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const T p2 = T(1ull << (i + 1));  // 2**(i+1), exact
    const T w = p2 * zj;
    // floor(w + 0.5) exactly as the reference rounds it (w + 0.5 itself
    // rounds for |w| >= 2^52 / 2^23).  d * 2**-(i+1) is an exact scaling, so
    // the FMA rounds the sum exactly like "/ 2**(i+1)" followed by "+".
    const T d = M<T>::fabs(w - M<T>::floor(w + C<T>(0.5)));
    r[i & 7] = M<T>::fma(d, T(1.0 / double(1ull << (i + 1))), r[i & 7]);
  }
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

// Weierstrass series constants a_k = 0.5**k and c_k = 2.0*np.pi*3.0**k
// (kernels.py:100-104), as NumPy computed them in each dtype (pack.py),
// mirrored into __constant__ memory by rb_initialize so the unrolled k loop
// reads them as constant-bank operands.
template <class T> struct WeierTab { T a[21]; T c[21]; };
#ifndef RB_WEI_UNROLL
#define RB_WEI_UNROLL 7
#endif
constexpr int kWeiUnroll = RB_WEI_UNROLL;   // series terms unrolled per pass (register budget)
#ifndef RB_WEI_UNROLL_F32
#define RB_WEI_UNROLL_F32 21          // float: all 21 terms (c_k as constant-bank operands): +3-4 %
#endif
constexpr int kWeiUnrollF32 = RB_WEI_UNROLL_F32;
static __constant__ WeierTab<double> kWei64;
static __constant__ WeierTab<float> kWei32;
template <class T> __device__ __forceinline__ const WeierTab<T>& wei_tab();
template <> __device__ __forceinline__ const WeierTab<double>& wei_tab<double>() { return kWei64; }
template <> __device__ __forceinline__ const WeierTab<float>& wei_tab<float>() { return kWei32; }

// sum_k a_k cos(c_k (zj + 0.5)) for one coordinate; c_k * w is the
// reference's individually rounded product, cos is evaluated of exactly it.
template <class T> static __device__ __noinline__ T weier_coord_big(T w, const WeierTab<T>& W) {
  T s = T(0);
  for (int k = 0; k < 21; ++k) s = s + W.a[k] * M<T>::cos(W.c[k] * w);
  return s;
}
template <class T> __device__ __forceinline__ T weier_coord(T zj, const WeierTab<T>& W);
template <> __device__ __forceinline__ double weier_coord<double>(double zj, const WeierTab<double>& W) {
  const double w = zj + 0.5;
  if (!(fabs(w) * W.c[20] < kTrigBig)) return weier_coord_big<double>(w, W);
  double s = 0.0;
#pragma unroll kWeiUnroll
  for (int k = 0; k < 21; ++k) {
    const double x = W.c[k] * w;
    int q;
    const double r = trig_reduce_pi(x, q);
    s = fma(W.a[k], flip_sign(cos_poly6(r * r), q), s);
  }
  return s;
}
template <> __device__ __forceinline__ float weier_coord<float>(float zj, const WeierTab<float>& W) {
  const float w = zj + 0.5f;
  if (!(fabsf(w) * W.c[20] < (float)kTrigBig)) return weier_coord_big<float>(w, W);
  // sum_k 2^-k cos_k as a Horner chain from k = 20 down (a_k = 0.5^k, so
  // s * 0.5 is exact): no a_k loads in the loop
  float s = 0.0f;
#pragma unroll kWeiUnrollF32
  for (int k = 20; k >= 0; --k) {
    const float x = W.c[k] * w;
    int q;
    const float r = trig_reduce_pi_f(x, q);
    s = fmaf(s, 0.5f, flip_sign(cos_polyf(r * r), q));
  }
  return s;
}

// NP (float64 only; float32 sums are always in NumPy's order): HappyCat /
// HGBat sum in NumPy's pairwise order -- the exact-order re-evaluation
// (fixup_kernel), where z carries NumPy's bits and r2, sz must too.
template <class T, int K, bool NP = false>
__device__ __forceinline__ T kernel_value_k(const Pt<T>& P) {
  const T* z = P.z;
  const int d = P.d, l8 = P.l8;
  auto square = [&](int i) { const T a = z[i]; return a * a; };
  if constexpr (K == K_SPHERE) {                                      // :52-54
    return pw8<T>(0, d, square, l8);
  } else if constexpr (K == K_ELLIPSOID) {                            // :57-60
    return pw8<T>(0, d, [&](int i) { const T a = z[i]; return T(i + 1) * a * a; }, l8);
  } else if constexpr (K == K_ELLIPTIC) {                             // :63-67
    const T* c = P.ctab;
    return pw8<T>(0, d, [&](int i) { const T a = z[i]; return c[i] * a * a; }, l8);
  } else if constexpr (K == K_DISCUS) {                               // :70-72
    const T rest = pw8<T>(1, d - 1, square, l8);
    return C<T>(1.0e6) * z[0] * z[0] + rest;
  } else if constexpr (K == K_CIGAR) {                                // :75-77
    const T rest = pw8<T>(1, d - 1, square, l8);
    return z[0] * z[0] + C<T>(1.0e6) * rest;
  } else if constexpr (K == K_POWERS) {                               // :80-84
    const T* e = P.ctab;
    return M<T>::sqrt(pw8<T>(0, d, [&](int i) { return apow<T>(M<T>::fabs(z[i]), e[i]); }, l8));
  } else if constexpr (K == K_SHARP_VALLEY) {                         // :87-89
    const T rest = pw8<T>(1, d - 1, square, l8);
    return z[0] * z[0] + C<T>(100.0) * M<T>::sqrt(rest);
  } else if constexpr (K == K_STEP) {                                 // :92-95
    return pw8<T>(0, d, [&](int i) { const T r = M<T>::floor(z[i] + C<T>(0.5)); return r * r; }, l8);
  } else if constexpr (K == K_WEIERSTRASS) {                          // :98-106
    // Per coordinate j (lane j mod 8) the 21 terms in k order, then the
    // 8 lane partials by butterfly: a fixed order per point (bit-identical
    // across batches), not NumPy's pairwise order over the flattened
    // (d, 21) grid -- the terms are bounded by a_k and sum to O(d), so the
    // reordering moves the value by ~1e-16 (fp64) / ~1e-8 (fp32) relative,
    // far inside the parity bars.
    const WeierTab<T>& W = wei_tab<T>();
    T acc = T(0);
    for (int j = l8; j < d; j += 8) acc = acc + weier_coord<T>(z[j], W);
    acc = acc + __shfl_xor_sync(RB_FULL, acc, 1, 8);
    acc = acc + __shfl_xor_sync(RB_FULL, acc, 2, 8);
    acc = acc + __shfl_xor_sync(RB_FULL, acc, 4, 8);
    return acc - P.ctab[42];
  } else if constexpr (K == K_GRIEWANK) {                             // :109-112
    // ctab: float32 np.sqrt(arange(1, d+1)) (divided by, as the reference);
    // float64 its reciprocal (multiplied by, to tolerance) -- pack.py
    const T* sq_i = P.ctab;
    const T s = pw8<T>(0, d, square, l8);
    auto factor = [&](int i) {
      return M<T>::cos(sizeof(T) == 8 ? z[i] * sq_i[i] : z[i] / sq_i[i]);
    };
    // fp32: the left fold of np.prod through shared memory (the sum above
    // has read z already); fp64: lane partial products
    const T p = sizeof(T) == 4 ? prod8_fold<T>(d, factor, l8, const_cast<T*>(z))
                               : prod8<T>(d, factor, l8);
    return (s / C<T>(4000.0) - p) + C<T>(1.0);
  } else if constexpr (K == K_RASTRIGIN) {                            // :115-117
    return pw8<T>(0, d, [&](int i) {
      const T a = z[i];
      return (a * a - C<T>(10.0) * M<T>::cos(C<T>(kTwoPi) * a)) + C<T>(10.0);
    }, l8);
  } else if constexpr (K == K_SCHAFFERS_F7) {                         // :120-127
    if (d < 2) return T(0);
    const T s = pw8<T>(0, d - 1, [&](int i) {
      const T w = M<T>::sqrt(sq(z[i]) + sq(z[i + 1]));
      return M<T>::sqrt(w) * (C<T>(1.0) + sq(M<T>::sin(C<T>(50.0) * apow<T>(w, C<T>(0.2)))));
    }, l8);
    return sq(s / T(d - 1));
  } else if constexpr (K == K_GRIE_ROSEN) {                           // :140-142
    return pw8<T>(0, d, [&](int i) {
      const int n = (i + 1 == d) ? 0 : i + 1;
      return griewank_1d(rosen_link(z[i], z[n]));
    }, l8);
  } else if constexpr (K == K_ROSENBROCK) {                           // :145-149
    return pw8<T>(0, d - 1, [&](int i) { return rosen_link(z[i], z[i + 1]); }, l8);
  } else if constexpr (K == K_SCHWEFEL) {                             // :168-171
    const T c10000d = C<T>(10000.0 * d);
    const T s = pw8<T>(0, d, [&](int i) {
      return schwefel_g1(z[i] + C<T>(420.9687462275036), c10000d);
    }, l8);
    return C<T>(418.9829 * d) - s;
  } else if constexpr (K == K_KATSUURA) {                             // :174-184
    auto logt = [&](int j) { return M<T>::log(C<T>(1.0) + T(j + 1) * katsuura_row(z[j])); };
    const T lp = P.ctab[0] * pw8<T>(0, d, logt, l8);
    return P.ctab[1] * M<T>::expm1(lp);
  } else if constexpr (K == K_LUNACEK) {                              // :187-193
    const T s1 = pw8<T>(0, d, [&](int i) { const T a = z[i] - C<T>(2.5); return a * a; }, l8);
    const T s2 = pw8<T>(0, d, [&](int i) { const T b = z[i] - C<T>(-2.5); return b * b; }, l8);
    const T cs = pw8<T>(0, d, [&](int i) {
      return M<T>::cos(C<T>(kTwoPi) * (z[i] - C<T>(2.5)));
    }, l8);
    const T alt = C<T>(1.0 * d) + C<T>(0.9) * s2;
    const T funnel = (alt < s1) ? alt : s1;   // np.minimum (finite operands)
    return funnel + C<T>(10.0) * (T(d) - cs);
  } else if constexpr (K == K_ACKLEY) {                               // :196-201
    const T s = pw8<T>(0, d, square, l8);
    const T cs = pw8<T>(0, d, [&](int i) { return M<T>::cos(C<T>(kTwoPi) * z[i]); }, l8);
    const T rms = M<T>::sqrt(s / T(d));
    const T mc = cs / T(d);
    return ((C<T>(-20.0) * M<T>::exp(C<T>(-0.2) * rms) - M<T>::exp(mc)) + C<T>(20.0)) + C<T>(kE);
  } else if constexpr (K == K_HAPPYCAT) {                             // :204-209
    // NP: NumPy-order sums, so with the exact-order z r2 and sz carry the
    // reference's bits (rb_device.cuh exact64_kernel)
    const T r2 = NP ? pw8_np<T>(0, d, square, l8) : pw8<T>(0, d, square, l8);
    const T sz = NP ? pw8_np<T>(0, d, [&](int i) { return z[i]; }, l8)
                    : pw8<T>(0, d, [&](int i) { return z[i]; }, l8);
    const T S = r2 + T(d);
    mark_ill(P, isfinite(S) && !(M<T>::fabs(r2 - T(d)) >= T(0.1) * S));
    return (M<T>::pow(M<T>::fabs(r2 - T(d)), C<T>(0.25)) + (C<T>(0.5) * r2 + sz) / T(d)) +
           C<T>(0.5);
  } else if constexpr (K == K_HGBAT) {                                // :212-217
    const T r2 = NP ? pw8_np<T>(0, d, square, l8) : pw8<T>(0, d, square, l8);
    const T sz = NP ? pw8_np<T>(0, d, [&](int i) { return z[i]; }, l8)
                    : pw8<T>(0, d, [&](int i) { return z[i]; }, l8);
    const T U = r2 * r2 + sz * sz;
    mark_ill(P, isfinite(U) && !(M<T>::fabs(r2 * r2 - sz * sz) >= T(0.1) * U));
    return (M<T>::sqrt(M<T>::fabs(r2 * r2 - sz * sz)) + (C<T>(0.5) * r2 + sz) / T(d)) +
           C<T>(0.5);
  } else if constexpr (K == K_SCHAFFERS_F6) {                         // :226-228
    return pw8<T>(0, d, [&](int i) {
      const int n = (i + 1 == d) ? 0 : i + 1;
      return f6_link(z[i], z[n]);
    }, l8);
  } else {
    return T(0);
  }
}

template <class T, bool NP = false>
__device__ T kernel_value(int k, const Pt<T>& P) {
  switch (k) {
#define RB_CASE(K) \
  case K: return kernel_value_k<T, K, NP>(P);
    RB_CASE(K_SPHERE) RB_CASE(K_ELLIPSOID) RB_CASE(K_ELLIPTIC) RB_CASE(K_DISCUS)
    RB_CASE(K_CIGAR) RB_CASE(K_POWERS) RB_CASE(K_SHARP_VALLEY) RB_CASE(K_STEP)
    RB_CASE(K_WEIERSTRASS) RB_CASE(K_GRIEWANK) RB_CASE(K_RASTRIGIN) RB_CASE(K_SCHAFFERS_F7)
    RB_CASE(K_GRIE_ROSEN) RB_CASE(K_ROSENBROCK) RB_CASE(K_SCHWEFEL) RB_CASE(K_KATSUURA)
    RB_CASE(K_LUNACEK) RB_CASE(K_ACKLEY) RB_CASE(K_HAPPYCAT) RB_CASE(K_HGBAT)
    RB_CASE(K_SCHAFFERS_F6)
#undef RB_CASE
    default: return T(0);
  }
}

}  // namespace rb
