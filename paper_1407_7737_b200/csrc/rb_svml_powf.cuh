// Bit-exact restatement of NumPy's float32 array power.
//
// NumPy >= 1.22 on x86-64 with AVX512_SKX evaluates float32 ``np.power`` on
// (loadable-stride) arrays with its bundled Intel SVML routine
// ``__svml_powf16`` (numpy/_core/src/umath/loops_umath_fp.dispatch.c.src,
// "la" variant; NumPy 2.3.5 in this image).  The reference hits it in
// ``w**0.2`` (kernels.py:125), ``np.abs(z) ** expo`` (kernels.py:84) and
// ``d2**-0.5`` (composition.py:136).  Its result differs from the correctly
// rounded power by 1 ulp for ~20-36 % of inputs, and SCHAFFERSF7 amplifies a
// 1-ulp change of w**0.2 by ~25x through sin(50 w^0.2), which alone breaks a
// 1e-5 float32 tolerance at small d.  So the
// float32 path replays the routine's main path operation by operation:
//
//   log2 stage: x = m * 2^(e+1), m in [1/2, 1) (vgetmantps/vgetexpps);
//     r = RNE_{1/32}(rcp14(m)) in [1, 2] (vrcp14ps + vrndscaleps) — rcp14 is
//     implementation defined, but after rounding to the 1/32 grid it is a
//     step function of m with the 33 breakpoints below (brute-forced over all
//     2^23 mantissas on this CPU family, tools/svml/rcp_breaks.c);
//     t = r*m - 1; log2 x = (e + [r<1.5] + Lhi[r]) + t/ln2 + poly(t)*t + Llo[r]
//     as a hi/lo pair (fma-based error terms);
//   product: Q = y * log2 x in round-toward-zero with its low part;
//   exp2 stage: Q = n + j/16 + f, 2^Q = 2^n * T[j] * (1 + f*(ln2 + f*(c2 + f*c3))).
// Every step uses the rounding mode of the original instruction (rn/rz/rd),
// which CUDA exposes as __fmaf_r?, __fadd_r?, __fmul_r?.
//
// The routine's rare-lane callout (x <= 0, x or y non-finite, |Q| > 125.5)
// is not replayed: +0 is handled exactly, anything else falls back to the
// double-precision power rounded to float (never reached by the suite's
// inputs except |z| < ~1e-6 in POWERS, whose terms are below 1e-37).
//
// Verified bit-for-bit against np.power on the host by tools/svml/verify.py
// (CPU build of this header) and on the GPU by tests/test_svml_gpu.py.
#pragma once
#include <stdint.h>
#if !defined(__CUDACC__)
#include <immintrin.h>
#include <math.h>
#include <string.h>
#endif

#if defined(__CUDACC__)
// global (L1-cached) rather than __constant__: the lookups are indexed by
// each lane's own mantissa bits, and divergent constant-bank reads serialise
#define RB_SVML_TAB static __device__ const
#else
#define RB_SVML_TAB static const
#endif

namespace rb_svml {

// __svml_spow_data_internal_avx512 (value tables, as float bit patterns)
#define RB_SVML_TABLES                                                                          \
  RB_SVML_TAB uint32_t kLhi[32] = {                                                            \
      0x00000000u, 0xbd35d000u, 0xbdb32000u, 0xbe046400u, 0xbe2e0000u, 0xbe567c00u, 0xbe7de000u, \
      0xbe922000u, 0xbea4d400u, 0xbeb71200u, 0xbec8de00u, 0xbeda4000u, 0xbeeb3a00u, 0xbefbd400u, \
      0xbf060800u, 0xbf0dfa00u, 0x3ed48000u, 0x3ec54400u, 0x3eb65800u, 0x3ea7b800u, 0x3e996000u, \
      0x3e8b4e00u, 0x3e7b0000u, 0x3e5fe400u, 0x3e454400u, 0x3e2b2000u, 0x3e116c00u, 0x3df05800u, \
      0x3dbeb000u, 0x3d8dd800u, 0x3d3ba000u, 0x3cba2000u};                                      \
  RB_SVML_TAB uint32_t kLlo[32] = {                                                            \
      0x00000000u, 0xb6d3758fu, 0x3510536fu, 0x369dcc96u, 0xb651cfdfu, 0x3687492cu, 0xb635c813u, \
      0xb5f561c1u, 0x35f6865du, 0x36f19318u, 0x35aedc1du, 0x36a0463cu, 0xb69f0197u, 0xb5ad1961u, \
      0xb6201ac7u, 0x36ee16a3u, 0xb5d1cfdfu, 0x36c055feu, 0x3676865du, 0xb589a627u, 0xb48e4789u, \
      0x33a6c7e3u, 0xb69d5be7u, 0xb642c000u, 0x364055feu, 0xb68f5801u, 0x36b70aadu, 0x35d74798u, \
      0x3492d9f7u, 0x364a9801u, 0xb6566c4du, 0xb48bcf06u};                                      \
  RB_SVML_TAB uint32_t kExp2[16] = {                                                           \
      0x3f800000u, 0x3f85aac3u, 0x3f8b95c2u, 0x3f91c3d3u, 0x3f9837f0u, 0x3f9ef532u, 0x3fa5fed7u, \
      0x3fad583fu, 0x3fb504f3u, 0x3fbd08a4u, 0x3fc5672au, 0x3fce248cu, 0x3fd744fdu, 0x3fe0ccdfu, \
      0x3feac0c7u, 0x3ff5257du};                                                                \
  /* first m (bits) of each step of RNE_{1/32}(rcp14(m)), m in [1/2, 1) */                      \
  RB_SVML_TAB uint32_t kRcpBreak[33] = {                                                       \
      0x3f000000u, 0x3f010300u, 0x3f031380u, 0x3f053500u, 0x3f076800u, 0x3f09ae80u, 0x3f0c0780u, \
      0x3f0e7900u, 0x3f10fe80u, 0x3f139b00u, 0x3f164f80u, 0x3f192000u, 0x3f1c0900u, 0x3f1f1280u, \
      0x3f223700u, 0x3f257f00u, 0x3f28e900u, 0x3f2c7780u, 0x3f302b80u, 0x3f340b80u, 0x3f381680u, \
      0x3f3c5280u, 0x3f40c100u, 0x3f456680u, 0x3f4a4500u, 0x3f4f6580u, 0x3f54c780u, 0x3f5a7480u, \
      0x3f607000u, 0x3f66c400u, 0x3f6d7300u, 0x3f748a80u, 0x3f7c1180u};

RB_SVML_TABLES

// coefficients (same table, broadcast rows)
constexpr uint32_t kPa = 0x3e93c705u, kPb = 0xbeb8b3edu, kPc = 0x3ef6384fu, kPd = 0xbf38aa3bu,
                   kPlo = 0x32a570ccu, kInvLn2 = 0x3fb8aa3bu, kShifter = 0x494007f0u,
                   kE3 = 0x3d6854cbu, kE2 = 0x3e75f16cu, kLn2 = 0x3f317222u, kLimit = 0x42fb0000u;

// --- primitive ops with explicit rounding
#if defined(__CUDACC__)
__device__ __forceinline__ float fbits(uint32_t b) { return __uint_as_float(b); }
__device__ __forceinline__ uint32_t bitsf(float f) { return __float_as_uint(f); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float fma_rz(float a, float b, float c) { return __fmaf_rz(a, b, c); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float add_rz(float a, float b) { return __fadd_rz(a, b); }
__device__ __forceinline__ float add_rd(float a, float b) { return __fadd_rd(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float sub_rd(float a, float b) { return __fsub_rd(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float mul_rz(float a, float b) { return __fmul_rz(a, b); }
__device__ __forceinline__ float floor_(float a) { return floorf(a); }
__device__ __forceinline__ int clz32(uint32_t v) { return __clz(v); }
__device__ __forceinline__ float fallback_pow(float x, float y) { return (float)pow((double)x, (double)y); }
#define RB_SVML_DEV __device__ __forceinline__
#else
static inline float fbits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static inline uint32_t bitsf(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }
#define RB_R(op, mode, ...) _mm_cvtss_f32(op(__VA_ARGS__, mode | _MM_FROUND_NO_EXC))
static inline float fma_rn(float a, float b, float c) { return RB_R(_mm_fmadd_round_ss, _MM_FROUND_TO_NEAREST_INT, _mm_set_ss(a), _mm_set_ss(b), _mm_set_ss(c)); }
static inline float fma_rz(float a, float b, float c) { return RB_R(_mm_fmadd_round_ss, _MM_FROUND_TO_ZERO, _mm_set_ss(a), _mm_set_ss(b), _mm_set_ss(c)); }
static inline float add_rn(float a, float b) { return RB_R(_mm_add_round_ss, _MM_FROUND_TO_NEAREST_INT, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float add_rz(float a, float b) { return RB_R(_mm_add_round_ss, _MM_FROUND_TO_ZERO, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float add_rd(float a, float b) { return RB_R(_mm_add_round_ss, _MM_FROUND_TO_NEG_INF, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float sub_rn(float a, float b) { return RB_R(_mm_sub_round_ss, _MM_FROUND_TO_NEAREST_INT, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float sub_rd(float a, float b) { return RB_R(_mm_sub_round_ss, _MM_FROUND_TO_NEG_INF, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float mul_rn(float a, float b) { return RB_R(_mm_mul_round_ss, _MM_FROUND_TO_NEAREST_INT, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float mul_rz(float a, float b) { return RB_R(_mm_mul_round_ss, _MM_FROUND_TO_ZERO, _mm_set_ss(a), _mm_set_ss(b)); }
static inline float floor_(float a) { return floorf(a); }
static inline int clz32(uint32_t v) { return __builtin_clz(v); }
static inline float fallback_pow(float x, float y) { return (float)pow((double)x, (double)y); }
#define RB_SVML_DEV static inline
#endif

// __svml_powf16 main path for one lane.
RB_SVML_DEV float powf_np(float x, float y) {
  const uint32_t xb = bitsf(x);
  const uint32_t ay = bitsf(y) & 0x7fffffffu;
  if (xb == 0u) {                                   // +0: exact IEEE result
    if (ay == 0u) return 1.0f;
    return (bitsf(y) >> 31) ? fbits(0x7f800000u) : 0.0f;
  }
  if ((xb >> 31) || xb >= 0x7f800000u || ay >= 0x7f800000u) return fallback_pow(x, y);

  // vgetmantps [1/2,1) / vgetexpps (denormals normalised)
  uint32_t ex = (xb >> 23) & 0xffu, man = xb & 0x7fffffu;
  int e;
  if (ex == 0u) {
    const int sh = clz32(man) - 8;
    man = (man << sh) & 0x7fffffu;
    e = -126 - sh;
  } else {
    e = (int)ex - 127;
  }
  const float m = fbits(0x3f000000u | man);
  float ef = (float)e;

  // r = RNE_{1/32}(rcp14(m)) from the step breakpoints
  int k = 0;
#pragma unroll
  for (int step = 32; step >= 1; step >>= 1)
    if (k + step <= 32 && man >= (kRcpBreak[k + step] & 0x7fffffu)) k += step;
  const float r = 2.0f - (float)k * 0.03125f;

  const float t = fma_rn(r, m, -1.0f);
  float p = fma_rn(fbits(kPa), t, fbits(kPb));
  const uint32_t idx = (bitsf(r) >> 18) & 31u;
  p = fma_rn(p, t, fbits(kPc));
  if (r < 1.5f) ef = add_rn(ef, 1.0f);
  const float T = add_rn(fbits(kLhi[idx]), ef);
  p = fma_rn(p, t, fbits(kPd));
  p = fma_rn(p, t, fbits(kPlo));
  const float H = fma_rn(fbits(kInvLn2), t, T);
  const float L = fma_rn(p, t, fbits(kLlo[idx]));
  const float HmT = sub_rn(H, T);
  const float S = add_rn(H, L);
  const float err = fma_rn(fbits(kInvLn2), t, -HmT);
  const float P = mul_rz(S, y);
  const float SmH = sub_rn(S, H);
  const float Perr = fma_rz(y, S, -P);
  const float Lr = sub_rn(L, SmH);
  const float Slo = add_rn(Lr, err);
  const float Plo = fma_rz(y, Slo, Perr);
  const float Q = add_rz(P, Plo);
  if (!(fabsf(Q) <= fbits(kLimit))) return fallback_pow(x, y);   // over/underflow lanes
  const float QmP = sub_rn(Q, P);
  const float SH = add_rd(Q, fbits(kShifter));
  const float f0 = sub_rd(Q, floor_(Q * 16.0f) * 0.0625f);        // vreduceps M=4, RD
  const float Qlo = sub_rn(Plo, QmP);
  const uint32_t shb = bitsf(SH);
  const float tj = fbits(kExp2[shb & 15u]);
  float f = add_rn(f0, Qlo);
  f = fbits(bitsf(f) & 0xbfffffffu);
  const float scale = fbits((shb << 19) & 0x7f800000u);
  const float tf = mul_rn(tj, f);
  float q = fma_rn(fbits(kE3), f, fbits(kE2));
  q = fma_rn(f, q, fbits(kLn2));
  const float R = fma_rn(tf, q, tj);
  return mul_rn(R, scale);
}

}  // namespace rb_svml
