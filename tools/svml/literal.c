// Literal AVX-512 transcription of NumPy's __svml_powf16 main path, with
// intermediates exported, to debug the scalar restatement (rb_svml_powf.cuh).
#include <immintrin.h>
#include <stdint.h>
#include <string.h>

#define B(off) _mm512_loadu_ps((const float*)((const char*)TAB + (off)))
#define RN (_MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC)
#define RZ (_MM_FROUND_TO_ZERO | _MM_FROUND_NO_EXC)
#define RD (_MM_FROUND_TO_NEG_INF | _MM_FROUND_NO_EXC)
uint32_t TAB[384];
void literal(const float* xs, const float* ys, float* out, float* inter, long n) {
  for (long i = 0; i < n; i += 16) {
    float bx[16], by[16];
    for (int k = 0; k < 16; ++k) { bx[k] = i + k < n ? xs[i + k] : 1.f; by[k] = i + k < n ? ys[i + k] : 1.f; }
    __m512 x = _mm512_loadu_ps(bx), y = _mm512_loadu_ps(by);
    __m512 m = _mm512_getmant_round_ps(x, _MM_MANT_NORM_p5_1, _MM_MANT_SIGN_nan, _MM_FROUND_NO_EXC);
    __m512 one = B(0x180), ca = B(0x1c0), cb = B(0x200), c15 = B(0x140), cc = B(0x240);
    __m512 e = _mm512_getexp_round_ps(x, _MM_FROUND_NO_EXC);
    __m512 rc = _mm512_rcp14_ps(m);
    __m512 r = _mm512_roundscale_ps(rc, 0x58);
    __m512 t = _mm512_fmsub_round_ps(r, m, one, RN);
    __mmask16 k1 = _mm512_cmp_ps_mask(r, c15, _CMP_LT_OQ);
    __m512 p = _mm512_fmadd_round_ps(ca, t, cb, RN);
    __m512i idx = _mm512_srli_epi32(_mm512_castps_si512(r), 18);
    p = _mm512_fmadd_round_ps(p, t, cc, RN);
    e = _mm512_mask_add_round_ps(e, k1, e, one, RN);
    __m512 lhi = _mm512_permutex2var_ps(B(0x0), idx, B(0x40));
    __m512 llo = _mm512_permutex2var_ps(B(0x80), idx, B(0xc0));
    __m512 T = _mm512_add_round_ps(lhi, e, RN);
    p = _mm512_fmadd_round_ps(p, t, B(0x280), RN);
    p = _mm512_fmadd_round_ps(p, t, B(0x2c0), RN);
    __m512 H = _mm512_fmadd_round_ps(B(0x300), t, T, RN);
    __m512 L = _mm512_fmadd_round_ps(p, t, llo, RN);
    __m512 HmT = _mm512_sub_round_ps(H, T, RN);
    __m512 S = _mm512_add_round_ps(H, L, RN);
    __m512 err = _mm512_fmsub_round_ps(B(0x300), t, HmT, RN);
    __m512 P = _mm512_mul_round_ps(S, y, RZ);
    __m512 SmH = _mm512_sub_round_ps(S, H, RN);
    __m512 Perr = _mm512_fmsub_round_ps(y, S, P, RZ);
    __m512 Lr = _mm512_sub_round_ps(L, SmH, RN);
    __m512 Slo = _mm512_add_round_ps(Lr, err, RN);
    __m512 Plo = _mm512_fmadd_round_ps(y, Slo, Perr, RZ);
    __m512 Q = _mm512_add_round_ps(P, Plo, RZ);
    __m512 QmP = _mm512_sub_round_ps(Q, P, RN);
    __m512 SH = _mm512_add_round_ps(Q, B(0x340), RD);
    __m512 f0 = _mm512_reduce_round_ps(Q, 0x41, _MM_FROUND_NO_EXC);
    __m512 Qlo = _mm512_sub_round_ps(Plo, QmP, RN);
    __m512 tj = _mm512_permutexvar_ps(_mm512_castps_si512(SH), B(0x100));
    __m512 f = _mm512_add_round_ps(f0, Qlo, RN);
    __m512i shb = _mm512_slli_epi32(_mm512_castps_si512(SH), 19);
    f = _mm512_and_ps(f, B(0x380));
    __m512 scale = _mm512_and_ps(_mm512_castsi512_ps(shb), B(0x5c0));
    __m512 tf = _mm512_mul_round_ps(tj, f, RN);
    __m512 q = _mm512_fmadd_round_ps(B(0x3c0), f, B(0x400), RN);
    q = _mm512_fmadd_round_ps(f, q, B(0x440), RN);
    __m512 R = _mm512_fmadd_round_ps(tf, q, tj, RN);
    __m512 res = _mm512_mul_round_ps(R, scale, RN);
    float o[16]; _mm512_storeu_ps(o, res);
    __m512 iv[8] = {t, T, H, L, Q, f0, Qlo, f};
    for (int k = 0; k < 16 && i + k < n; ++k) {
      out[i + k] = o[k];
      for (int j = 0; j < 8; ++j) { float tmp[16]; _mm512_storeu_ps(tmp, iv[j]); inter[(i + k) * 8 + j] = tmp[k]; }
    }
  }
}
