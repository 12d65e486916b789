// Brute force: r(m) = rndscale(rcp14(m), 5 fraction bits, RNE) for every
// float m in [0.5, 1); print the breakpoints where r changes (numpy SVML
// __svml_powf16 table index selection).  Build: gcc -O2 -mavx512f
#include <immintrin.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
static float r_of(float m) {
  __m512 v = _mm512_set1_ps(m);
  __m512 rc = _mm512_rcp14_ps(v);
  __m512 r = _mm512_roundscale_ps(rc, 0x58);
  float out[16]; _mm512_storeu_ps(out, r); return out[0];
}
int main(void) {
  uint32_t lo = 0x3f000000u, hi = 0x3f800000u;  // [0.5, 1)
  float prev = -1.f; long mism = 0;
  for (uint32_t b = lo; b < hi; ++b) {
    float m; memcpy(&m, &b, 4);
    float r = r_of(m);
    float ideal = nearbyintf((float)(32.0 / (double)m)) / 32.0f;  // RNE of exact 1/m on the 1/32 grid
    if (r != ideal) ++mism;
    if (r != prev) { printf("0x%08x %.9g r=%.9g\n", b, m, r); prev = r; }
  }
  fprintf(stderr, "mismatches vs exact rounding: %ld\n", mism);
  return 0;
}
