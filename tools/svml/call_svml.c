// Call NumPy's bundled __svml_powf16 directly (address = dlsym(PyInit) + delta).
#include <dlfcn.h>
#include <immintrin.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
typedef __m512 (*powf16_t)(__m512, __m512);
static powf16_t fn;
int svml_init(const char* so, long init_off, long pow_off) {
  void* h = dlopen(so, RTLD_NOW | RTLD_GLOBAL);
  if (!h) { fprintf(stderr, "%s\n", dlerror()); return 1; }
  char* init = (char*)dlsym(h, "PyInit__multiarray_umath");
  if (!init) return 2;
  fn = (powf16_t)(init - init_off + pow_off);
  return 0;
}
void svml_pow(const float* x, const float* y, float* out, long n) {
  for (long i = 0; i < n; i += 16) {
    float bx[16], by[16], bo[16];
    for (int k = 0; k < 16; ++k) { bx[k] = i + k < n ? x[i + k] : 1.f; by[k] = i + k < n ? y[i + k] : 1.f; }
    __m512 r = fn(_mm512_loadu_ps(bx), _mm512_loadu_ps(by));
    _mm512_storeu_ps(bo, r);
    for (int k = 0; k < 16 && i + k < n; ++k) out[i + k] = bo[k];
  }
}
