// CPU build of csrc/rb_svml_powf.cuh for tools/svml/verify.py (ctypes).
#include "../../paper_1407_7737_b200/csrc/rb_svml_powf.cuh"
extern "C" void powf_np_batch(const float* x, const float* y, float* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = rb_svml::powf_np(x[i], y[i]);
}
