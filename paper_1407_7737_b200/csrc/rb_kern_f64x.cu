// Function-specialised hybrid / composition kernels for double (functions
// 23..36, rb_fnspec.cuh).  Own translation unit so the build parallelises;
// it owns its __constant__ Weierstrass table.
#include "rb_fnspec.cuh"

namespace rb {

extern const void* const kernels_spec_f64[FN_COUNT_SPEC] = {
    (const void*)evaluate_kernel<double, SPEC_BASE + 23>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 24>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 25>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 26>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 27>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 28>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 29>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 30>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 31>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 32>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 33>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 34>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 35>,
    (const void*)evaluate_kernel<double, SPEC_BASE + 36>,
};

cudaError_t set_weier_f64x(const double* a_then_c) {
  return cudaMemcpyToSymbol(kWei64, a_then_c, sizeof(WeierTab<double>));
}

void phase_read_f64x(unsigned long long out[8], bool reset) {
  for (int i = 0; i < 8; ++i) out[i] = 0;
#ifdef RB_PHASE_TIMING
  cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  }
#else
  (void)reset;
#endif
}

}  // namespace rb
