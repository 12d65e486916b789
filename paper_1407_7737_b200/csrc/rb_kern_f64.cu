// Instantiations of the evaluation kernel for double: one per basic kernel
// (single-segment functions 0..22) plus the generic hybrid/composition
// variant.  Compiled as its own unit so the build parallelises.
#include "rb_device.cuh"

namespace rb {

extern const void* const kernels_f64[N_VARIANTS] = {
    (const void*)evaluate_kernel<double, 0>,  (const void*)evaluate_kernel<double, 1>,
    (const void*)evaluate_kernel<double, 2>,  (const void*)evaluate_kernel<double, 3>,
    (const void*)evaluate_kernel<double, 4>,  (const void*)evaluate_kernel<double, 5>,
    (const void*)evaluate_kernel<double, 6>,  (const void*)evaluate_kernel<double, 7>,
    (const void*)evaluate_kernel<double, 8>,  (const void*)evaluate_kernel<double, 9>,
    (const void*)evaluate_kernel<double, 10>, (const void*)evaluate_kernel<double, 11>,
    (const void*)evaluate_kernel<double, 12>, (const void*)evaluate_kernel<double, 13>,
    (const void*)evaluate_kernel<double, 14>, (const void*)evaluate_kernel<double, 15>,
    (const void*)evaluate_kernel<double, 16>, (const void*)evaluate_kernel<double, 17>,
    (const void*)evaluate_kernel<double, 18>, (const void*)evaluate_kernel<double, 19>,
    (const void*)evaluate_kernel<double, 20>, (const void*)evaluate_kernel<double, GENERIC>,
};

// The exact-order re-evaluation of marked rows (any function; float64).
extern const void* const fixup_f64 = (const void*)fixup_kernel<double>;
// Large dimensions: tiles in global scratch (rb_device.cuh evaluate_big_kernel).
extern const void* const big_f64 = (const void*)evaluate_big_kernel<double>;
// Plan image builders (rb_device.cuh enter_plan), [MT2].
extern const void* const plan_image_f64[2] = {(const void*)plan_image_kernel<double, false>,
                                              (const void*)plan_image_kernel<double, true>};

// Series constants of this unit's Weierstrass kernels (rb_kernels.cuh);
// each translation unit owns its __constant__ copy.
cudaError_t set_weier_f64(const double* a_then_c) {
  return cudaMemcpyToSymbol(kWei64, a_then_c, sizeof(WeierTab<double>));
}

// Phase timing counters of this unit (zeros unless built with RB_PHASE_TIMING).
void phase_read_f64(unsigned long long out[8], bool reset) {
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
