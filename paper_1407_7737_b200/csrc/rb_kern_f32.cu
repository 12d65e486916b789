// Instantiations of the evaluation kernel for float: one per basic kernel
// (single-segment functions 0..22) plus the generic hybrid/composition
// variant.  Compiled as its own unit so the build parallelises.
#include "rb_device.cuh"

namespace rb {

extern const void* const kernels_f32[N_VARIANTS] = {
    (const void*)evaluate_kernel<float, 0>,  (const void*)evaluate_kernel<float, 1>,
    (const void*)evaluate_kernel<float, 2>,  (const void*)evaluate_kernel<float, 3>,
    (const void*)evaluate_kernel<float, 4>,  (const void*)evaluate_kernel<float, 5>,
    (const void*)evaluate_kernel<float, 6>,  (const void*)evaluate_kernel<float, 7>,
    (const void*)evaluate_kernel<float, 8>,  (const void*)evaluate_kernel<float, 9>,
    (const void*)evaluate_kernel<float, 10>, (const void*)evaluate_kernel<float, 11>,
    (const void*)evaluate_kernel<float, 12>, (const void*)evaluate_kernel<float, 13>,
    (const void*)evaluate_kernel<float, 14>, (const void*)evaluate_kernel<float, 15>,
    (const void*)evaluate_kernel<float, 16>, (const void*)evaluate_kernel<float, 17>,
    (const void*)evaluate_kernel<float, 18>, (const void*)evaluate_kernel<float, 19>,
    (const void*)evaluate_kernel<float, 20>, (const void*)evaluate_kernel<float, GENERIC>,
};

// Large dimensions: tiles in global scratch (rb_device.cuh evaluate_big_kernel).
extern const void* const big_f32 = (const void*)evaluate_big_kernel<float>;
// Plan image builder (rb_device.cuh enter_plan).
extern const void* const plan_image_f32 = (const void*)plan_image_kernel<float, false>;

// Series constants of this unit's Weierstrass kernels (rb_kernels.cuh);
// each translation unit owns its __constant__ copy.
cudaError_t set_weier_f32(const float* a_then_c) {
  return cudaMemcpyToSymbol(kWei32, a_then_c, sizeof(WeierTab<float>));
}

// Phase timing counters of this unit (zeros unless built with RB_PHASE_TIMING).
void phase_read_f32(unsigned long long out[8], bool reset) {
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
