// Microbenchmark: FP64 DFMA, DMMA (mma.sync f64), FP32 FFMA / FMUL+FADD issue
// rates and fp64/fp32 cos throughput on one B200.  Writes one JSON object to
// stdout.  Used to fill the compute-roofline denominators.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

template<int ILP>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0; for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}
template<int ILP>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0; for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678f) out[0] = s;
}
// The exact-order rotate's instruction pair: a rounded product and a rounded
// add, both operands live (the product depends on the accumulator, so no
// part of the chain is loop-invariant: r01's version multiplied two
// invariants, ptxas hoisted the FMULs and the loop timed FADD alone).
template<int ILP>
__global__ void k_fmuladd(float* out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __fadd_rn(__fmul_rn(acc[i], a), b);
  }
  float s = 0; for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678f) out[0] = s;
}
// float64 DMUL + DADD pair (the exact-order float64 re-evaluation)
template<int ILP>
__global__ void k_dmuladd(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __dadd_rn(__dmul_rn(acc[i], a), b);
  }
  double s = 0; for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}
// packed FP32 (sm_100 FFMA2 / FADD2), the exact-order rotate's instruction
// pair: product as fma(a, b, -0) with an opaque -0, then a separate add
template<int ILP>
__global__ void k_ffma2(float* out, int iters, float a, float b) {
  float2 acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __ffma2_rn(acc[i], A, B);
  }
  float s = 0; for (int i = 0; i < ILP; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.678f) out[0] = s;
}
template<int ILP>
__global__ void k_fmul2_fadd2(float* out, int iters, float a, float nz) {
  float2 acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  const float2 Z = make_float2(nz, nz);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      acc[i] = __fadd2_rn(acc[i], __ffma2_rn(acc[i], make_float2(a, a), Z));
  }
  float s = 0; for (int i = 0; i < ILP; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.678f) out[0] = s;
}
template<int ILP>
__global__ void k_dmma_k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = 0.5;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0; for (int i = 0; i < ILP; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
template<int ILP>
__global__ void k_dmma_k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < ILP; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_cos64(double* out, int iters, double scale) {
  double x = (blockIdx.x * blockDim.x + threadIdx.x) * scale, s = 0;
  for (int it = 0; it < iters; ++it) { s += cos(x); x += 0.37 * scale; }
  if (s == 12345.678) out[0] = s;
}
__global__ void k_cos32(float* out, int iters, float scale) {
  float x = (blockIdx.x * blockDim.x + threadIdx.x) * scale, s = 0;
  for (int it = 0; it < iters; ++it) { s += cosf(x); x += 0.37f * scale; }
  if (s == 12345.678f) out[0] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout; CK(cudaMalloc(&dout, 64));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double nthr = (double)blocks * threads;
  printf("{\"sms\": %d", sms);
  float ms = timeit([&]{ k_dfma<8><<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9); });
  printf(", \"dfma_tflops\": %.2f", nthr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_ffma<8><<<blocks, threads>>>((float*)dout, iters, 1.0000001f, 1e-9f); });
  printf(", \"ffma_tflops\": %.2f", nthr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_fmuladd<8><<<blocks, threads>>>((float*)dout, iters, 1.0000001f, 1e-9f); });
  printf(", \"fmul_fadd_tflops\": %.2f", nthr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_dmuladd<8><<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9); });
  printf(", \"dmul_dadd_tflops\": %.2f", nthr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_ffma2<8><<<blocks, threads>>>((float*)dout, iters, 1.0000001f, 1e-9f); });
  printf(", \"ffma2_tflops\": %.2f", nthr * iters * 8 * 4 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_fmul2_fadd2<8><<<blocks, threads>>>((float*)dout, iters, 1.0000001f, -0.0f); });
  printf(", \"fmul2_fadd2_tflops\": %.2f", nthr * iters * 8 * 4 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_dmma_k4<4><<<blocks, threads>>>(dout, iters / 4); });
  printf(", \"dmma_m16n8k4_tflops\": %.2f", nthr / 32 * (iters / 4) * 4 * 16 * 8 * 4 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_dmma_k16<4><<<blocks, threads>>>(dout, iters / 16); });
  printf(", \"dmma_m16n8k16_tflops\": %.2f", nthr / 32 * (iters / 16) * 4 * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&]{ k_cos64<<<blocks, threads>>>(dout, 256, 1e-3); });
  printf(", \"cos64_small_gops\": %.2f", nthr * 256 / (ms * 1e-3) / 1e9);
  ms = timeit([&]{ k_cos64<<<blocks, threads>>>(dout, 256, 1e4); });
  printf(", \"cos64_large_gops\": %.2f", nthr * 256 / (ms * 1e-3) / 1e9);
  ms = timeit([&]{ k_cos32<<<blocks, threads>>>((float*)dout, 256, 1e-3f); });
  printf(", \"cos32_small_gops\": %.2f", nthr * 256 / (ms * 1e-3) / 1e9);
  ms = timeit([&]{ k_cos32<<<blocks, threads>>>((float*)dout, 256, 1e4f); });
  printf(", \"cos32_large_gops\": %.2f", nthr * 256 / (ms * 1e-3) / 1e9);
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
