// DMMA (mma.sync m16n8k4 f64) throughput vs independent accumulator chains
// per warp and warps per SM: what occupancy / ILP the rotate needs.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(double* out, int iters) {
  double acc[C][4];
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < 4; ++i) acc[c][i] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1.0, b = a0 * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                   : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < 4; ++i) s += acc[c][i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int C>
void run(int warps_per_sm, int sms, double* d) {
  const int iters = 4096 / C;
  const int threads = 32 * (warps_per_sm > 32 ? 32 : warps_per_sm);
  const int blocks = sms * (warps_per_sm * 32 / threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<C><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e0);
  k<C><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = (double)blocks * threads / 32 * iters * C * 16 * 8 * 4 * 2;
  printf("chains %d warps/SM %2d: %6.2f TFLOP/s\n", C, warps_per_sm, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8192 * sizeof(double));
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w, sms, d); run<2>(w, sms, d); run<4>(w, sms, d); run<8>(w, sms, d);
  }
  return 0;
}
