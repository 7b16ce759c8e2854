// Measured fp64 FMA peak of this B200 (the roofline denominator of the elasticity operator,
// k_el_apply, which is DFMA bound): 8 independent DFMA chains per thread, full occupancy,
// grid a multiple of the SM count; CUDA events around a launch after warm-up.
// Output: one JSON line {"fp64_tflops": ..., "sm_count": ..., "ms": ...}.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-9 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * blocks * (double)threads * iters * 16 * 8;
  printf("{\"fp64_tflops\": %.3f, \"sm_count\": %d, \"ms\": %.4f, \"err\": \"%s\"}\n", flops / (best * 1e-3) / 1e12,
         sms, best, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
