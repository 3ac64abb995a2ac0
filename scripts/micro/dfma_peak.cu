// FP64 FMA throughput microbenchmark (the ALU peak the transform kernel is
// measured against, K10).  8 independent DFMA chains per thread,
// 148 x 8 CTAs of 256 threads, CUDA events.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_peak dfma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  k<<<blocks, threads>>>(d, 16, 0.999, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * (double)iters * blocks * threads;
  printf("{\"fp64_fma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f}\n", flops / (best * 1e-3) / 1e12, sms, best);
  return 0;
}
