// FP64 throughput microbenchmark: DFMA (independent chains) and IEEE DSQRT,
// all 148 SMs, timed with CUDA events.  Writes one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
  const double m = 0.9999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __fma_rn(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dsqrt_kernel(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 2.0 + threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __dsqrt_rn(a[k]) + 1.5;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  // warm up clocks
  for (int w = 0; w < 20; ++w) dfma_kernel<<<blocks, threads>>>(d, iters);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, threads>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double dfma = (double)blocks * threads * iters * 8 * reps / (ms / 1e3);
  for (int w = 0; w < 3; ++w) dsqrt_kernel<<<blocks, threads>>>(d, iters / 8);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) dsqrt_kernel<<<blocks, threads>>>(d, iters / 8);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double dsq = (double)blocks * threads * (iters / 8) * 8 * reps / (ms / 1e3);
  printf("{\"dfma_per_s\": %.6g, \"fp64_tflops\": %.4f, \"dsqrt_per_s\": %.6g, \"sms\": %d}\n",
         dfma, 2 * dfma / 1e12, dsq, sms);
  return 0;
}
