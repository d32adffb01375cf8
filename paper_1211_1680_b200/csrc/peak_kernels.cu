// FP64 peak microbenchmark: independent DFMA chains, one CTA per SM slot.
// Used by bench.py as the measured denominator of the Legendre-stage roofline.
#include "common.cuh"
#include "s2w_internal.h"

namespace s2w {

constexpr int PK_CHAINS = 8;

__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
  double x[PK_CHAINS];
#pragma unroll
  for (int c = 0; c < PK_CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < PK_CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < PK_CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// DMMA (mma.sync m8n8k4 f64) throughput: 8 independent accumulator tiles.
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

cudaError_t measure_dmma_peak(double* tflops, cudaStream_t st) {
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d;
  cudaError_t e = cudaMalloc(&d, sizeof(double));
  if (e != cudaSuccess) return e;
  const int iters = 1 << 12, blocks = sms * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  dmma_peak_kernel<<<blocks, threads, 0, st>>>(d, iters);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, st);
    dmma_peak_kernel<<<blocks, threads, 0, st>>>(d, iters);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  // per warp-level mma: 8*8*4 FMAs = 512 flops
  const double flops = 512.0 * 8 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (best * 1e-3) / 1e12;
  return e;
}

cudaError_t measure_fp64_peak(double* tflops, cudaStream_t st) {
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d;
  cudaError_t e = cudaMalloc(&d, sizeof(double));
  if (e != cudaSuccess) return e;
  const int iters = 1 << 14, blocks = sms * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fp64_peak_kernel<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, st);
    fp64_peak_kernel<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  const double flops = 2.0 * PK_CHAINS * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return e;
}

}  // namespace s2w
