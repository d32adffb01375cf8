// Microbenchmark (development aid): do DMMA (mma.sync f64) and DFMA issue
// concurrently on sm_100a?  Each warp runs `nd` independent DMMA tiles and
// `nf` independent DFMA chains per iteration; compare the mixed kernel's time
// with the pure ones.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mp scripts/mixed_pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF>
__global__ void __launch_bounds__(256) mixed(double* out, int iters, double a, double b) {
  double c[ND > 0 ? ND : 1][2];
  double x[NF > 0 ? NF : 1];
  for (int t = 0; t < ND; ++t) c[t][0] = c[t][1] = 0.0;
  for (int f = 0; f < NF; ++f) x[f] = threadIdx.x * 1e-9 + f;
  const double ma = 1.0 + threadIdx.x * 1e-9, mb = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < ND; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(ma), "d"(mb));
#pragma unroll
    for (int f = 0; f < NF; ++f) x[f] = fma(x[f], a, b);
  }
  double s = 0;
  for (int t = 0; t < ND; ++t) s += c[t][0] + c[t][1];
  for (int f = 0; f < NF; ++f) s += x[f];
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF>
float run(double* d, int iters) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mixed<ND, NF><<<sms * 8, 256>>>(d, iters, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    mixed<ND, NF><<<sms * 8, 256>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double dm = 512.0 * ND * iters * sms * 8 * 8, df = 2.0 * NF * iters * sms * 8 * 256.0;
  printf("ND=%d NF=%2d: %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n", ND, NF, best,
         dm / best / 1e9, df / best / 1e9, (dm + df) / best / 1e9);
  return best;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  const int it = 1 << 12;
  run<8, 0>(d, it);
  run<0, 16>(d, it);
  run<8, 16>(d, it);
  run<8, 8>(d, it);
  run<4, 16>(d, it);
  run<8, 32>(d, it);
  return 0;
}
