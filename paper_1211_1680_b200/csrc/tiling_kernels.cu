// Harmonic-space tiling (transform.py:117-172): per-degree products with the
// kernel tables, multiresolution truncation (a prefix of the flat l^2+l+m
// layout, sht.py:131-137) and zero-padded recombination.  HBM-bound streaming
// kernels: one read of f and one write per output (analysis); one read per
// input and one write of f (synthesis).
#include <algorithm>
#include "common.cuh"
#include "s2w_internal.h"

namespace s2w {

__device__ __forceinline__ int degree_of(long long i) {
  int l = (int)sqrt((double)i);
  while ((long long)l * l > i) --l;
  while ((long long)(l + 1) * (l + 1) <= i) ++l;
  return l;
}

__global__ void tile_analysis_kernel(TileArgs a) {
  const long long L2 = (long long)a.L * a.L;
  const long long n = L2 * a.n_sets;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int set = (int)(g / L2);
    const long long i = g - set * L2;
    const int l = degree_of(i);
    const double2 f = a.f_in[g];
    for (int j = 0; j < a.n_k; ++j) {
      const long long bj2 = (long long)a.band[j] * a.band[j];
      if (i < bj2) a.ptr[j][set * bj2 + i] = cscale(f, __ldg(&a.fac[(size_t)j * a.L + l]));
    }
  }
}

__global__ void tile_synthesis_kernel(TileArgs a) {
  const long long L2 = (long long)a.L * a.L;
  const long long n = L2 * a.n_sets;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int set = (int)(g / L2);
    const long long i = g - set * L2;
    const int l = degree_of(i);
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < a.n_k; ++j) {
      const long long bj2 = (long long)a.band[j] * a.band[j];
      if (i < bj2) {
        const double2 v = cscale(a.ptr[j][set * bj2 + i], __ldg(&a.fac[(size_t)j * a.L + l]));
        acc = cadd(acc, v);
      }
    }
    a.f_out[g] = acc;
  }
}

static int tile_grid(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_tile_analysis(const TileArgs& a, cudaStream_t st) {
  const long long n = (long long)a.L * a.L * a.n_sets;
  if (n == 0) return cudaSuccess;
  tile_analysis_kernel<<<tile_grid(n), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_tile_synthesis(const TileArgs& a, cudaStream_t st) {
  const long long n = (long long)a.L * a.L * a.n_sets;
  if (n == 0) return cudaSuccess;
  tile_synthesis_kernel<<<tile_grid(n), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Real <-> complex128 map layouts of the numpy drop-in (the reference stores
// real maps as complex128 with zero imaginary parts, grid.py:155-160): the
// conversion runs here instead of as host passes over the arrays.
__global__ void real_to_complex_kernel(const double* in, double2* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = make_double2(in[i], 0.0);
}
__global__ void complex_real_part_kernel(const double2* in, double* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i].x;
}
static int elem_grid(long long n) { return (int)std::min<long long>((n + 255) / 256, 148LL * 16); }

cudaError_t launch_real_to_complex(const double* in, double2* out, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  real_to_complex_kernel<<<elem_grid(n), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}
cudaError_t launch_complex_real_part(const double2* in, double* out, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  complex_real_part_kernel<<<elem_grid(n), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace s2w
