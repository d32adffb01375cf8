// Shared helpers for the s2w (spherical wavelet) sm_100a kernels.
//
// Complex numbers are double2 {x = re, y = im}, the same interleaved layout
// numpy complex128 uses, so host buffers cross the C-ABI without repacking.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define S2W_DEV __device__ __forceinline__

S2W_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
S2W_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
S2W_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
S2W_DEV double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
S2W_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
S2W_DEV double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i
S2W_DEV double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }
// multiply by +i
S2W_DEV double2 cmul_pi(double2 a) { return make_double2(-a.y, a.x); }

// Exact power of two 2^e for |e| <= 1022 (normal range), built from bits.
S2W_DEV double pow2i(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// Work descriptors shared between host planner and kernels.
struct S2WRowSpan {  // generic [begin, end) pair
  int lo, hi;
};
