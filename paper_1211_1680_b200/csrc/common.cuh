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

// ------------------------------------------------------------------ bulk copies (TMA)
// One-shot global -> shared bulk copies completed on an mbarrier
// (cp.async.bulk, the non-tensor TMA path): one elected thread arms the
// barrier with the byte count and issues the copies; every thread waits on
// the barrier's phase.  Sizes and both addresses must be multiples of 16.
S2W_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
S2W_DEV void mbar_init(uint64_t* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
S2W_DEV void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes)
               : "memory");
}
S2W_DEV void mbar_wait(uint64_t* mb, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n S2W_MBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra S2W_MBW_%=;\n}\n" ::"r"(smem_u32(mb)),
      "r"(parity)
      : "memory");
}
S2W_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mb))
      : "memory");
}
// Order this thread's earlier generic-proxy shared-memory accesses before
// later async-proxy (bulk copy) writes to the same memory.
S2W_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
S2W_DEV bool bulk_ok(const void* p, size_t bytes) {
  return (((uintptr_t)p | bytes) & 15) == 0 && bytes > 0;
}
S2W_DEV void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
