// Shared-memory power-of-two FFT engine (FP64 complex) for sm_100a.
//
// One row of M = 2^LOGM complex doubles (M <= 8192, 128 KiB) lives in shared
// memory and is transformed by GS = fft_gs(LOGM) threads.  Sizes are
// compile-time, so every span, loop bound and swizzle offset is an immediate.
//
// Forward: in-place decimation-in-frequency (DIF), natural order in,
// bit-reversed order out, as K = (LOGM-1)/4 radix-16 passes followed by one
// "core" pass of radix 2^CB (CB = LOGM - 4K in [1, 4]) at span 1.  Inverse:
// the exact adjoint sweep (DIT): bit-reversed in, natural out, unnormalised.
// Every use in this library is a cyclic convolution (Bluestein chirp-z, the MW
// theta-weight convolution), so fft_conv fuses the last forward pass, the
// product with the spectrum table (which the host stores in the same
// bit-reversed order) and the first inverse pass into one shared-memory pass:
// 2K + 1 passes per convolution (7 at M = 8192).
//
// Radix-16 butterflies run in registers as four radix-2 DIF stages; register
// i then holds output brev4(i), which is multiplied by the pass twiddle
// u^brev4(i), u = W_{16 s}^j (s = span, j = position in the span), u read
// from a per-pass table (host-built, contiguous in j) and its powers formed
// by at most four rounding levels of products.
//
// Bank conflicts: element e is stored at swz(e) = e ^ (((e >> 3) ^ (e >> 4)) & 7),
// a permutation within 128-byte rows which (checked exhaustively for every
// pass pattern of LOGM = 3..13) makes each quarter-warp's 16-byte accesses
// hit 8 distinct bank groups.  swz is linear over XOR, so for disjoint bit
// fields swz(a + b) = swz(a) ^ swz(b): the per-element offsets of a butterfly
// are compile-time constants.
#pragma once
#include "common.cuh"

// Bits 9-11 enter the XOR too, so bit-reversed gathers (8 lanes with
// consecutive indices read slots that differ only in bits 9-11) hit distinct
// banks as well; all pass patterns of log2 M = 3..13 stay conflict-free.
__host__ __device__ constexpr int swz(int i) { return i ^ (((i >> 3) ^ (i >> 4) ^ (i >> 9)) & 7); }

__host__ __device__ constexpr int brev4(int r) {
  return ((r & 1) << 3) | ((r & 2) << 1) | ((r & 4) >> 1) | ((r & 8) >> 3);
}

// threads per row and radix-16 pass count / core radix bits for M = 2^LOGM
__host__ __device__ constexpr int fft_gs(int logm) {
  return logm >= 13 ? 512 : logm <= 9 ? 32 : (1 << (logm - 4));
}
// CTA size bound of the row kernels (M = 8192 needs 512 threads of <= 128
// registers; smaller rows run 256-thread CTAs with up to 255 registers)
__host__ __device__ constexpr int fft_maxthr(int logm) { return logm >= 13 ? 512 : 256; }
__host__ __device__ constexpr int fft_k16(int logm) { return (logm - 1) / 4; }
// twiddle-table length (sum of the spans of the radix-16 passes) and offset of pass p
__host__ __device__ constexpr int fft_tw_off(int logm, int p) {
  int o = 0;
  for (int q = 0; q < p; ++q) o += 1 << (logm - 4 * (q + 1));
  return o;
}
__host__ __device__ constexpr int fft_ntw(int logm) { return fft_tw_off(logm, fft_k16(logm)); }

#define S2W_RSQRT2 0.70710678118654752440
#define S2W_C16 0.92387953251128675613
#define S2W_S16 0.38268343236508977173

// v * W16^q (CONJ: v * conj(W16^q)), W16 = exp(-2 pi i / 16), q in [0, 8).
// Always called with q a constant after unrolling, so the switch folds away.
template <bool CONJ>
S2W_DEV double2 mul_w16(int q, double2 v) {
  const double sg = CONJ ? -1.0 : 1.0;  // sign of the imaginary part of the factor
  switch (q & 7) {
    case 0:
      return v;
    case 4:
      return CONJ ? cmul_pi(v) : cmul_mi(v);
    case 2:  // (1 - i)/sqrt2
      return make_double2((v.x + sg * v.y) * S2W_RSQRT2, (v.y - sg * v.x) * S2W_RSQRT2);
    case 6:  // (-1 - i)/sqrt2
      return make_double2((sg * v.y - v.x) * S2W_RSQRT2, -(v.y + sg * v.x) * S2W_RSQRT2);
    default: {
      const double wr = (q & 7) == 1 ? S2W_C16 : (q & 7) == 3 ? S2W_S16 : (q & 7) == 5 ? -S2W_S16 : -S2W_C16;
      const double wi = sg * ((q & 7) == 1 ? -S2W_S16 : (q & 7) == 3 ? -S2W_C16 : (q & 7) == 5 ? -S2W_C16 : -S2W_S16);
      return make_double2(fma(v.x, wr, -v.y * wi), fma(v.x, wi, v.y * wr));
    }
  }
}

// Radix-2^LR DIF butterfly in registers: natural in, register i = output brev(i).
template <int LR>
S2W_DEV void dif(double2* v) {
  constexpr int R = 1 << LR;
#pragma unroll
  for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int b0 = 0; b0 < R; b0 += 2 * h) {
#pragma unroll
      for (int a = 0; a < h; ++a) {
        const double2 p = v[b0 + a], q = v[b0 + a + h];
        v[b0 + a] = cadd(p, q);
        v[b0 + a + h] = mul_w16<false>(a * (8 / h), csub(p, q));
      }
    }
  }
}

// Adjoint of dif: register i = input brev(i), natural out (unnormalised).
template <int LR>
S2W_DEV void adj(double2* v) {
  constexpr int R = 1 << LR;
#pragma unroll
  for (int h = 1; h < R; h <<= 1) {
#pragma unroll
    for (int b0 = 0; b0 < R; b0 += 2 * h) {
#pragma unroll
      for (int a = 0; a < h; ++a) {
        const double2 p = v[b0 + a];
        const double2 t = mul_w16<true>(a * (8 / h), v[b0 + a + h]);
        v[b0 + a] = cadd(p, t);
        v[b0 + a + h] = csub(p, t);
      }
    }
  }
}

// w[k] = u^k, k = 1..15 (w[0] unused)
S2W_DEV void powers16(double2* w, double2 u) {
  w[1] = u;
  w[2] = cmul(u, u);
  w[3] = cmul(w[2], u);
  w[4] = cmul(w[2], w[2]);
  w[5] = cmul(w[4], u);
  w[6] = cmul(w[4], w[2]);
  w[7] = cmul(w[4], w[3]);
  w[8] = cmul(w[4], w[4]);
#pragma unroll
  for (int k = 1; k < 8; ++k) w[8 + k] = cmul(w[8], w[k]);
}

// The register part of one radix-16 pass with pass twiddle u = W_{16 s}^j.
// Forward: v[k] = element j + k s in, register i = output brev4(i) out (the
// in-place DIF layout).  INV: the adjoint, that layout in, natural out.
template <bool INV>
S2W_DEV void bfly16(double2* v, double2 u) {
  // twiddle powers u^1..u^7 and u^8; u^(8+k) = u^8 u^k formed at use (the
  // same products as powers16, with half of them live at a time)
  double2 w[8];
  w[1] = u;
  w[2] = cmul(u, u);
  w[3] = cmul(w[2], u);
  w[4] = cmul(w[2], w[2]);
  w[5] = cmul(w[4], u);
  w[6] = cmul(w[4], w[2]);
  w[7] = cmul(w[4], w[3]);
  const double2 w8 = cmul(w[4], w[4]);
  if constexpr (!INV) dif<4>(v);
#pragma unroll
  for (int kk = 1; kk < 16; ++kk) {
    const double2 wk = kk < 8 ? w[kk] : (kk == 8 ? w8 : cmul(w8, w[kk - 8]));
    const int i = brev4(kk);
    v[i] = INV ? cmulc(v[i], wk) : cmul(v[i], wk);
  }
  if constexpr (INV) adj<4>(v);
}

// One radix-16 pass at span 2^LS (forward DIF, or its adjoint when INV).
// TWS: stride into the twiddle table (2 when a half-size transform borrows
// the table of the engine size: W_{16s}^j = W_{32s}^{2j}).
template <int LOGM, int GS, int LS, bool INV, int TWS = 1>
S2W_DEV void pass16(double2* __restrict__ buf, const double2* __restrict__ tw, int gtid) {
  constexpr int NB = (1 << LOGM) / 16;
  constexpr int S = 1 << LS;
#pragma unroll
  for (int it = 0; it < (NB + GS - 1) / GS; ++it) {
    const int b = gtid + it * GS;
    if (NB % GS != 0 && b >= NB) break;
    const int j = b & (S - 1);
    const int sb = swz(((b >> LS) << (LS + 4)) + j);
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = buf[sb ^ swz(k << LS)];
    bfly16<INV>(v, tw[j * TWS]);
#pragma unroll
    for (int k = 0; k < 16; ++k) buf[sb ^ swz(k << LS)] = v[k];
  }
}

// Core pass: last forward pass (radix 2^CB, span 1), product with the
// bit-reversed spectrum table, first inverse pass.  The table is stored
// transposed, entry (b, i) at i NB + b (capi.cu core_transpose): a warp's
// loads are contiguous.
template <int LOGM, int GS>
S2W_DEV void conv_core(double2* __restrict__ buf, const double2* __restrict__ tab, int gtid) {
  constexpr int CB = LOGM - 4 * fft_k16(LOGM);
  constexpr int R = 1 << CB;
  constexpr int NB = (1 << LOGM) / R;
#pragma unroll
  for (int it = 0; it < (NB + GS - 1) / GS; ++it) {
    const int b = gtid + it * GS;
    if (NB % GS != 0 && b >= NB) break;
    const int sb = swz(b * R);
    double2 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[sb ^ swz(i)];
    dif<CB>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = cmul(v[i], __ldg(&tab[i * NB + b]));
    adj<CB>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) buf[sb ^ swz(i)] = v[i];
  }
}

// conv_core with a real spectrum (a real, even convolution kernel): half the
// table bytes and registers.
template <int LOGM, int GS>
S2W_DEV void conv_core_real(double2* __restrict__ buf, const double* __restrict__ tab, int gtid) {
  constexpr int CB = LOGM - 4 * fft_k16(LOGM);
  constexpr int R = 1 << CB;
  constexpr int NB = (1 << LOGM) / R;
#pragma unroll
  for (int it = 0; it < (NB + GS - 1) / GS; ++it) {
    const int b = gtid + it * GS;
    if (NB % GS != 0 && b >= NB) break;
    const int sb = swz(b * R);
    double t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = __ldg(&tab[i * NB + b]);
    double2 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[sb ^ swz(i)];
    dif<CB>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = cscale(v[i], t[i]);
    adj<CB>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) buf[sb ^ swz(i)] = v[i];
  }
}

// Barrier between the innermost radix-16 pass (span 2^CB) and the core pass
// (radix 2^CB at span 1).  When CB = 4 (LOGM = 8, 12) and every thread has one
// butterfly per pass, both passes of a 256-element block belong to the same 16
// threads (pass: block b >> 4, position b & 15; core: elements 16 b ..), i.e.
// to one half-warp: a warp-level barrier orders them and the warps run pass,
// core and inverse pass without waiting for one another.
template <int LOGM, int GS>
S2W_DEV void sync_core() {
  if constexpr (LOGM - 4 * fft_k16(LOGM) == 4 && GS * 16 == (1 << LOGM) && GS >= 32) __syncwarp();
  else __syncthreads();
}

// Barrier between the radix-16 passes at spans 2^LS and 2^(LS-4): the 2^(LS+4)
// elements of a block of the wider pass belong to the same 2^LS consecutive
// threads in both (one butterfly per thread), so at LS <= 5 that is one warp.
template <int LOGM, int GS, int LS>
S2W_DEV void sync_pass() {
  if constexpr (LS <= 5 && GS * 16 == (1 << LOGM) && GS >= 32) __syncwarp();
  else __syncthreads();
}

// tw: table of the size 2^(LOGM + TWSH) (TWSH = 0 or 1), i.e. for a
// half-size transform the engine's own table read at stride 2.
// Ends synced for the core pass (sync_core), i.e. for the whole CTA unless
// sync_core is the warp-level barrier.
template <int LOGM, int GS, int P, int TWSH = 0>
S2W_DEV void fwd_passes(double2* buf, const double2* tw, int gtid) {
  if constexpr (P < fft_k16(LOGM)) {
    pass16<LOGM, GS, LOGM - 4 * (P + 1), false, 1 << TWSH>(
        buf, tw + fft_tw_off(LOGM + TWSH, P), gtid);
    if constexpr (P == fft_k16(LOGM) - 1) sync_core<LOGM, GS>();
    else sync_pass<LOGM, GS, LOGM - 4 * (P + 1)>();
    fwd_passes<LOGM, GS, P + 1, TWSH>(buf, tw, gtid);
  }
}
// Precondition: the core pass's writes ordered by sync_core (P = last pass).
template <int LOGM, int GS, int P, int PMIN = 0>
S2W_DEV void inv_passes(double2* buf, const double2* tw, int gtid) {
  if constexpr (P >= PMIN) {
    pass16<LOGM, GS, LOGM - 4 * (P + 1), true>(buf, tw + fft_tw_off(LOGM, P), gtid);
    if constexpr (P > PMIN) sync_pass<LOGM, GS, LOGM - 4 * P>();  // next: span 2^(LS + 4)
    else __syncthreads();
    inv_passes<LOGM, GS, P - 1, PMIN>(buf, tw, gtid);
  }
}

// Last forward pass alone (radix 2^CB at span 1, no product).
template <int LOGM, int GS>
S2W_DEV void fwd_core(double2* __restrict__ buf, int gtid) {
  constexpr int CB = LOGM - 4 * fft_k16(LOGM);
  constexpr int R = 1 << CB;
  constexpr int NB = (1 << LOGM) / R;
#pragma unroll
  for (int it = 0; it < (NB + GS - 1) / GS; ++it) {
    const int b = gtid + it * GS;
    if (NB % GS != 0 && b >= NB) break;
    const int sb = swz(b * R);
    double2 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[sb ^ swz(i)];
    dif<CB>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) buf[sb ^ swz(i)] = v[i];
  }
}

// Forward DFT of the first 2^LOGN elements (natural order in, bit-reversed
// order out: X_q at swz(fft_brev<LOGN>(q))), unnormalised.  TWSH as in
// fwd_passes.  Precondition: row written and synced.  Ends synced.
template <int LOGN, int GS, int TWSH>
S2W_DEV void fft_fwd(double2* buf, const double2* tw, int gtid) {
  fwd_passes<LOGN, GS, 0, TWSH>(buf, tw, gtid);
  fwd_core<LOGN, GS>(buf, gtid);
  __syncthreads();
}

template <int LOGN>
S2W_DEV int fft_brev(int q) { return (int)(__brev((unsigned)q) >> (32 - LOGN)); }

// Cyclic convolution of the row with the table's sequence: forward FFT,
// product, inverse FFT.  tw: the pass twiddles (fft_ntw(LOGM) entries,
// shared memory).  Precondition: row written and synced.  Ends synced.
template <int LOGM, int GS>
S2W_DEV void fft_conv(double2* buf, const double2* tw, const double2* __restrict__ tab,
                      int gtid) {
  fwd_passes<LOGM, GS, 0>(buf, tw, gtid);
  conv_core<LOGM, GS>(buf, tab, gtid);
  sync_core<LOGM, GS>();
  inv_passes<LOGM, GS, fft_k16(LOGM) - 1>(buf, tw, gtid);
}

// fft_conv with a real spectrum table (conv_core_real).
template <int LOGM, int GS>
S2W_DEV void fft_conv_real(double2* buf, const double2* tw, const double* __restrict__ tab, int gtid) {
  fwd_passes<LOGM, GS, 0>(buf, tw, gtid);
  conv_core_real<LOGM, GS>(buf, tab, gtid);
  sync_core<LOGM, GS>();
  inv_passes<LOGM, GS, fft_k16(LOGM) - 1>(buf, tw, gtid);
}

// fft_conv_real without its outer radix-16 passes (the first forward and the
// last inverse pass, at span 2^(LOGM-4)): for callers whose GS = 2^(LOGM-4)
// threads run those two in registers (thread j owns the elements j + GS k of
// both) around their own data movement.  Row synced on entry; ends synced.
template <int LOGM, int GS>
S2W_DEV void fft_conv_real_inner(double2* buf, const double2* tw, const double* __restrict__ tab,
                                 int gtid) {
  fwd_passes<LOGM, GS, 1>(buf, tw, gtid);
  conv_core_real<LOGM, GS>(buf, tab, gtid);
  sync_core<LOGM, GS>();
  inv_passes<LOGM, GS, fft_k16(LOGM) - 1, 1>(buf, tw, gtid);
}

// Forward DFT (as fft_fwd) whose first radix-16 pass input the caller holds in
// registers: v[k] = element gtid + GS k, GS = 2^(LOGN-4).  Every thread must
// be done reading the row (a barrier) before the call.  Ends synced.
template <int LOGN, int GS>
S2W_DEV void fft_fwd_from_regs(double2* buf, const double2* tw, double2* v, int gtid) {
  static_assert(GS == (1 << (LOGN - 4)), "one outer butterfly per thread");
  bfly16<false>(v, tw[gtid]);
  const int sb = swz(gtid);
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[sb ^ swz(k << (LOGN - 4))] = v[k];
  __syncthreads();
  fwd_passes<LOGN, GS, 1, 0>(buf, tw, gtid);
  fwd_core<LOGN, GS>(buf, gtid);
  __syncthreads();
}

// Copy the pass twiddles into shared memory (all threads of the CTA).
template <int LOGM>
S2W_DEV void load_tw(double2* __restrict__ s_tw, const double2* __restrict__ g_tw) {
  for (int i = threadIdx.x; i < fft_ntw(LOGM); i += blockDim.x) s_tw[i] = __ldg(&g_tw[i]);
}

// ------------------------------------------------------------------ octant twiddles
// W_M^k = exp(-2 pi i k / M) for arbitrary k from an octant table
// oct[r] = (cos, sin)(2 pi r / M), r in [0, M/8] (split mode's W_M^j factors).
S2W_DEV int oct_slot(int r) { return r ^ (((r >> 3) ^ (r >> 6) ^ (r >> 9)) & 7); }
__host__ __device__ constexpr int oct_alloc(int logM) { return ((1 << (logM - 3)) + 8) & ~7; }

S2W_DEV double2 twiddle(int k, const double2* __restrict__ oct, int logM) {
  const int sh = logM - 3;
  const int M8 = 1 << sh;
  const int q = (k >> sh) & 7;
  int r = k & (M8 - 1);
  if (q & 1) r = M8 - r;
  const double2 e = oct[oct_slot(r)];
  const bool swap = ((q + 1) & 2) != 0;  // q in {1, 2, 5, 6}
  double c = swap ? e.y : e.x;
  double s = swap ? e.x : e.y;
  if (q >= 2 && q <= 5) c = -c;  // cos(phi) < 0
  if (q >= 4) s = -s;            // sin(phi) < 0
  return make_double2(c, -s);
}

S2W_DEV void load_octant(double2* __restrict__ s_oct, const double2* __restrict__ g_oct, int logM) {
  const int n = (1 << (logM - 3)) + 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_oct[oct_slot(i)] = __ldg(&g_oct[i]);
}
