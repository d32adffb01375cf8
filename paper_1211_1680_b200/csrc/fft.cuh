// Shared-memory power-of-two FFT engine (FP64 complex) for sm_100a.
//
// One row of M = 2^logM complex doubles lives in shared memory (M <= 8192,
// i.e. 128 KiB).  The forward transform is an in-place decimation-in-frequency
// (DIF) Cooley-Tukey sweep of radix-8 passes (plus one radix-4/2 pass when
// logM is not a multiple of 3): natural-order input, bit-reversed output.
// The inverse is the exact adjoint sweep (DIT): bit-reversed input, natural
// output, unnormalised (x M).  Every use in this library is a convolution
// (Bluestein chirp-z, the MW theta-weight convolution), so the bit-reversed
// spectrum is multiplied by a table that the host stored in the same
// bit-reversed order and never has to be permuted.
//
// Bank conflicts: a 16-byte complex spans 4 banks; strided radix passes would
// hit the same banks, so element i is stored at swz(i) = i ^ ((i >> 3) & 7),
// which permutes within 128-byte rows and makes the stride-1/2/4/8/contiguous
// access patterns of all passes conflict-free.
#pragma once
#include "common.cuh"

S2W_DEV int swz(int i) { return i ^ ((i >> 3) & 7); }

template <int R> S2W_DEV int brev(int r);
template <> S2W_DEV int brev<2>(int r) { return r; }
template <> S2W_DEV int brev<4>(int r) { return ((r & 1) << 1) | (r >> 1); }
template <> S2W_DEV int brev<8>(int r) { return ((r & 1) << 2) | (r & 2) | (r >> 2); }

#define S2W_RSQRT2 0.70710678118654752440

// (a + i b) * W8^1 = (a + i b)(1 - i)/sqrt2
S2W_DEV double2 mul_w8_1(double2 v) {
  return make_double2((v.x + v.y) * S2W_RSQRT2, (v.y - v.x) * S2W_RSQRT2);
}
// * W8^3 = (-1 - i)/sqrt2
S2W_DEV double2 mul_w8_3(double2 v) {
  return make_double2((v.y - v.x) * S2W_RSQRT2, -(v.x + v.y) * S2W_RSQRT2);
}
// * conj(W8^1) = (1 + i)/sqrt2
S2W_DEV double2 mul_w8c_1(double2 v) {
  return make_double2((v.x - v.y) * S2W_RSQRT2, (v.x + v.y) * S2W_RSQRT2);
}
// * conj(W8^3) = (-1 + i)/sqrt2
S2W_DEV double2 mul_w8c_3(double2 v) {
  return make_double2(-(v.x + v.y) * S2W_RSQRT2, (v.x - v.y) * S2W_RSQRT2);
}

// In-register radix butterflies.  Forward: in-place DIF radix-2 stages, so
// register i ends up holding X[brev(i)].  Inverse: the adjoint, taking
// brev-ordered input to natural-order output (unnormalised).
template <int R> S2W_DEV void bfly_fwd(double2* v);
template <int R> S2W_DEV void bfly_inv(double2* v);

template <> S2W_DEV void bfly_fwd<2>(double2* v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
template <> S2W_DEV void bfly_inv<2>(double2* v) { bfly_fwd<2>(v); }

template <> S2W_DEV void bfly_fwd<4>(double2* v) {
  double2 a0 = cadd(v[0], v[2]), a2 = csub(v[0], v[2]);
  double2 a1 = cadd(v[1], v[3]), a3 = cmul_mi(csub(v[1], v[3]));
  v[0] = cadd(a0, a1);
  v[1] = csub(a0, a1);
  v[2] = cadd(a2, a3);
  v[3] = csub(a2, a3);
}
template <> S2W_DEV void bfly_inv<4>(double2* v) {
  // adjoint: stage span-1 first, then span-2 with conj twiddles
  double2 a0 = cadd(v[0], v[1]), a1 = csub(v[0], v[1]);
  double2 a2 = cadd(v[2], v[3]), a3 = csub(v[2], v[3]);
  a3 = cmul_pi(a3);
  v[0] = cadd(a0, a2);
  v[2] = csub(a0, a2);
  v[1] = cadd(a1, a3);
  v[3] = csub(a1, a3);
}

template <> S2W_DEV void bfly_fwd<8>(double2* v) {
  // stage span 4
  double2 b0 = cadd(v[0], v[4]), b4 = csub(v[0], v[4]);
  double2 b1 = cadd(v[1], v[5]), b5 = mul_w8_1(csub(v[1], v[5]));
  double2 b2 = cadd(v[2], v[6]), b6 = cmul_mi(csub(v[2], v[6]));
  double2 b3 = cadd(v[3], v[7]), b7 = mul_w8_3(csub(v[3], v[7]));
  // stage span 2
  double2 c0 = cadd(b0, b2), c2 = csub(b0, b2);
  double2 c1 = cadd(b1, b3), c3 = cmul_mi(csub(b1, b3));
  double2 c4 = cadd(b4, b6), c6 = csub(b4, b6);
  double2 c5 = cadd(b5, b7), c7 = cmul_mi(csub(b5, b7));
  // stage span 1
  v[0] = cadd(c0, c1);
  v[1] = csub(c0, c1);
  v[2] = cadd(c2, c3);
  v[3] = csub(c2, c3);
  v[4] = cadd(c4, c5);
  v[5] = csub(c4, c5);
  v[6] = cadd(c6, c7);
  v[7] = csub(c6, c7);
}
template <> S2W_DEV void bfly_inv<8>(double2* v) {
  // adjoint of the above: span 1, span 2 (conj), span 4 (conj)
  double2 c0 = cadd(v[0], v[1]), c1 = csub(v[0], v[1]);
  double2 c2 = cadd(v[2], v[3]), c3 = csub(v[2], v[3]);
  double2 c4 = cadd(v[4], v[5]), c5 = csub(v[4], v[5]);
  double2 c6 = cadd(v[6], v[7]), c7 = csub(v[6], v[7]);
  // span 2: (a, b) -> (a + conj(w) b, a - conj(w) b), w = 1 or -i
  double2 t;
  double2 b0 = cadd(c0, c2), b2 = csub(c0, c2);
  t = cmul_pi(c3);
  double2 b1 = cadd(c1, t), b3 = csub(c1, t);
  double2 b4 = cadd(c4, c6), b6 = csub(c4, c6);
  t = cmul_pi(c7);
  double2 b5 = cadd(c5, t), b7 = csub(c5, t);
  // span 4: w = W8^i
  v[0] = cadd(b0, b4);
  v[4] = csub(b0, b4);
  t = mul_w8c_1(b5);
  v[1] = cadd(b1, t);
  v[5] = csub(b1, t);
  t = cmul_pi(b6);
  v[2] = cadd(b2, t);
  v[6] = csub(b2, t);
  t = mul_w8c_3(b7);
  v[3] = cadd(b3, t);
  v[7] = csub(b3, t);
}

// Octant-table slot of entry r: XOR-swizzled so that power-of-two strides
// (tstep = 8, 64, 512 in the radix-8 passes) hit distinct 16-byte bank groups.
S2W_DEV int oct_slot(int r) { return r ^ (((r >> 3) ^ (r >> 6) ^ (r >> 9)) & 7); }
// entries allocated for an octant table of M = 2^logM (slot range rounded to 8)
__host__ __device__ constexpr int oct_alloc(int logM) { return ((1 << (logM - 3)) + 8) & ~7; }

// W_M^k = exp(-2 pi i k / M) from an octant table oct[r] = (cos, sin)(2 pi r / M),
// r in [0, M/8], held in shared memory (M/8 + 1 entries: 16 KiB at M = 8192).
S2W_DEV double2 twiddle(int k, const double2* __restrict__ oct, int logM) {
  const int sh = logM - 3;
  const int M8 = 1 << sh;
  const int q = (k >> sh) & 7;
  int r = k & (M8 - 1);
  if (q & 1) r = M8 - r;
  const double2 e = oct[oct_slot(r)];
  const bool swap = ((q + 1) & 2) != 0;          // q in {1, 2, 5, 6}
  double c = swap ? e.y : e.x;
  double s = swap ? e.x : e.y;
  if (q >= 2 && q <= 5) c = -c;                  // cos(phi) < 0
  if (q >= 4) s = -s;                            // sin(phi) < 0
  return make_double2(c, -s);
}

// Twiddles of one radix-R butterfly: w[r] = u^r, u = W_M^ts (one table lookup,
// then products; at most 3 roundings deep for R = 8).
template <int R>
S2W_DEV void twiddle_powers(double2* w, int ts, const double2* __restrict__ oct, int logM) {
  const double2 u = twiddle(ts, oct, logM);
  w[1] = u;
  if (R >= 4) {
    w[2] = cmul(u, u);
    w[3] = cmul(w[2], u);
  }
  if (R >= 8) {
    w[4] = cmul(w[2], w[2]);
    w[5] = cmul(w[4], u);
    w[6] = cmul(w[3], w[3]);
    w[7] = cmul(w[4], w[3]);
  }
}

// One radix-R pass of span s = 2^log2s over a row of M elements.
template <int R, bool INV>
S2W_DEV void fft_pass(double2* __restrict__ buf, int logM, int log2s,
                      const double2* __restrict__ oct, int gtid, int gsize) {
  const int M = 1 << logM;
  const int s = 1 << log2s;
  const int nb = M / R;
  const int tstep = M / (R * s);
  for (int b = gtid; b < nb; b += gsize) {
    const int blk = b >> log2s, j = b & (s - 1);
    const int base = blk * R * s + j;
    double2 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[swz(base + i * s)];
    if (!INV) {
      bfly_fwd<R>(v);
      if (j) {
        double2 w[R];
        twiddle_powers<R>(w, j * tstep, oct, logM);
#pragma unroll
        for (int i = 1; i < R; ++i) v[i] = cmul(v[i], w[brev<R>(i)]);
      }
    } else {
      if (j) {
        double2 w[R];
        twiddle_powers<R>(w, j * tstep, oct, logM);
#pragma unroll
        for (int i = 1; i < R; ++i) v[i] = cmulc(v[i], w[brev<R>(i)]);
      }
      bfly_inv<R>(v);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) buf[swz(base + i * s)] = v[i];
  }
}

// Copy the octant table (M/8 + 1 entries) from global into shared memory.
S2W_DEV void load_octant(double2* __restrict__ s_oct, const double2* __restrict__ g_oct, int logM) {
  const int n = (1 << (logM - 3)) + 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_oct[oct_slot(i)] = __ldg(&g_oct[i]);
}

// Forward DIF FFT: natural -> bit-reversed.  Ends with a __syncthreads.
// Precondition: the row is fully written and visible (caller synced).
S2W_DEV void fft_fwd(double2* buf, int logM, const double2* __restrict__ tw, int gtid,
                     int gsize) {
  // tw: shared-memory octant table (load_octant)
  int ls = logM;
  while (ls >= 3) {
    ls -= 3;
    fft_pass<8, false>(buf, logM, ls, tw, gtid, gsize);
    __syncthreads();
  }
  if (ls == 2) {
    fft_pass<4, false>(buf, logM, 0, tw, gtid, gsize);
    __syncthreads();
  } else if (ls == 1) {
    fft_pass<2, false>(buf, logM, 0, tw, gtid, gsize);
    __syncthreads();
  }
}

// Inverse (adjoint) DIT FFT: bit-reversed -> natural, unnormalised.
S2W_DEV void fft_inv(double2* buf, int logM, const double2* __restrict__ tw, int gtid,
                     int gsize) {
  const int rem = logM % 3;
  int ls = 0;
  if (rem == 2) {
    fft_pass<4, true>(buf, logM, 0, tw, gtid, gsize);
    __syncthreads();
    ls = 2;
  } else if (rem == 1) {
    fft_pass<2, true>(buf, logM, 0, tw, gtid, gsize);
    __syncthreads();
    ls = 1;
  }
  while (ls < logM) {
    fft_pass<8, true>(buf, logM, ls, tw, gtid, gsize);
    __syncthreads();
    ls += 3;
  }
}

// buf[p] *= tab[p] for all p (tab stored in the same bit-reversed order).
// Unrolled so that 8 table loads per thread are in flight at once.
S2W_DEV void pointwise_mul(double2* buf, int M, const double2* __restrict__ tab, int gtid,
                           int gsize) {
  for (int p0 = gtid; p0 < M; p0 += 8 * gsize) {
    double2 t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = p0 + u * gsize;
      t[u] = (p < M) ? __ldg(&tab[p]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = p0 + u * gsize;
      if (p < M) buf[swz(p)] = cmul(buf[swz(p)], t[u]);
    }
  }
}

// Cyclic convolution core: forward DIF FFT, pointwise product with the
// bit-reversed table, inverse DIT FFT -- with the last forward pass, the
// product and the first inverse pass (all of span 1 over blocks of R
// contiguous elements, no twiddles) fused into one shared-memory pass.
// Precondition: row written and synced.  Ends with a __syncthreads.
template <int R>
S2W_DEV void conv_core_pass(double2* __restrict__ buf, int M, const double2* __restrict__ tab,
                            int gtid, int gsize) {
  for (int b = gtid; b < M / R; b += gsize) {
    double2 v[R], t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = __ldg(&tab[b * R + i]);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[swz(b * R + i)];
    bfly_fwd<R>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = cmul(v[i], t[i]);
    bfly_inv<R>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) buf[swz(b * R + i)] = v[i];
  }
}

S2W_DEV void fft_conv(double2* buf, int logM, const double2* __restrict__ oct,
                      const double2* __restrict__ tab, int gtid, int gsize) {
  const int M = 1 << logM;
  const int rem = logM % 3;
  const int lastR = rem == 0 ? 8 : (1 << rem);
  const int lastl = rem == 0 ? 3 : rem;
  // forward: radix-8 passes down to span lastR
  for (int ls = logM - 3; ls >= lastl; ls -= 3) {
    fft_pass<8, false>(buf, logM, ls, oct, gtid, gsize);
    __syncthreads();
  }
  if (lastR == 8) conv_core_pass<8>(buf, M, tab, gtid, gsize);
  else if (lastR == 4) conv_core_pass<4>(buf, M, tab, gtid, gsize);
  else conv_core_pass<2>(buf, M, tab, gtid, gsize);
  __syncthreads();
  for (int ls = lastl; ls < logM; ls += 3) {
    fft_pass<8, true>(buf, logM, ls, oct, gtid, gsize);
    __syncthreads();
  }
}
