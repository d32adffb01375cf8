// Prime-factor (Good-Thomas) DFT of length N = 4095 = 13 * 7 * 5 * 9 in
// shared memory: the odd ring / theta transform length 2L-1 at L = 2048.
//
// The coprime factors make the 1-D DFT a 4-D DFT with no twiddle factors:
// the element with input index n sits at shared-memory slot n (natural
// order) and has coordinate n_i = (n mod P_i) * (N/P_i)^-1 mod P_i along
// axis i, so the P_i elements of an axis-i line are the slots
// (P_i r + j N/P_i) mod N, j = 0..P_i-1, already in coordinate order.  After
// the four axis passes (in-place small DFTs) slot n holds the output bin k
// whose CRT residues equal n's coordinates:
//     X[k] sits at pfa_pos(k) = sum_i (k mod P_i) (N/P_i)  mod N.
// This replaces the Bluestein chirp-z convolution (two 8192-point FFTs per
// 4095-point DFT) by ~60 flops per point over four shared-memory passes.
// Line strides P_i * 16 bytes with P_i odd keep every quarter-warp's 16-byte
// accesses on distinct bank groups.
//
// Small DFTs of odd length P use the conjugate-pair form:
//     X_k     = x_0 + sum_j (x_j + x_{P-j}) cos(2 pi jk/P) - i (x_j - x_{P-j}) sin(2 pi jk/P)
//     X_{P-k} = same with +i,
// with the cos/sin values as compile-time immediates (correctly rounded).
#pragma once
#include "common.cuh"

constexpr int PFA_N = 4095;

template <int P>
struct PfaTrig;
template <>
struct PfaTrig<5> {
  static S2W_DEV constexpr double c(int r) {
    return r == 0 ? 1.0
                    : r == 1 ? 0.30901699437494745
                    : r == 2 ? -0.8090169943749475
                    : r == 3 ? -0.8090169943749475 : 0.30901699437494745;
  }
  static S2W_DEV constexpr double s(int r) {
    return r == 0 ? 0.0
                    : r == 1 ? 0.9510565162951535
                    : r == 2 ? 0.5877852522924731
                    : r == 3 ? -0.5877852522924731 : -0.9510565162951535;
  }
};
template <>
struct PfaTrig<7> {
  static S2W_DEV constexpr double c(int r) {
    return r == 0 ? 1.0
                    : r == 1 ? 0.6234898018587335
                    : r == 2 ? -0.2225209339563144
                    : r == 3 ? -0.9009688679024191
                    : r == 4 ? -0.9009688679024191
                    : r == 5 ? -0.2225209339563144 : 0.6234898018587335;
  }
  static S2W_DEV constexpr double s(int r) {
    return r == 0 ? 0.0
                    : r == 1 ? 0.7818314824680298
                    : r == 2 ? 0.9749279121818236
                    : r == 3 ? 0.4338837391175581
                    : r == 4 ? -0.4338837391175581
                    : r == 5 ? -0.9749279121818236 : -0.7818314824680298;
  }
};
template <>
struct PfaTrig<9> {
  static S2W_DEV constexpr double c(int r) {
    return r == 0 ? 1.0
                    : r == 1 ? 0.766044443118978
                    : r == 2 ? 0.17364817766693036
                    : r == 3 ? -0.5
                    : r == 4 ? -0.9396926207859084
                    : r == 5 ? -0.9396926207859084
                    : r == 6 ? -0.5
                    : r == 7 ? 0.17364817766693036 : 0.766044443118978;
  }
  static S2W_DEV constexpr double s(int r) {
    return r == 0 ? 0.0
                    : r == 1 ? 0.6427876096865394
                    : r == 2 ? 0.984807753012208
                    : r == 3 ? 0.8660254037844386
                    : r == 4 ? 0.3420201433256687
                    : r == 5 ? -0.3420201433256687
                    : r == 6 ? -0.8660254037844386
                    : r == 7 ? -0.984807753012208 : -0.6427876096865394;
  }
};
template <>
struct PfaTrig<13> {
  static S2W_DEV constexpr double c(int r) {
    return r == 0 ? 1.0
                    : r == 1 ? 0.8854560256532099
                    : r == 2 ? 0.5680647467311558
                    : r == 3 ? 0.12053668025532305
                    : r == 4 ? -0.3546048870425356
                    : r == 5 ? -0.7485107481711011
                    : r == 6 ? -0.970941817426052
                    : r == 7 ? -0.970941817426052
                    : r == 8 ? -0.7485107481711011
                    : r == 9 ? -0.3546048870425356
                    : r == 10 ? 0.12053668025532305
                    : r == 11 ? 0.5680647467311558 : 0.8854560256532099;
  }
  static S2W_DEV constexpr double s(int r) {
    return r == 0 ? 0.0
                    : r == 1 ? 0.46472317204376856
                    : r == 2 ? 0.8229838658936564
                    : r == 3 ? 0.992708874098054
                    : r == 4 ? 0.9350162426854148
                    : r == 5 ? 0.6631226582407952
                    : r == 6 ? 0.23931566428755777
                    : r == 7 ? -0.23931566428755777
                    : r == 8 ? -0.6631226582407952
                    : r == 9 ? -0.9350162426854148
                    : r == 10 ? -0.992708874098054
                    : r == 11 ? -0.8229838658936564 : -0.46472317204376856;
  }
};

// In-place DFT of odd length P in registers (INV: exp(+2 pi i nk/P), unnormalised).
template <int P, bool INV>
S2W_DEV void dft_odd(double2* v) {
  constexpr int H = (P - 1) / 2;
  double2 a[H], b[H];
  const double2 x0 = v[0];
  double2 s0 = x0;
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    a[j - 1] = cadd(v[j], v[P - j]);
    b[j - 1] = csub(v[j], v[P - j]);
    s0 = cadd(s0, a[j - 1]);
  }
  v[0] = s0;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const double c = PfaTrig<P>::c((j * k) % P), s = PfaTrig<P>::s((j * k) % P);
      A.x = fma(a[j - 1].x, c, A.x);
      A.y = fma(a[j - 1].y, c, A.y);
      B.x = fma(b[j - 1].x, s, B.x);
      B.y = fma(b[j - 1].y, s, B.y);
    }
    // forward: X_k = A - iB, X_{P-k} = A + iB (inverse: swapped)
    const double2 lo = make_double2(A.x + B.y, A.y - B.x);
    const double2 hi = make_double2(A.x - B.y, A.y + B.x);
    v[k] = INV ? hi : lo;
    v[P - k] = INV ? lo : hi;
  }
}

// DFT of length P in registers: the conjugate-pair form for odd P, the
// butterfly for P = 2.
template <int P, bool INV>
S2W_DEV void dft_p(double2* v) {
  if constexpr (P == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else {
    dft_odd<P, INV>(v);
  }
}

// One axis pass of a length-NN prime-factor DFT: every line of axis P
// (slots (P r + j NN/P) mod NN) through dft_p.
template <int NN, int P, bool INV>
S2W_DEV void pfa_pass_n(double2* __restrict__ buf, int tid, int nthr) {
  constexpr int A = NN / P;  // also the number of lines
  for (int r = tid; r < A; r += nthr) {
    double2 v[P];
    int idx[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      int i = P * r + j * A;
      if (i >= NN) i -= NN;
      idx[j] = i;
      v[j] = buf[i];
    }
    dft_p<P, INV>(v);
#pragma unroll
    for (int j = 0; j < P; ++j) buf[idx[j]] = v[j];
  }
}
template <int P, bool INV>
S2W_DEV void pfa_pass(double2* __restrict__ buf, int tid, int nthr) {
  pfa_pass_n<PFA_N, P, INV>(buf, tid, nthr);
}

// pfa_pass_n whose input comes from src(i, g) (element i of the row to be
// transformed; g = j * (NN / P) + r its position in gather order, contiguous
// across the threads) instead of buf[i]: every line of axis P is gathered into
// registers, then -- after a barrier, so src may read buf itself -- transformed
// and written to its slots.  Replaces a separate staging pass of the row
// through shared memory.  Not synced at the end.
template <int NN, int P, bool INV, int T, class Src>
S2W_DEV void pfa_pass_gather(double2* __restrict__ buf, int tid, Src src) {
  constexpr int A = NN / P;              // number of lines
  constexpr int RR = (A + T - 1) / T;    // lines per thread
  double2 v[RR][P];
#pragma unroll
  for (int rr = 0; rr < RR; ++rr) {
    const int r = tid + rr * T;
    if (RR * T != A && r >= A) break;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      int i = P * r + j * A;
      if (i >= NN) i -= NN;
      v[rr][j] = src(i, j * A + r);
    }
  }
  __syncthreads();
#pragma unroll
  for (int rr = 0; rr < RR; ++rr) {
    const int r = tid + rr * T;
    if (RR * T != A && r >= A) break;
    dft_p<P, INV>(v[rr]);
#pragma unroll
    for (int j = 0; j < P; ++j) {
      int i = P * r + j * A;
      if (i >= NN) i -= NN;
      buf[i] = v[rr][j];
    }
  }
}

// pfa4095 with the row supplied by src (see pfa_pass_gather): the axis-9 pass
// comes first (455 lines: two per thread at T = 256, 18 values in registers),
// the axes commute.  Every thread may still be reading buf through src on
// entry.  Ends synced.
template <bool INV, int T, class Src>
S2W_DEV void pfa4095_from(double2* buf, int tid, Src src) {
  pfa_pass_gather<PFA_N, 9, INV, T>(buf, tid, src);
  __syncthreads();
  pfa_pass<13, INV>(buf, tid, T);
  __syncthreads();
  pfa_pass<7, INV>(buf, tid, T);
  __syncthreads();
  pfa_pass<5, INV>(buf, tid, T);
  __syncthreads();
}

// Slot of output bin k after pfa4095: sum_i (k mod P_i)(N/P_i) mod N, and
// since P_i (N/P_i) = N that is k * sum_i N/P_i = 2174 k (mod N).  Additive:
// pfa_pos(k + d) = pfa_pos(k) + pfa_pos(d) (mod N).
constexpr int PFA_STEP = 315 + 585 + 819 + 455;  // 2174
S2W_DEV int pfa_pos(int k) { return (int)(((unsigned)k * (unsigned)PFA_STEP) % (unsigned)PFA_N); }
S2W_DEV int pfa_next(int pos, int dpos) {
  const int p = pos + dpos;
  return p >= PFA_N ? p - PFA_N : p;
}

// Unnormalised DFT_4095 of buf[0..4095) (natural order in, pfa_pos order out).
// Precondition: input written and synced.  Ends synced.
template <bool INV>
S2W_DEV void pfa4095(double2* buf, int tid, int nthr) {
  pfa_pass<13, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass<7, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass<5, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass<9, INV>(buf, tid, nthr);
  __syncthreads();
}

// ------------------------------------------------------------------ N = 8191 (L = 4096)
// 8191 is prime, so its DFT is Rader's: with the primitive root g = 17,
//     X_0 = sum_n x_n,   X_{g^-p} = x_0 + sum_q x_{g^q} w^{g^(q-p)},
// the second term a cyclic convolution of length 8190 = 2 * 9 * 5 * 7 * 13
// (a_q = x_{g^q} with d_j = w^{g^-j}), done by the prime-factor engine:
// forward PFA_8190 (natural order in, bin k at slot 253 k mod 8190 out),
// product with the precomputed spectrum of d stored in that slot order (and
// divided by 8190), inverse PFA_8190 (slot order in, natural order out).
// No permutation passes: the input gather g^q and the output map
// bin g^-p -> p are table lookups.  The inverse DFT is conj(DFT(conj x)).
constexpr int RADER_N = 8191, RADER_M = 8190, RADER_G = 17;
constexpr int RADER_STEP = 4095 + 910 + 1638 + 1170 + 630 - RADER_M;  // 253: slot of bin k = 253 k

template <bool INV>
S2W_DEV void pfa8190(double2* buf, int tid, int nthr) {
  pfa_pass_n<RADER_M, 13, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass_n<RADER_M, 7, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass_n<RADER_M, 5, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass_n<RADER_M, 9, INV>(buf, tid, nthr);
  __syncthreads();
  pfa_pass_n<RADER_M, 2, INV>(buf, tid, nthr);
  __syncthreads();
}

struct RaderTabs {
  const int* gpow;   // [8190] g^q mod 8191
  const int* plog;   // [8191] bin g^-p -> p (bin 0 unused)
  const double2* D;  // [8190] DFT_8190(d)_k / 8190 at slot 253 k mod 8190
};

// DFT_8191 (INV: unnormalised inverse) of buf[0, 8191) (natural order,
// written and synced) by T threads.  Leaves the convolution in buf[0, 8190)
// and returns x_0 and X_0 (of the conjugated input when INV); the outputs are
// then rader_bin(...).  s_part: T/32 double2 of shared scratch.  Ends synced.
//
// rader8191_from: the row comes from src(n, g) (sample n; g = its position in
// gather order, n = g^q at g = q and n = 0 at g = RADER_M) instead of buf[n];
// src may read buf (all reads precede the first barrier).
template <int T, bool INV, class Src>
S2W_DEV void rader8191_from(double2* buf, const RaderTabs& R, double2* s_part, double2& x0, double2& X0,
                            Src src) {
  constexpr int U = (RADER_M + T - 1) / T;
  const int tid = threadIdx.x;
  double2 v[U];
  double2 sum = make_double2(0.0, 0.0);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int q = tid + u * T;
    v[u] = make_double2(0.0, 0.0);
    if (q < RADER_M) {
      v[u] = src(__ldg(&R.gpow[q]), q);
      if (INV) v[u] = cconj(v[u]);
      sum = cadd(sum, v[u]);  // every n >= 1 is some g^q exactly once
    }
  }
  x0 = src(0, RADER_M);
  if (INV) x0 = cconj(x0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum.x += __shfl_xor_sync(0xffffffffu, sum.x, o);
    sum.y += __shfl_xor_sync(0xffffffffu, sum.y, o);
  }
  __syncthreads();
  if ((tid & 31) == 0) s_part[tid >> 5] = sum;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int q = tid + u * T;
    if (q < RADER_M) buf[q] = v[u];
  }
  __syncthreads();
  X0 = x0;
  for (int w = 0; w < T / 32; ++w) X0 = cadd(X0, s_part[w]);
  pfa8190<false>(buf, tid, T);
  for (int s = tid; s < RADER_M; s += T) buf[s] = cmul(buf[s], __ldg(&R.D[s]));
  __syncthreads();
  pfa8190<true>(buf, tid, T);
}

template <int T, bool INV>
S2W_DEV void rader8191(double2* buf, const RaderTabs& R, double2* s_part, double2& x0, double2& X0) {
  rader8191_from<T, INV>(buf, R, s_part, x0, X0, [&](int n, int) { return buf[n]; });
}

// Output bin b of rader8191 (conjugated back when INV).
template <bool INV>
S2W_DEV double2 rader_bin(const double2* buf, const RaderTabs& R, double2 x0, double2 X0, int b) {
  const double2 y = b ? cadd(x0, buf[__ldg(&R.plog[b])]) : X0;
  return INV ? cconj(y) : y;
}
