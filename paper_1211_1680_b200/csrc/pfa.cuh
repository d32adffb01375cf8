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

// One axis pass: every line of axis P (stride N/P) through dft_odd.
template <int P, bool INV>
S2W_DEV void pfa_pass(double2* __restrict__ buf, int tid, int nthr) {
  constexpr int A = PFA_N / P;  // also the number of lines
  for (int r = tid; r < A; r += nthr) {
    double2 v[P];
    int idx[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      int i = P * r + j * A;
      if (i >= PFA_N) i -= PFA_N;
      idx[j] = i;
      v[j] = buf[i];
    }
    dft_odd<P, INV>(v);
#pragma unroll
    for (int j = 0; j < P; ++j) buf[idx[j]] = v[j];
  }
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
