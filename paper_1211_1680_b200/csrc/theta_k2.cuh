// The MW theta stage pieces shared by fft_kernels.cu (theta kernels) and
// legendre_kernels.cu (the Legendre analysis with the theta stage fused in):
// parity pairs of theta columns and the N = 4095 (L = 2048) column-pair
// transform theta_k2_row (see fft_kernels.cu, "k2").
#pragma once
#include "fft.cuh"
#include "pfa.cuh"
#include "s2w_internal.h"

namespace s2w {

// ---------------------------------------------------------------- MW theta stage
// Parity pairing: the operator (extension -> band-limited |sin| product ->
// first k rings) commutes with the reflection R: n -> N-1-n.  An even-m row
// x is extended evenly, an odd-m row y oddly, except at the pole sample n=k-1
// (its own mirror) where both keep their value.  So z = x~ + y~ is transformed
// once and split: with delta = y(k-1) and r = response to a unit pole sample
// (even), the even part of the result is H_x + delta r and the odd part is
// H_y - delta r.
struct ThetaPair {
  const double2* ge;  // even-m input row (nullptr: none)
  const double2* go;  // odd-m input row
  double2* he;
  double2* ho;
  double2 delta;      // odd row's pole sample
};

S2W_DEV ThetaPair theta_pair(const ThetaArgs& a, int row, bool valid) {
  ThetaPair P{nullptr, nullptr, nullptr, nullptr, make_double2(0.0, 0.0)};
  if (!valid) return P;
  const int set = row / a.n_pairs, pi = row - set * a.n_pairs;
  const int2 pr = a.pairs[pi];
  const size_t base = (size_t)set * a.n_bins;
  if (pr.x >= 0) {
    P.ge = a.in + (base + pr.x) * a.k;
    P.he = a.out + (base + pr.x) * a.k;
  }
  if (pr.y >= 0) {
    P.go = a.in + (base + pr.y) * a.k;
    P.ho = a.out + (base + pr.y) * a.k;
    P.delta = __ldg(&P.go[a.k - 1]);
  }
  return P;
}

// extended sample n < N of the paired row
S2W_DEV double2 theta_ext(const ThetaPair& P, int n, int k) {
  const bool lo = n < k;
  const int src = lo ? n : 2 * k - 2 - n;
  const double2 e = P.ge ? __ldg(&P.ge[src]) : make_double2(0.0, 0.0);
  const double2 o = P.go ? __ldg(&P.go[src]) : make_double2(0.0, 0.0);
  return lo ? cadd(e, o) : csub(e, o);
}

// write ring t < k from w_t = result(t), w_r = result(N-1-t)
S2W_DEV void theta_store(const ThetaPair& P, const ThetaArgs& a, int t, double2 wt, double2 wr) {
  const double2 r = a.pole_resp ? __ldg(&a.pole_resp[t]) : make_double2(0.0, 0.0);
  const double2 dr = cmul(P.delta, r);
  if (P.he) P.he[t] = csub(cscale(cadd(wt, wr), 0.5), dr);
  if (P.ho) P.ho[t] = cadd(cscale(csub(wt, wr), 0.5), dr);
}


constexpr int K2_N = 4095, K2_M = 4096, K2_K = 2048;
constexpr int K2_NTW = 272;  // fft_ntw(12)
static_assert(K2_NTW == fft_ntw(12), "4096-point pass twiddles");

constexpr size_t k2_theta_smem_bytes() { return ((size_t)K2_M + K2_K + K2_NTW) * 16 + 16; }

// Arm the barrier and issue the bulk copies of the 4096-point pass twiddles
// and a theta column pair (ge -> dst[0, k), go -> dst[k, 2k)).
S2W_DEV void k2_issue(uint64_t* mb, double2* tw, const double2* gtw, double2* dst, const double2* ge,
                      const double2* go) {
  constexpr unsigned col = K2_K * 16u;
  mbar_init(mb, 1);
  mbar_expect_tx(mb, K2_NTW * 16u + (ge ? col : 0u) + (go ? col : 0u));
  bulk_g2s(tw, gtw, K2_NTW * 16u, mb);
  if (ge) bulk_g2s(dst, ge, col, mb);
  if (go) bulk_g2s(dst + K2_K, go, col, mb);
}

// Steps 3-8 of the theta column-pair transform on an engine of M = 2^LOGM
// points (N = M - 1 MW samples on the circle, k = M/2 rings, T = M/16
// threads): the Fourier coefficients a_q = X_bin e^{-i pi q/N} / N (X_bin =
// bin_value(bin), the DFT_N of the extended pair) split by the parity of q,
// the two parity-class |sin| convolutions, the evaluation input and the
// length-M FFT on the analysis rings.  On return buf holds that FFT
// (bit-reversed, swizzled) and every thread is synced.
//
// Thread tid owns the elements tid + T kk (kk = 0..15) of every outer
// radix-16 pass (span T), so the data movement between the transforms runs in
// the registers of those passes:
//  * 3 -> 4: even q = 2a is element a (mod M) of the even-class row, odd
//    q = 2a+1 goes to side slot a (mod k).  The thread gathers the elements
//    tid + T kk of both classes (|a| < M/4: kk in 0..3 and 12..15, the rest
//    is the zero padding) and feeds the even ones to its first butterfly: no
//    zero fill, no extra trip through shared memory.
//  * 4 -> 5 -> 6: the last inverse pass of the even class (H'(2a) at element
//    a), the class swap (even outputs -> side, odd coefficients -> buf) and
//    the first forward pass of the odd class, with no barrier in between.
//  * 7 -> 8: X'_n = conj(H'(q)) e^{-i pi q/M}, n = q mod M, is gathered as
//    element tid + T u: the input of the first butterfly of the FFT.
// x: 16 registers of scratch.  Precondition: bin_value's source written and
// synced, side unused.
template <int LOGM, int T, class Bin>
S2W_DEV void theta_classes(double2* buf, double2* side, const double2* tw, const FftTablesDev& F,
                           const double* __restrict__ wtab, double2* x, Bin bin_value) {
  constexpr int M = 1 << LOGM, k = M / 2, N = M - 1;
  static_assert(T == M / 16, "one outer radix-16 butterfly per thread");
  const int tid = threadIdx.x;
  const int sb = swz(tid);
  {
    // (side is free until here: the odd class goes there at once)
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      if (kk >= 4 && kk < 12) {
        x[kk] = make_double2(0.0, 0.0);
        continue;
      }
      const int aa = tid + T * kk - (kk < 4 ? 0 : M);  // [-M/4, M/4)
      const int be = 2 * aa + (aa < 0 ? N : 0);        // bin of q = 2 aa
      const int bo = be + 1;                           // bin of q = 2 aa + 1
      x[kk] = aa > -(M / 4) ? cmul(bin_value(be), __ldg(&F.phA[be])) : make_double2(0.0, 0.0);
      side[(tid + T * kk) & (k - 1)] = cmul(bin_value(bo), __ldg(&F.phA[bo]));
    }
    __syncthreads();
    bfly16<false>(x, tw[tid]);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) buf[sb ^ swz(kk * T)] = x[kk];
  }
  __syncthreads();
  fft_conv_real_inner<LOGM, T>(buf, tw, wtab, tid);
  {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) x[kk] = buf[sb ^ swz(kk * T)];
    const double2 u = tw[tid];
    bfly16<true>(x, u);  // x[kk] = H'(2a), a = tid + T kk (mod M)
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      if (kk >= 4 && kk < 12) {
        x[kk] = make_double2(0.0, 0.0);  // |a| >= M/4: not needed / zero padding
      } else {
        const int sl = (tid + T * kk) & (k - 1);
        const double2 od = side[sl];
        side[sl] = x[kk];
        x[kk] = od;
      }
    }
    bfly16<false>(x, u);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) buf[sb ^ swz(kk * T)] = x[kk];
  }
  __syncthreads();
  fft_conv_real_inner<LOGM, T>(buf, tw, wtab, tid);
  pass16<LOGM, T, LOGM - 4, true>(buf, tw, tid);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int n = tid + u * T;
    const int q = n < k ? n : n - M;
    double2 h = make_double2(0.0, 0.0);
    if (q > -k) h = (q & 1) ? buf[swz(((q - 1) >> 1) & (M - 1))] : side[(q >> 1) & (k - 1)];
    x[u] = cmul(cconj(h), __ldg(&F.ph2d[n]));
  }
  __syncthreads();
  fft_fwd_from_regs<LOGM, T>(buf, tw, x, tid);
}

// One theta column pair (row `row` of a) on the CTA's T threads.  smem:
// k2_theta_smem_bytes() of 16-byte aligned shared memory.  pf > 0: also
// prefetch row + pf into L2.  Precondition: every thread is done with smem
// (a barrier) and, if smem held generic-proxy writes, each writer executed
// fence_proxy_async() before that barrier.  Ends with the stores issued.
template <int T>
S2W_DEV void theta_k2_row(const ThetaArgs& a, int row, double2* smem, int pf) {
  double2* buf = smem;               // [4096]
  double2* side = smem + K2_M;       // [2048]
  double2* tw = side + K2_K;         // [272]
  uint64_t* mb = reinterpret_cast<uint64_t*>(tw + K2_NTW);
  constexpr int k = K2_K, U = K2_M / T;
  const FftTablesDev& F = a.T;
  const int tid = threadIdx.x;
  bool has_e, has_o;
  {
    // (the pair is re-read for the stores: nothing stays live across the FFTs)
    const ThetaPair P = theta_pair(a, row, true);
    has_e = P.ge != nullptr;
    has_o = P.go != nullptr;
    if (tid == 0) {
      k2_issue(mb, tw, F.tw12, buf, P.ge, P.go);
      if (pf) {
        const ThetaPair Pn = theta_pair(a, row + pf, true);
        if (Pn.ge) bulk_prefetch_l2(Pn.ge, K2_K * 16u);
        if (Pn.go) bulk_prefetch_l2(Pn.go, K2_K * 16u);
      }
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
  // 1-2. DFT_N of the parity extension to the full circle: the extended
  //      samples are formed in the gather of the first prime-factor pass
  double2 x[U];
  pfa4095_from<false, T>(buf, tid, [&](int n, int) {
    const bool lo = n < k;
    const int src = lo ? n : 2 * k - 2 - n;
    const double2 e = has_e ? buf[src] : make_double2(0.0, 0.0);
    const double2 o = has_o ? buf[k + src] : make_double2(0.0, 0.0);
    return lo ? cadd(e, o) : csub(e, o);
  });
  // 3-8. coefficient split, parity-class convolutions, evaluation FFT (N2 = 4096)
  static_assert(U == 16, "theta_classes scratch");
  theta_classes<12, T>(buf, side, tw, F, F.w2s, x, [&](int bin) { return buf[pfa_pos(bin)]; });
  // rings j and N2-1-j, split by parity
  const ThetaPair P = theta_pair(a, row, true);
#pragma unroll 4
  for (int t = tid; t < k; t += T) {
    const double2 wt = cconj(buf[swz(fft_brev<12>(t))]);
    const double2 wr = cconj(buf[swz(fft_brev<12>(K2_M - 1 - t))]);
    theta_store(P, a, t, wt, wr);
  }
}


}  // namespace s2w
