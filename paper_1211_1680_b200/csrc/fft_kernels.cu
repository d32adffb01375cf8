// Ring (phi) FFT and MW theta-stage kernels.
//
//  phi_fwd_kernel : map rows (theta-major) -> G_m(theta_t) = DFT_N(row)/N, written
//                   m-major ([mi][t]) so the theta stage and the Legendre
//                   analysis read contiguous columns.  Replaces the np.fft.fft /
//                   rfft calls of sh_analysis_stack (sht.py:322,335).
//  phi_inv_kernel : G ring-major ([t][mi]) -> map rows, unnormalised inverse DFT
//                   (np.fft.ifft/irfft with norm="forward", sht.py:266-273), plus the
//                   MW south-pole pinning of sht.py:274-279.
//  theta_kernel   : MW forward theta stage per order m (absent from the reference,
//                   whose MW analysis raises at sht.py:300-303): parity extension to
//                   the full circle, DFT_N, convolution with the Fourier series of
//                   |sin theta|, and evaluation of the result on the L analysis rings
//                   theta''_j = (2j+1) pi / 2L (an inverse DFT of length 2L), which are
//                   symmetric about the equator.  See DESIGN.md.
//
// All odd-length DFTs (N = 2L-1) are Bluestein chirp-z transforms over the
// power-of-two shared-memory FFT in fft.cuh.
#include <algorithm>
#include <stdlib.h>

#include "fft.cuh"
#include "pfa.cuh"
#include "s2w_internal.h"
#include "theta_k2.cuh"

namespace s2w {

// 32-byte store (STG.E.256 on sm_100a): one full sector.  p must be 32-byte aligned.
S2W_DEV void st_global_32(double2* p, double2 lo, double2 hi) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(lo.x), "d"(lo.y), "d"(hi.x),
               "d"(hi.y)
               : "memory");
}
S2W_DEV bool aligned32(const void* p) { return ((uintptr_t)p & 31) == 0; }

// resident CTAs per SM the row kernels are compiled for (register cap):
// two for the 4096-point rows (k = 729 .. 1024 class grids), else one
#ifndef S2W_ROW_MINB12
#define S2W_ROW_MINB12 2
#endif
__host__ __device__ constexpr int fft_minb(int logm) { return (logm >= 10 && logm <= 12) ? S2W_ROW_MINB12 : 1; }

__device__ __forceinline__ double2 load_map_elem(const double* __restrict__ in, long long idx,
                                                 int real) {
  if (real) return make_double2(__ldg(&in[idx]), 0.0);
  return __ldg(reinterpret_cast<const double2*>(in) + idx);
}

// Hard threshold of the denoiser (denoise.py:92): |v| < t -> 0 (t <= 0: no-op;
// complex magnitudes as np.abs, i.e. hypot).
S2W_DEV double hard_thresh(double v, double t) { return fabs(v) < t ? 0.0 : v; }
S2W_DEV double2 hard_thresh(double2 v, double t) {
  return (t > 0.0 && hypot(v.x, v.y) < t) ? make_double2(0.0, 0.0) : v;
}

// ---------------------------------------------------------------- phi forward
template <int LOGM>
__global__ void __launch_bounds__(fft_maxthr(LOGM), fft_minb(LOGM)) phi_fwd_kernel(PhiFwdArgs a) {
  // Real maps: two rings per transform (z = x + i y; X_k = (Z_k + conj Z_{N-k})/2,
  // Y_k = (Z_k - conj Z_{N-k})/2i), halving the FFT work.
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int M = 1 << LOGM, GS = fft_gs(LOGM);
  const int N = T.N;
  const int grp = threadIdx.x / GS, gtid = threadIdx.x % GS;
  double2* buf = smem + (size_t)grp * M;
  double2* tw = smem + (size_t)a.rpc * M;
  load_tw<LOGM>(tw, T.tw);
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;  // transforms per set
  const int row = blockIdx.x * a.rpc + grp;
  const bool valid = row < a.n_sets * per;
  const int set = valid ? row / per : 0;
  const int p = valid ? row - set * per : 0;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && valid && ta + 1 < a.n_rings;
  const long long base_a = ((long long)set * a.n_rings + ta) * N;

  for (int n0 = gtid; n0 < M; n0 += 8 * GS) {
    double2 x[8], c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      const bool in = valid && n < N;
      if (!a.real) {
        x[u] = in ? __ldg(reinterpret_cast<const double2*>(a.in) + base_a + n)
                  : make_double2(0.0, 0.0);
      } else {
        x[u] = make_double2(in ? __ldg(&a.in[base_a + n]) : 0.0,
                            (in && vb) ? __ldg(&a.in[base_a + N + n]) : 0.0);
      }
      c[u] = in ? __ldg(&T.chirp[n]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      if (n < M) buf[swz(n)] = cmul(x[u], c[u]);
    }
  }
  __syncthreads();
  fft_conv<LOGM, GS>(buf, tw, T.bl_fwd, gtid);
  if (!valid) return;
  for (int mi = gtid; mi < a.n_bins; mi += GS) {
    const double2 z = cmul(__ldg(&T.chirp[mi]), buf[swz(mi)]);
    if (!a.real) {
      fwd_row(a, set, mi)[ta] = cscale(z, a.scale);
    } else {
      const int mr = mi ? N - mi : 0;
      const double2 zr = cconj(cmul(__ldg(&T.chirp[mr]), buf[swz(mr)]));
      const double h = 0.5 * a.scale;
      fwd_row(a, set, mi)[ta] = cscale(cadd(z, zr), h);
      if (vb) fwd_row(a, set, mi)[ta + 1] = cscale(cmul_mi(csub(z, zr)), h);
    }
  }
}

// ---------------------------------------------------------------- phi inverse
template <int LOGM>
__global__ void __launch_bounds__(fft_maxthr(LOGM), fft_minb(LOGM)) phi_inv_kernel(PhiInvArgs a) {
  // Real maps: two rings per transform (Z = X + i Y of their Hermitian spectra;
  // the two real rings are Re and Im of the inverse DFT).
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int M = 1 << LOGM, GS = fft_gs(LOGM);
  const int N = T.N;
  const int grp = threadIdx.x / GS, gtid = threadIdx.x % GS;
  double2* buf = smem + (size_t)grp * M;
  double2* tw = smem + (size_t)a.rpc * M;
  load_tw<LOGM>(tw, T.tw);
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x * a.rpc + grp;
  const bool valid = row < a.n_sets * per;
  const int set = valid ? row / per : 0;
  const int p = valid ? row - set * per : 0;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && valid && ta + 1 < a.n_rings;
  const double2* Ga = a.in + ((size_t)set * a.n_rings + ta) * a.n_bins;
  const double2* Gb = Ga + a.n_bins;

  for (int n0 = gtid; n0 < M; n0 += 8 * GS) {
    double2 x[8], c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      x[u] = make_double2(0.0, 0.0);
      c[u] = make_double2(0.0, 0.0);
      if (valid && n < N) {
        if (!a.real) {
          x[u] = __ldg(&Ga[n]);
        } else {
          // Hermitian spectra of the two rings (irfft ignores Im of the DC bin)
          double2 X, Y = make_double2(0.0, 0.0);
          if (n < a.n_bins) {
            X = __ldg(&Ga[n]);
            if (vb) Y = __ldg(&Gb[n]);
            if (n == 0) X.y = Y.y = 0.0;
          } else {
            X = cconj(__ldg(&Ga[N - n]));
            if (vb) Y = cconj(__ldg(&Gb[N - n]));
          }
          x[u] = cadd(X, cmul_pi(Y));
        }
        c[u] = __ldg(&T.chirp[n]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      if (n < M) buf[swz(n)] = cmulc(x[u], c[u]);
    }
  }
  __syncthreads();
  fft_conv<LOGM, GS>(buf, tw, T.bl_inv, gtid);
  if (!valid) return;
  const int pole_ring = (T.N + 1) / 2 - 1 - a.t_offset;  // local index of the MW pole ring
  const bool pa = a.mw_pole && ta == pole_ring, pb = a.mw_pole && vb && ta + 1 == pole_ring;
  const double2 pva = pa ? __ldg(&Ga[0]) : make_double2(0.0, 0.0);
  const double2 pvb = pb ? __ldg(&Gb[0]) : make_double2(0.0, 0.0);
  const size_t ob = ((size_t)set * a.n_rings + ta) * N;
  for (int q = gtid; q < N; q += GS) {
    const double2 v = cmulc(buf[swz(q)], __ldg(&T.chirp[q]));
    if (a.real) {
      a.out[ob + q] = hard_thresh(pa ? pva.x : v.x, a.thresh);
      if (vb) a.out[ob + N + q] = hard_thresh(pb ? pvb.x : v.y, a.thresh);
    } else {
      reinterpret_cast<double2*>(a.out)[ob + q] = hard_thresh(pa ? pva : v, a.thresh);
    }
  }
}

// ---------------------------------------------------------------- phi at N = 4095
// Ring DFTs of length 4095 (L = 2048) by the prime-factor engine (pfa.cuh):
// one ring (or one real ring pair) per CTA, 64 KiB of shared memory, same
// outputs and layouts as phi_fwd_kernel / phi_inv_kernel.
constexpr int PFA_T = 128;

__global__ void __launch_bounds__(PFA_T) phi_fwd_pfa_kernel(PhiFwdArgs a) {
  extern __shared__ double2 smem[];
  double2* buf = smem;
  const int N = PFA_N, tid = threadIdx.x;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x;
  const int set = row / per, p = row - set * per;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && ta + 1 < a.n_rings;
  const long long base_a = ((long long)set * a.n_rings + ta) * N;
  for (int n = tid; n < N; n += PFA_T) {
    double2 x;
    if (!a.real) x = __ldg(reinterpret_cast<const double2*>(a.in) + base_a + n);
    else x = make_double2(__ldg(&a.in[base_a + n]), vb ? __ldg(&a.in[base_a + N + n]) : 0.0);
    buf[n] = x;
  }
  __syncthreads();
  pfa4095<false>(buf, tid, PFA_T);
  for (int mi = tid; mi < a.n_bins; mi += PFA_T) {
    const double2 z = buf[pfa_pos(mi)];
    if (!a.real) {
      fwd_row(a, set, mi)[ta] = cscale(z, a.scale);
    } else {
      const double2 zr = cconj(buf[pfa_pos(mi ? N - mi : 0)]);
      const double h = 0.5 * a.scale;
      const double2 r0 = cscale(cadd(z, zr), h), r1 = cscale(cmul_mi(csub(z, zr)), h);
      double2* o = fwd_row(a, set, mi) + ta;
      if (vb && aligned32(o)) st_global_32(o, r0, r1);  // the ring pair: one sector
      else {
        o[0] = r0;
        if (vb) o[1] = r1;
      }
    }
  }
}

__global__ void __launch_bounds__(PFA_T) phi_inv_pfa_kernel(PhiInvArgs a) {
  extern __shared__ double2 smem[];
  double2* buf = smem;
  const int N = PFA_N, tid = threadIdx.x;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x;
  const int set = row / per, p = row - set * per;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && ta + 1 < a.n_rings;
  const double2* Ga = a.in + ((size_t)set * a.n_rings + ta) * a.n_bins;
  const double2* Gb = Ga + a.n_bins;
  for (int n = tid; n < N; n += PFA_T) {
    double2 x;
    if (!a.real) {
      x = __ldg(&Ga[n]);
    } else {
      double2 X, Y = make_double2(0.0, 0.0);
      if (n < a.n_bins) {
        X = __ldg(&Ga[n]);
        if (vb) Y = __ldg(&Gb[n]);
        if (n == 0) X.y = Y.y = 0.0;
      } else {
        X = cconj(__ldg(&Ga[N - n]));
        if (vb) Y = cconj(__ldg(&Gb[N - n]));
      }
      x = cadd(X, cmul_pi(Y));
    }
    buf[n] = x;
  }
  __syncthreads();
  pfa4095<true>(buf, tid, PFA_T);
  const int pole_ring = (N + 1) / 2 - 1 - a.t_offset;
  const bool pa = a.mw_pole && ta == pole_ring, pb = a.mw_pole && vb && ta + 1 == pole_ring;
  const double2 pva = pa ? __ldg(&Ga[0]) : make_double2(0.0, 0.0);
  const double2 pvb = pb ? __ldg(&Gb[0]) : make_double2(0.0, 0.0);
  const size_t ob = ((size_t)set * a.n_rings + ta) * N;
  for (int q = tid; q < N; q += PFA_T) {
    const double2 v = buf[pfa_pos(q)];
    if (a.real) {
      a.out[ob + q] = hard_thresh(pa ? pva.x : v.x, a.thresh);
      if (vb) a.out[ob + N + q] = hard_thresh(pb ? pvb.x : v.y, a.thresh);
    } else {
      reinterpret_cast<double2*>(a.out)[ob + q] = hard_thresh(pa ? pva : v, a.thresh);
    }
  }
}

// PFA: N = 4095, the DFT_N of step 2 runs on the prime-factor engine
// (natural order in the first 4095 slots, no chirps).
template <int LOGM, bool PFA = false>
__global__ void __launch_bounds__(fft_maxthr(LOGM), fft_minb(LOGM)) theta_kernel(ThetaArgs a) {
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int M = 1 << LOGM, GS = fft_gs(LOGM);
  const int N = T.N, k = a.k;
  const int grp = threadIdx.x / GS, gtid = threadIdx.x % GS;
  double2* buf = smem + (size_t)grp * M;
  double2* tw = smem + (size_t)a.rpc * M;
  load_tw<LOGM>(tw, T.tw);
  const int row = blockIdx.x * a.rpc + grp;
  const bool valid = row < a.n_sets * a.n_pairs;
  const ThetaPair P = theta_pair(a, row, valid);

  // 1. parity extension to the full circle, times the Bluestein chirp
  for (int n0 = gtid; n0 < M; n0 += 8 * GS) {
    double2 x[8], c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      const bool in = valid && n < N;
      x[u] = in ? theta_ext(P, n, k) : make_double2(0.0, 0.0);
      c[u] = in ? (PFA ? make_double2(1.0, 0.0) : __ldg(&T.chirp[n])) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      if (n < M) buf[PFA ? n : swz(n)] = cmul(x[u], c[u]);
    }
  }
  __syncthreads();
  if constexpr (PFA) {
    // 2-3. DFT_N by the prime-factor engine; a_{m'} = X_bin e^{-i pi m'/N} / N
    //      (= ph1 conj(c_bin)), moved to the swizzled length-M circle
    static_assert(!PFA || 8 * GS >= PFA_N, "one pass of register moves");
    pfa4095<false>(buf, gtid, GS);
    double2 av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int bin = gtid + u * GS;
      av[u] = (bin < N) ? cmulc(cmul(buf[pfa_pos(bin)], __ldg(&T.ph1[bin])), __ldg(&T.chirp[bin]))
                        : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int bin = gtid + u * GS;
      if (bin < N) buf[swz(bin < k ? bin : M - N + bin)] = av[u];
    }
  } else {
  // 2. DFT_N (Bluestein)
  fft_conv<LOGM, GS>(buf, tw, T.bl_fwd, gtid);
  // 3. Fourier coefficients a_{m'} = c_bin e^{-i pi m'/N} conv[bin] / N, laid out
  //    over the length-M circle (negative m' at the top)
  for (int b0 = gtid; b0 < N; b0 += 8 * GS) {
    double2 ph[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int bin = b0 + u * GS;
      ph[u] = (bin < N) ? __ldg(&T.ph1[bin]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int bin = b0 + u * GS;
      if (bin >= N) continue;
      const double2 v = cmul(buf[swz(bin)], ph[u]);
      buf[swz(bin < k ? bin : M - N + bin)] = v;
    }
  }
  }
  __syncthreads();
  for (int n = k + gtid; n < M - k + 1; n += GS) buf[swz(n)] = make_double2(0.0, 0.0);
  __syncthreads();
  // 4. convolution with the |sin theta| series (precomputed spectrum)
  fft_conv<LOGM, GS>(buf, tw, T.wconv, gtid);
  // 5. evaluation on the analysis rings theta''_j = (2j+1) pi / N2 (N2 = 2k):
  //    Bluestein input X_n = H'(q) e^{i pi q/N2} conj(c2_n), n = q mod N2.
  //    H'(q) sits at q (q >= 0) and M + q (q < 0); the moves read [M-k+1, M)
  //    and write [k, N2), disjoint.
  //    When N2 = M/2 (k a power of two) the inverse DFT_N2 is a direct
  //    half-size FFT instead: w = conj(DFT_N2(conj X')), X'_n = H'(q) e^{i pi q/N2}.
  const int N2 = T.N2;
  const bool pow2 = 2 * N2 == M;
  const double2* phs = pow2 ? T.ph2d : T.ph2;
  for (int n0 = gtid; n0 < N2; n0 += 8 * GS) {
    double2 ph[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      ph[u] = (n < N2) ? __ldg(&phs[n]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      if (n >= N2) continue;
      double2 v = (n < k) ? buf[swz(n)]
                          : (n > N2 - k ? buf[swz(M - N2 + n)] : make_double2(0.0, 0.0));
      if (pow2) v = cconj(v);
      buf[swz(n)] = cmul(v, ph[u]);
    }
  }
  __syncthreads();
  if (pow2) {
    // 6. direct FFT of length N2 = M/2; rings j and N2-1-j, split by parity
    fft_fwd<LOGM - 1, GS, 1>(buf, tw, gtid);
    if (!valid) return;
    for (int t = gtid; t < k; t += GS) {
      const int tr = N2 - 1 - t;
      const double2 wt = cconj(buf[swz(fft_brev<LOGM - 1>(t))]);
      const double2 wr = cconj(buf[swz(fft_brev<LOGM - 1>(tr))]);
      theta_store(P, a, t, wt, wr);
    }
    return;
  }
  for (int n = N2 + gtid; n < M; n += GS) buf[swz(n)] = make_double2(0.0, 0.0);
  __syncthreads();
  // 6. inverse DFT_N2 (Bluestein); rings j and N2-1-j (its mirror 2 pi - theta''_j),
  //    split by parity
  fft_conv<LOGM, GS>(buf, tw, T.bl_ev, gtid);
  if (!valid) return;
  for (int t = gtid; t < k; t += GS) {
    const int tr = N2 - 1 - t;
    const double2 wt = cmulc(buf[swz(t)], __ldg(&T.chirp2[t]));
    const double2 wr = cmulc(buf[swz(tr)], __ldg(&T.chirp2[tr]));
    theta_store(P, a, t, wt, wr);
  }
}

// ---------------------------------------------------------------- MW synthesis theta stage
// Resampling of a pair (even m, odd m) of columns from the analysis rings
// theta''_j = (2j+1) pi / N2 (N2 = 2k, symmetric, where the Legendre synthesis
// ran) to the MW rings theta_t = (2t+1) pi / N: parity extension to the full
// circle (2 pi - theta''_j = theta''_{N2-1-j}), DFT_N2 -> Fourier coefficients
// b_q (|q| < k, exact: G is a trig polynomial of degree k-1), inverse DFT_N at
// the MW points, parity split via theta_{N-1-t} = 2 pi - theta_t.
S2W_DEV double2 theta_syn_ext(const double2* ge, const double2* go, int n, int k) {
  const bool lo = n < k;
  const int src = lo ? n : 2 * k - 1 - n;
  const double2 e = ge ? __ldg(&ge[src]) : make_double2(0.0, 0.0);
  const double2 o = go ? __ldg(&go[src]) : make_double2(0.0, 0.0);
  return lo ? cadd(e, o) : csub(e, o);
}

struct ThetaSynRow {
  const double2 *ge, *go;
  double2* out;
  int ce, co;  // output columns (-1: none)
};

S2W_DEV ThetaSynRow theta_syn_row(const ThetaSynArgs& a, int row, bool valid) {
  ThetaSynRow R{nullptr, nullptr, nullptr, -1, -1};
  if (!valid) return R;
  const int set = row / a.n_pairs, pi = row - set * a.n_pairs;
  const int2 pr = a.pairs[pi];
  const size_t base = (size_t)set * a.n_bins;
  if (pr.x >= 0) R.ge = a.in + (base + pr.x) * a.k;
  if (pr.y >= 0) R.go = a.in + (base + pr.y) * a.k;
  R.out = a.out + (size_t)set * a.k * a.n_bins;
  R.ce = pr.x;
  R.co = pr.y;
  return R;
}

S2W_DEV void theta_syn_store(const ThetaSynRow& R, const ThetaSynArgs& a, int t, double2 wt,
                             double2 wr) {
  const double2 ve = cscale(cadd(wt, wr), 0.5), vo = cscale(csub(wt, wr), 0.5);
  double2* row = R.out + (size_t)t * a.n_bins;
  // the pair's columns are adjacent bins (theta_pairs): one 32-byte store
  // (a full sector) where the row alignment allows it
  if (R.ce >= 0 && R.co == R.ce + 1 && ((uintptr_t)(row + R.ce) & 31) == 0) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(row + R.ce), "d"(ve.x),
                 "d"(ve.y), "d"(vo.x), "d"(vo.y) : "memory");
  } else if (R.co >= 0 && R.ce == R.co + 1 && ((uintptr_t)(row + R.co) & 31) == 0) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(row + R.co), "d"(vo.x),
                 "d"(vo.y), "d"(ve.x), "d"(ve.y) : "memory");
  } else {
    if (R.ce >= 0) row[R.ce] = ve;
    if (R.co >= 0) row[R.co] = vo;
  }
}

// PFA: N = 4095, the inverse DFT_N of step 4 runs on the prime-factor engine.
template <int LOGM, bool PFA = false>
__global__ void __launch_bounds__(fft_maxthr(LOGM), fft_minb(LOGM)) theta_syn_kernel(ThetaSynArgs a) {
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int M = 1 << LOGM, GS = fft_gs(LOGM);
  const int N = T.N, N2 = T.N2, k = a.k;
  const int grp = threadIdx.x / GS, gtid = threadIdx.x % GS;
  double2* buf = smem + (size_t)grp * M;
  double2* tw = smem + (size_t)a.rpc * M;
  load_tw<LOGM>(tw, T.tw);
  const int row = blockIdx.x * a.rpc + grp;
  const bool valid = row < a.n_sets * a.n_pairs;
  const ThetaSynRow R = theta_syn_row(a, row, valid);

  // 1. parity extension on the 2k analysis points (times the chirp c2 unless
  //    N2 = M/2, where the DFT_N2 is a direct half-size FFT)
  const bool pow2 = 2 * N2 == M;
  for (int n0 = gtid; n0 < M; n0 += 8 * GS) {
    double2 x[8], c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      const bool in = valid && n < N2;
      x[u] = in ? theta_syn_ext(R.ge, R.go, n, k) : make_double2(0.0, 0.0);
      c[u] = in ? (pow2 ? make_double2(1.0, 0.0) : __ldg(&T.chirp2[n])) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + u * GS;
      if (n < M) buf[swz(n)] = cmul(x[u], c[u]);
    }
  }
  __syncthreads();
  // 2. DFT_N2 (Bluestein, or direct)
  if (pow2) fft_fwd<LOGM - 1, GS, 1>(buf, tw, gtid);
  else fft_conv<LOGM, GS>(buf, tw, T.bl_fwd2, gtid);
  // 3. inverse-DFT_N input X_n = DFT_N2[src(n)] ph4[n]; src = n (n < k) or
  //    n + 1 (= N2 + n - N, n >= k): overlapping moves, so all values are read
  //    into registers first (N <= 8 GS)
  double2 xv[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int n = gtid + u * GS;
    xv[u] = make_double2(0.0, 0.0);
    if (n < N) {
      const int src = n < k ? n : n + 1;
      xv[u] = pow2 ? cmul(buf[swz(fft_brev<LOGM - 1>(src))], __ldg(&T.ph4d[n]))
                   : cmul(buf[swz(src)], __ldg(&T.ph4[n]));
    }
  }
  __syncthreads();
  if constexpr (PFA) {
    // 4. inverse DFT_N by the prime-factor engine (input without the Bluestein
    //    chirp conj(c_n) folded into ph4: times c_n); rings t and N-1-t
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = gtid + u * GS;
      if (n < N) buf[n] = cmul(xv[u], __ldg(&T.chirp[n]));
    }
    __syncthreads();
    pfa4095<true>(buf, gtid, GS);
    if (!valid) return;
    for (int t = gtid; t < k; t += GS)
      theta_syn_store(R, a, t, buf[pfa_pos(t)], buf[pfa_pos(N - 1 - t)]);
    return;
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int n = gtid + u * GS;
    if (n < N) buf[swz(n)] = xv[u];
  }
  for (int n = N + gtid; n < M; n += GS) buf[swz(n)] = make_double2(0.0, 0.0);
  __syncthreads();
  // 4. inverse DFT_N (Bluestein) at the MW points; rings t and N-1-t
  fft_conv<LOGM, GS>(buf, tw, T.bl_inv, gtid);
  if (!valid) return;
  for (int t = gtid; t < k; t += GS) {
    const int tr = N - 1 - t;
    const double2 wt = cmulc(buf[swz(t)], __ldg(&T.chirp[t]));
    const double2 wr = cmulc(buf[swz(tr)], __ldg(&T.chirp[tr]));
    theta_syn_store(R, a, t, wt, wr);
  }
}

// =====================================================================
// Split mode for M > 8192 (L > 2048): the length-M cyclic convolution is
// done as two shared-memory FFT pairs of length F = M/2 (DIF first stage
// s_j = a_j + a_{j+F}, d_j = (a_j - a_{j+F}) W_M^j; even / odd spectra),
// with the even half kept in a per-CTA global scratch (L2-resident):
//     y_j = u_j + W_M^-j v_j,   y_{j+F} = u_j - W_M^-j v_j.
// One row per CTA, persistent over rows.  Spectrum tables are stored as
// [even half | odd half], each bit-reversed over F.
// =====================================================================
constexpr int SPLIT_T = 512;

template <int LOGF, class Fill>
S2W_DEV void split_conv(double2* buf, double2* u_out, const double2* __restrict__ tab,
                        const double2* twF, Fill fill) {
  static_assert(fft_gs(LOGF) == SPLIT_T, "split mode runs one engine row per CTA");
  constexpr int F = 1 << LOGF;
  for (int half = 0; half < 2; ++half) {
    fill(half);
    __syncthreads();
    fft_conv<LOGF, SPLIT_T>(buf, twF, tab + half * F, threadIdx.x);
    if (half == 0) {
      for (int j = threadIdx.x; j < F; j += SPLIT_T) u_out[j] = buf[swz(j)];
      __syncthreads();
    }
  }
}

S2W_DEV double2 wM(int j, const double2* octM, int logM) { return twiddle(j, octM, logM); }

template <int LOGF>
__global__ void __launch_bounds__(SPLIT_T) phi_fwd_split_kernel(PhiFwdArgs a) {
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int logM = LOGF + 1, F = 1 << LOGF;
  const int N = T.N;
  double2* buf = smem;
  double2* twF = smem + F;
  double2* octM = twF + ((fft_ntw(LOGF) + 7) & ~7);
  load_tw<LOGF>(twF, T.tw);
  load_octant(octM, T.octM, logM);
  double2* u = a.scratch + (size_t)blockIdx.x * 2 * F;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int n_rows = a.n_sets * per;
  __syncthreads();
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x) {
    const int set = row / per, p = row - set * per;
    const int ta = a.real ? 2 * p : p;
    const bool vb = a.real && ta + 1 < a.n_rings;
    const long long base_a = ((long long)set * a.n_rings + ta) * N;
    split_conv<LOGF>(buf, u, T.bl_fwd, twF, [&](int half) {
      for (int j = threadIdx.x; j < F; j += SPLIT_T) {
        double2 v = make_double2(0.0, 0.0);
        if (j < N) {
          if (!a.real) v = __ldg(reinterpret_cast<const double2*>(a.in) + base_a + j);
          else v = make_double2(__ldg(&a.in[base_a + j]), vb ? __ldg(&a.in[base_a + N + j]) : 0.0);
          v = cmul(v, __ldg(&T.chirp[j]));
          if (half) v = cmul(v, wM(j, octM, logM));
        }
        buf[swz(j)] = v;
      }
    });
    for (int mi = threadIdx.x; mi < a.n_bins; mi += SPLIT_T) {
      const double2 y = cadd(u[mi], cmulc(buf[swz(mi)], wM(mi, octM, logM)));
      const double2 z = cmul(__ldg(&T.chirp[mi]), y);
      if (!a.real) {
        fwd_row(a, set, mi)[ta] = cscale(z, a.scale);
      } else {
        const int mr = mi ? N - mi : 0;
        const double2 yr = cadd(u[mr], cmulc(buf[swz(mr)], wM(mr, octM, logM)));
        const double2 zr = cconj(cmul(__ldg(&T.chirp[mr]), yr));
        const double h = 0.5 * a.scale;
        fwd_row(a, set, mi)[ta] = cscale(cadd(z, zr), h);
        if (vb) fwd_row(a, set, mi)[ta + 1] = cscale(cmul_mi(csub(z, zr)), h);
      }
    }
    __syncthreads();
  }
}

template <int LOGF>
__global__ void __launch_bounds__(SPLIT_T) phi_inv_split_kernel(PhiInvArgs a) {
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int logM = LOGF + 1, F = 1 << LOGF;
  const int N = T.N;
  double2* buf = smem;
  double2* twF = smem + F;
  double2* octM = twF + ((fft_ntw(LOGF) + 7) & ~7);
  load_tw<LOGF>(twF, T.tw);
  load_octant(octM, T.octM, logM);
  double2* u = a.scratch + (size_t)blockIdx.x * 2 * F;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int n_rows = a.n_sets * per;
  const int pole_ring = (T.N + 1) / 2 - 1 - a.t_offset;
  __syncthreads();
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x) {
    const int set = row / per, p = row - set * per;
    const int ta = a.real ? 2 * p : p;
    const bool vb = a.real && ta + 1 < a.n_rings;
    const double2* Ga = a.in + ((size_t)set * a.n_rings + ta) * a.n_bins;
    const double2* Gb = Ga + a.n_bins;
    split_conv<LOGF>(buf, u, T.bl_inv, twF, [&](int half) {
      for (int n = threadIdx.x; n < F; n += SPLIT_T) {
        double2 v = make_double2(0.0, 0.0);
        if (n < N) {
          if (!a.real) {
            v = __ldg(&Ga[n]);
          } else {
            double2 X, Y = make_double2(0.0, 0.0);
            if (n < a.n_bins) {
              X = __ldg(&Ga[n]);
              if (vb) Y = __ldg(&Gb[n]);
              if (n == 0) X.y = Y.y = 0.0;
            } else {
              X = cconj(__ldg(&Ga[N - n]));
              if (vb) Y = cconj(__ldg(&Gb[N - n]));
            }
            v = cadd(X, cmul_pi(Y));
          }
          v = cmulc(v, __ldg(&T.chirp[n]));
          if (half) v = cmul(v, wM(n, octM, logM));
        }
        buf[swz(n)] = v;
      }
    });
    const bool pa = a.mw_pole && ta == pole_ring, pb = a.mw_pole && vb && ta + 1 == pole_ring;
    const double2 pva = pa ? __ldg(&Ga[0]) : make_double2(0.0, 0.0);
    const double2 pvb = pb ? __ldg(&Gb[0]) : make_double2(0.0, 0.0);
    const size_t ob = ((size_t)set * a.n_rings + ta) * N;
    for (int q = threadIdx.x; q < N; q += SPLIT_T) {
      const double2 y = cadd(u[q], cmulc(buf[swz(q)], wM(q, octM, logM)));
      const double2 v = cmulc(y, __ldg(&T.chirp[q]));
      if (a.real) {
        a.out[ob + q] = hard_thresh(pa ? pva.x : v.x, a.thresh);
        if (vb) a.out[ob + N + q] = hard_thresh(pb ? pvb.x : v.y, a.thresh);
      } else {
        reinterpret_cast<double2*>(a.out)[ob + q] = hard_thresh(pa ? pva : v, a.thresh);
      }
    }
    __syncthreads();
  }
}

template <int LOGF>
__global__ void __launch_bounds__(SPLIT_T) theta_split_kernel(ThetaArgs a) {
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int logM = LOGF + 1, F = 1 << LOGF;
  const int N = T.N, k = a.k;
  double2* buf = smem;
  double2* twF = smem + F;
  double2* octM = twF + ((fft_ntw(LOGF) + 7) & ~7);
  load_tw<LOGF>(twF, T.tw);
  load_octant(octM, T.octM, logM);
  double2* u = a.scratch + (size_t)blockIdx.x * 2 * F;   // even-half results
  double2* sv = u + F;                                  // saved row (a_bin, then X_bin)
  const int n_rows = a.n_sets * a.n_pairs;
  __syncthreads();
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x) {
    const ThetaPair P = theta_pair(a, row, true);
    // 1-2. DFT_N of the parity extension (Bluestein)
    split_conv<LOGF>(buf, u, T.bl_fwd, twF, [&](int half) {
      for (int n = threadIdx.x; n < F; n += SPLIT_T) {
        double2 v = make_double2(0.0, 0.0);
        if (n < N) {
          v = cmul(theta_ext(P, n, k), __ldg(&T.chirp[n]));
          if (half) v = cmul(v, wM(n, octM, logM));
        }
        buf[swz(n)] = v;
      }
    });
    // 3. a_bin = y_bin ph1_bin (saved for both halves of the next convolution)
    for (int b = threadIdx.x; b < N; b += SPLIT_T) {
      const double2 y = cadd(u[b], cmulc(buf[swz(b)], wM(b, octM, logM)));
      sv[b] = cmul(y, __ldg(&T.ph1[b]));
    }
    __syncthreads();
    // 4. |sin| convolution of A (A_q = a_q for q < k, A_{M-N+b} = a_b for b >= k)
    split_conv<LOGF>(buf, u, T.wconv, twF, [&](int half) {
      for (int j = threadIdx.x; j < F; j += SPLIT_T) {
        double2 v = make_double2(0.0, 0.0);
        double sign = 1.0;
        if (j < k) {
          v = sv[j];
        } else if (j >= F - k + 1) {
          v = sv[j - F + N];  // A_{j+F}
          sign = -1.0;
        }
        if (half) v = cscale(cmul(v, wM(j, octM, logM)), sign);
        buf[swz(j)] = v;
      }
    });
    // 5. evaluation input on the analysis rings (see theta_kernel):
    //    X_n = H'(q) e^{i pi q/N2} conj(c2_n), q = n (n < k) or n - N2 (n > N2 - k)
    const int N2 = T.N2;
    for (int n = threadIdx.x; n < N2; n += SPLIT_T) {
      double2 h = make_double2(0.0, 0.0);
      if (n < k) {
        h = cadd(u[n], cmulc(buf[swz(n)], wM(n, octM, logM)));
      } else if (n > N2 - k) {
        const int j = F + n - N2;  // position M + q = j + F
        h = csub(u[j], cmulc(buf[swz(j)], wM(j, octM, logM)));
      }
      sv[n] = (N2 == F) ? cmul(cconj(h), __ldg(&T.ph2d[n])) : cmul(h, __ldg(&T.ph2[n]));
    }
    __syncthreads();
    if (2 * N2 == 2 * F) {
      // 6. N2 = F (k a power of two): direct FFT of the engine size,
      //    w = conj(DFT(conj X')), X'_n = X_n / conj(c2_n) stored by step 5 via ph2d
      for (int n = threadIdx.x; n < F; n += SPLIT_T) buf[swz(n)] = sv[n];
      __syncthreads();
      fft_fwd<LOGF, SPLIT_T, 0>(buf, twF, threadIdx.x);
      for (int t = threadIdx.x; t < k; t += SPLIT_T) {
        const int tr = N2 - 1 - t;
        theta_store(P, a, t, cconj(buf[swz(fft_brev<LOGF>(t))]),
                    cconj(buf[swz(fft_brev<LOGF>(tr))]));
      }
    } else {
    // 6. inverse DFT_N2 (Bluestein); rings t and N2-1-t, split by parity
    split_conv<LOGF>(buf, u, T.bl_ev, twF, [&](int half) {
      for (int n = threadIdx.x; n < F; n += SPLIT_T) {
        double2 v = (n < N2) ? sv[n] : make_double2(0.0, 0.0);
        if (half && n < N2) v = cmul(v, wM(n, octM, logM));
        buf[swz(n)] = v;
      }
    });
    for (int t = threadIdx.x; t < k; t += SPLIT_T) {
      const int tr = N2 - 1 - t;
      const double2 zt = cadd(u[t], cmulc(buf[swz(t)], wM(t, octM, logM)));
      const double2 zr = cadd(u[tr], cmulc(buf[swz(tr)], wM(tr, octM, logM)));
      theta_store(P, a, t, cmulc(zt, __ldg(&T.chirp2[t])), cmulc(zr, __ldg(&T.chirp2[tr])));
    }
    }
    __syncthreads();
  }
}

template <int LOGF>
__global__ void __launch_bounds__(SPLIT_T) theta_syn_split_kernel(ThetaSynArgs a) {
  extern __shared__ double2 smem[];
  const FftTablesDev& T = a.T;
  constexpr int logM = LOGF + 1, F = 1 << LOGF;
  const int N = T.N, N2 = T.N2, k = a.k;
  double2* buf = smem;
  double2* twF = smem + F;
  double2* octM = twF + ((fft_ntw(LOGF) + 7) & ~7);
  load_tw<LOGF>(twF, T.tw);
  load_octant(octM, T.octM, logM);
  double2* u = a.scratch + (size_t)blockIdx.x * 2 * F;  // even-half results
  double2* sv = u + F;                                 // saved row (X_n)
  const int n_rows = a.n_sets * a.n_pairs;
  __syncthreads();
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x) {
    const ThetaSynRow R = theta_syn_row(a, row, true);
    if (N2 == F) {
      // 1-2. N2 = F (k a power of two): direct FFT of the engine size
      for (int n = threadIdx.x; n < F; n += SPLIT_T) buf[swz(n)] = theta_syn_ext(R.ge, R.go, n, k);
      __syncthreads();
      fft_fwd<LOGF, SPLIT_T, 0>(buf, twF, threadIdx.x);
      // 3. X_n = DFT_N2[src(n)] ph4d[n]
      for (int n = threadIdx.x; n < N; n += SPLIT_T) {
        const int src = n < k ? n : n + 1;
        sv[n] = cmul(buf[swz(fft_brev<LOGF>(src))], __ldg(&T.ph4d[n]));
      }
      __syncthreads();
    } else {
    // 1-2. DFT_N2 of the parity extension (Bluestein)
    split_conv<LOGF>(buf, u, T.bl_fwd2, twF, [&](int half) {
      for (int n = threadIdx.x; n < F; n += SPLIT_T) {
        double2 v = make_double2(0.0, 0.0);
        if (n < N2) {
          v = cmul(theta_syn_ext(R.ge, R.go, n, k), __ldg(&T.chirp2[n]));
          if (half) v = cmul(v, wM(n, octM, logM));
        }
        buf[swz(n)] = v;
      }
    });
    // 3. X_n = DFT_N2[src(n)] ph4[n]  (src < N2 <= F: the first output half)
    for (int n = threadIdx.x; n < N; n += SPLIT_T) {
      const int src = n < k ? n : n + 1;
      const double2 y = cadd(u[src], cmulc(buf[swz(src)], wM(src, octM, logM)));
      sv[n] = cmul(y, __ldg(&T.ph4[n]));
    }
    __syncthreads();
    }
    // 4. inverse DFT_N (Bluestein); rings t and N-1-t
    split_conv<LOGF>(buf, u, T.bl_inv, twF, [&](int half) {
      for (int n = threadIdx.x; n < F; n += SPLIT_T) {
        double2 v = (n < N) ? sv[n] : make_double2(0.0, 0.0);
        if (half && n < N) v = cmul(v, wM(n, octM, logM));
        buf[swz(n)] = v;
      }
    });
    for (int t = threadIdx.x; t < k; t += SPLIT_T) {
      const int tr = N - 1 - t;
      const double2 zt = cadd(u[t], cmulc(buf[swz(t)], wM(t, octM, logM)));
      const double2 zr = cadd(u[tr], cmulc(buf[swz(tr)], wM(tr, octM, logM)));
      theta_syn_store(R, a, t, cmulc(zt, __ldg(&T.chirp[t])), cmulc(zr, __ldg(&T.chirp[tr])));
    }
    __syncthreads();
  }
}

// =====================================================================
// k2: the N = 4095 (L = 2048) stages, one row (ring, or theta column pair)
// per CTA.  The row arrives by one bulk copy (TMA, cp.async.bulk) completed on
// an mbarrier -- no per-thread load loop -- and every buffer is sized for the
// prime-factor engine (4096 slots = 64 KiB), so two or three CTAs share an SM
// and one CTA's copies overlap another's shared-memory passes.
//  * phi_fwd_k2 / phi_inv_k2: ring DFTs (same I/O as phi_fwd/inv_kernel).
//  * theta_syn_k2: direct 4096-point FFT + prime-factor inverse DFT_4095.
//  * theta_k2: the |sin| convolution on the parity classes of the Fourier
//    index: w_hat(p) vanishes at odd p, so H'(q) = sum_m' a_m' w_hat(q - m')
//    couples only q and m' of equal parity.  Each class is a linear
//    convolution of <= 2048 coefficients whose outputs are needed at <= 2048
//    points, with kernel differences |q - m'|/2 <= 2047: two exact 4096-point
//    cyclic convolutions (kernel w_hat(2d)) replace the 8192-point one and the
//    row fits 96 KiB (two CTAs per SM).
// =====================================================================
#ifndef S2W_K2_T
#define S2W_K2_T 256
#endif
constexpr int K2_T = S2W_K2_T;
#ifndef S2W_K2_TT
#define S2W_K2_TT 256
#endif
constexpr int K2_TT = S2W_K2_TT;  // theta_k2 threads
#ifndef S2W_K2_PFT
#define S2W_K2_PFT S2W_K2_T
#endif
#ifndef S2W_K2_PIT
#define S2W_K2_PIT S2W_K2_T
#endif
// ring-DFT CTA sizes: the prime-factor passes have 315 / 585 / 819 / 455 lines,
// so 320 threads take 1 + 2 + 3 + 2 rounds where 256 take 2 + 3 + 4 + 2
constexpr int K2_PFT = S2W_K2_PFT, K2_PIT = S2W_K2_PIT;
#ifndef S2W_K2_PHI_MINB
#define S2W_K2_PHI_MINB 2
#endif
#ifndef S2W_K2_TSYN_MINB
#define S2W_K2_TSYN_MINB 2
#endif
#ifndef S2W_K2_PHIF_MINB
#define S2W_K2_PHIF_MINB S2W_K2_PHI_MINB
#endif


template <int T>
__global__ void __launch_bounds__(T, S2W_K2_PHIF_MINB) phi_fwd_k2_kernel(PhiFwdArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;
  uint64_t* mb = reinterpret_cast<uint64_t*>(smem + K2_M);
  constexpr int N = K2_N, U = (K2_N + T - 1) / T;
  const int tid = threadIdx.x;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x;
  const int set = row / per, p = row - set * per;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && ta + 1 < a.n_rings;
  const long long base_a = ((long long)set * a.n_rings + ta) * N;
  // rows are contiguous: a complex ring, or a real ring pair (launcher checks alignment)
  const unsigned bytes = a.real ? (vb ? 2u : 1u) * N * 8u : N * 16u;
  if (tid == 0) {
    mbar_init(mb, 1);
    mbar_expect_tx(mb, bytes);
    bulk_g2s(buf, a.in + (a.real ? base_a : 2 * base_a), bytes, mb);
    // the row of the CTA that will take this slot later: HBM stays busy
    const int nrow = row + a.pfd;
    if (a.pfd && nrow < (int)gridDim.x) {
      const int ns = nrow / per, np = nrow - ns * per;
      const long long nb = ((long long)ns * a.n_rings + (a.real ? 2 * np : np)) * N;
      const bool nvb = a.real && 2 * np + 1 < a.n_rings;
      bulk_prefetch_l2(a.in + (a.real ? nb : 2 * nb), a.real ? (nvb ? 2u : 1u) * N * 8u : N * 16u);
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
  if (a.real) {
    // [ring a | ring b] doubles -> interleaved z = a + i b
    const double* r = reinterpret_cast<const double*>(buf);
    double xr[U], xi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int n = tid + u * T;
      xr[u] = n < N ? r[n] : 0.0;
      xi[u] = (n < N && vb) ? r[N + n] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int n = tid + u * T;
      if (n < N) buf[n] = make_double2(xr[u], xi[u]);
    }
    __syncthreads();
  }
  pfa4095<false>(buf, tid, T);
  // Bin mi sits at slot 2174 mi mod N (pfa_pos is additive: the slot advances
  // by pfa_pos(T) per iteration).  Plain [set][bin][ring] output (no shard
  // offset tables): the row pointer advances by T rows per iteration and the
  // loop is unrolled so the shared-memory gathers of four bins are in flight
  // before the first store.
  const bool plain = !a.ofs && !a.peer_q;
  constexpr int dpos = (int)(((unsigned)T * (unsigned)PFA_STEP) % (unsigned)PFA_N);
  if (!a.real && plain) {
    double2* o = a.out + ((size_t)set * a.n_bins + tid) * a.n_rings + ta;
    const size_t step = (size_t)T * a.n_rings;
    const double sc = a.scale;
    int pos = pfa_pos(tid);
#pragma unroll 4
    for (int mi = tid; mi < a.n_bins; mi += T) {
      *o = cscale(buf[pos], sc);
      o += step;
      pos = pfa_next(pos, dpos);
    }
    return;
  }
  if (a.real && plain) {
    double2* o = a.out + ((size_t)set * a.n_bins + tid) * a.n_rings + ta;
    const size_t step = (size_t)T * a.n_rings;
    const double h = 0.5 * a.scale;
    // the ring pair as one 32-byte sector (the row step is a multiple of 32 bytes)
    const bool pair = vb && aligned32(o);
    int pos = pfa_pos(tid);
    int posr = pfa_pos(N - tid);  // slot of the mirror bin N - mi (bin 0: pfa_pos(N) = 0, itself)
#pragma unroll 4
    for (int mi = tid; mi < a.n_bins; mi += T) {
      const double2 z = buf[pos];
      const double2 zr = cconj(buf[posr]);
      const double2 r0 = cscale(cadd(z, zr), h), r1 = cscale(cmul_mi(csub(z, zr)), h);
      if (pair) st_global_32(o, r0, r1);
      else {
        o[0] = r0;
        if (vb) o[1] = r1;
      }
      o += step;
      pos = pfa_next(pos, dpos);
      posr -= dpos;  // bin N - (mi + T)
      if (posr < 0) posr += PFA_N;
    }
    return;
  }
  for (int mi = tid; mi < a.n_bins; mi += T) {
    const double2 z = buf[pfa_pos(mi)];
    if (!a.real) {
      fwd_row(a, set, mi)[ta] = cscale(z, a.scale);
    } else {
      const double2 zr = cconj(buf[pfa_pos(mi ? N - mi : 0)]);
      const double h = 0.5 * a.scale;
      const double2 r0 = cscale(cadd(z, zr), h), r1 = cscale(cmul_mi(csub(z, zr)), h);
      double2* o = fwd_row(a, set, mi) + ta;
      if (vb && aligned32(o)) st_global_32(o, r0, r1);  // the ring pair: one sector
      else {
        o[0] = r0;
        if (vb) o[1] = r1;
      }
    }
  }
}


template <int T>
__global__ void __launch_bounds__(T, S2W_K2_PHI_MINB + 1) phi_inv_k2_kernel(PhiInvArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;
  uint64_t* mb = reinterpret_cast<uint64_t*>(smem + K2_M);
  constexpr int N = K2_N, U = (K2_N + T - 1) / T;
  const int tid = threadIdx.x;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x;
  const int set = row / per, p = row - set * per;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && ta + 1 < a.n_rings;
  const int nb = a.n_bins;
  const double2* Ga = a.in + ((size_t)set * a.n_rings + ta) * nb;
  const double2* Gb = Ga + nb;
  const unsigned bytes = (vb ? 2u : 1u) * nb * 16u;
  if (tid == 0) {
    mbar_init(mb, 1);
    mbar_expect_tx(mb, bytes);
    bulk_g2s(buf, Ga, bytes, mb);
    const int nrow = row + a.pfd;
    if (a.pfd && nrow < (int)gridDim.x) {
      const int ns = nrow / per, np = nrow - ns * per;
      const int nta = a.real ? 2 * np : np;
      const bool nvb = a.real && nta + 1 < a.n_rings;
      bulk_prefetch_l2(a.in + ((size_t)ns * a.n_rings + nta) * nb, (nvb ? 2u : 1u) * nb * 16u);
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
  if (a.real) {
    // Hermitian spectra of the two rings (irfft ignores Im of the DC bin)
    double2 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int n = tid + u * T;
      x[u] = make_double2(0.0, 0.0);
      if (n < N) {
        const bool lo = n < nb;
        const int src = lo ? n : N - n;
        double2 X = buf[src], Y = vb ? buf[nb + src] : make_double2(0.0, 0.0);
        if (!lo) {
          X = cconj(X);
          Y = cconj(Y);
        }
        if (n == 0) X.y = Y.y = 0.0;
        x[u] = cadd(X, cmul_pi(Y));
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int n = tid + u * T;
      if (n < N) buf[n] = x[u];
    }
    __syncthreads();
  }
  pfa4095<true>(buf, tid, T);
  const int pole_ring = (N + 1) / 2 - 1 - a.t_offset;
  const bool pa = a.mw_pole && ta == pole_ring, pb = a.mw_pole && vb && ta + 1 == pole_ring;
  const double2 pva = pa ? __ldg(&Ga[0]) : make_double2(0.0, 0.0);
  const double2 pvb = pb ? __ldg(&Gb[0]) : make_double2(0.0, 0.0);
  const size_t ob = ((size_t)set * a.n_rings + ta) * N;
  constexpr int dpos = (int)(((unsigned)T * (unsigned)PFA_STEP) % (unsigned)PFA_N);
  int pos = pfa_pos(tid);  // slot of sample q: advances by pfa_pos(T) per iteration
#pragma unroll 4
  for (int q = tid; q < N; q += T) {
    const double2 v = buf[pos];
    pos = pfa_next(pos, dpos);
    if (a.real) {
      a.out[ob + q] = hard_thresh(pa ? pva.x : v.x, a.thresh);
      if (vb) a.out[ob + N + q] = hard_thresh(pb ? pvb.x : v.y, a.thresh);
    } else {
      reinterpret_cast<double2*>(a.out)[ob + q] = hard_thresh(pa ? pva : v, a.thresh);
    }
  }
}

template <int T>
__global__ void __launch_bounds__(T, S2W_K2_TSYN_MINB) theta_syn_k2_kernel(ThetaSynArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;           // [4096]
  double2* tw = smem + K2_M;     // [272]
  uint64_t* mb = reinterpret_cast<uint64_t*>(tw + K2_NTW);
  constexpr int N = K2_N, k = K2_K, U = K2_M / T;
  const FftTablesDev& F = a.T;
  const int tid = threadIdx.x;
  const ThetaSynRow R = theta_syn_row(a, blockIdx.x, true);
  if (tid == 0) {
    k2_issue(mb, tw, F.tw12, buf, R.ge, R.go);
    if (a.pfd && blockIdx.x + a.pfd < gridDim.x) {
      const ThetaSynRow Rn = theta_syn_row(a, blockIdx.x + a.pfd, true);
      if (Rn.ge) bulk_prefetch_l2(Rn.ge, K2_K * 16u);
      if (Rn.go) bulk_prefetch_l2(Rn.go, K2_K * 16u);
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
  // 1. parity extension on the 2k analysis points
  double2 x[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int n = tid + u * T;
    const bool lo = n < k;
    const int src = lo ? n : 2 * k - 1 - n;
    const double2 e = R.ge ? buf[src] : make_double2(0.0, 0.0);
    const double2 o = R.go ? buf[k + src] : make_double2(0.0, 0.0);
    x[u] = lo ? cadd(e, o) : csub(e, o);
  }
  __syncthreads();
  // 2. DFT_4096 (direct).  x[u] is element tid + 256 u, the input of this
  //    thread's first radix-16 butterfly: that pass runs in registers.
  fft_fwd_from_regs<12, T>(buf, tw, x, tid);
  // 3-4. inverse DFT_N by the prime-factor engine, its input (bit-reversed
  //      source slot, n >= k reads bin n + 1) formed in the gather of the
  //      first pass; rings t and N-1-t
  pfa4095_from<true, T>(buf, tid, [&](int n, int g) {
    const int src = n < k ? n : n + 1;
    return cmul(buf[swz(fft_brev<12>(src))], __ldg(&F.phS[g]));
  });
  constexpr int dpos = (int)(((unsigned)T * (unsigned)PFA_STEP) % (unsigned)PFA_N);
  int pos = pfa_pos(tid), posr = pfa_pos(N - 1 - tid);  // slots of rings t and N-1-t
#pragma unroll 4
  for (int t = tid; t < k; t += T) {
    theta_syn_store(R, a, t, buf[pos], buf[posr]);
    pos = pfa_next(pos, dpos);
    posr -= dpos;
    if (posr < 0) posr += PFA_N;
  }
}

template <int T>
__global__ void __launch_bounds__(T, T >= 512 ? 1 : 2) theta_k2_kernel(ThetaArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int pf = (a.pfd && blockIdx.x + a.pfd < gridDim.x) ? a.pfd : 0;
  theta_k2_row<T>(a, blockIdx.x, smem, pf);
}

// =====================================================================
// k4: the N = 8191 (L = 4096) stages.  8191 is prime: Rader's algorithm over
// the prime-factor DFT_8190 (pfa.cuh) replaces the 16384-point Bluestein
// convolutions of split mode, so a row fits shared memory (128 KiB + the theta
// side buffer): one CTA of 512 threads per SM, the row loaded by one bulk copy.
//  * phi_fwd_k4 / phi_inv_k4: ring DFTs (same I/O as phi_fwd/inv_kernel).
//  * theta_syn_k4: direct 8192-point FFT + Rader inverse DFT_8191.
//  * theta_k4: Rader DFT_8191, the |sin| convolution on the two parity
//    classes of the Fourier index (two 8192-point real-spectrum convolutions,
//    as theta_k2), evaluation by a direct 8192-point FFT.
// =====================================================================
constexpr int K4_N = 8191, K4_M = 8192, K4_K = 4096;
#ifndef S2W_K4_T
#define S2W_K4_T 512
#endif
constexpr int K4_T = S2W_K4_T;
constexpr int K4_NTW = 546;  // fft_ntw(13)
static_assert(K4_NTW == fft_ntw(13), "8192-point pass twiddles");

S2W_DEV RaderTabs rader_tabs(const FftTablesDev& F) { return RaderTabs{F.rgpow, F.rplog, F.rD}; }

template <int T>
__global__ void __launch_bounds__(T, 1) phi_fwd_k4_kernel(PhiFwdArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;                 // [8192]
  double2* part = smem + K4_M;         // [T/32]
  uint64_t* mb = reinterpret_cast<uint64_t*>(part + T / 32);
  constexpr int N = K4_N;
  const int tid = threadIdx.x;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x;
  const int set = row / per, p = row - set * per;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && ta + 1 < a.n_rings;
  const long long base_a = ((long long)set * a.n_rings + ta) * N;
  const unsigned bytes = a.real ? 2u * N * 8u : N * 16u;  // real rows come in pairs (launcher)
  if (tid == 0) {
    mbar_init(mb, 1);
    mbar_expect_tx(mb, bytes);
    bulk_g2s(buf, a.in + (a.real ? base_a : 2 * base_a), bytes, mb);
    // the row of the CTA that will take this slot later (as the k2 kernels)
    const int nrow = row + a.pfd;
    if (a.pfd && nrow < (int)gridDim.x) {
      const int ns = nrow / per, np = nrow - ns * per;
      const long long nb = ((long long)ns * a.n_rings + (a.real ? 2 * np : np)) * N;
      bulk_prefetch_l2(a.in + (a.real ? nb : 2 * nb), bytes);
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
  const RaderTabs R = rader_tabs(a.T);
  double2 x0, X0;
  if (a.real) {
    // [ring a | ring b] doubles -> z = a + i b, formed in Rader's input gather
    const double* r = reinterpret_cast<const double*>(buf);
    rader8191_from<T, false>(buf, R, part, x0, X0,
                             [&](int n, int) { return make_double2(r[n], vb ? r[N + n] : 0.0); });
  } else {
    rader8191<T, false>(buf, R, part, x0, X0);
  }
#pragma unroll 4
  for (int mi = tid; mi < a.n_bins; mi += T) {
    const double2 z = rader_bin<false>(buf, R, x0, X0, mi);
    if (!a.real) {
      fwd_row(a, set, mi)[ta] = cscale(z, a.scale);
    } else {
      const double2 zr = cconj(rader_bin<false>(buf, R, x0, X0, mi ? N - mi : 0));
      const double h = 0.5 * a.scale;
      const double2 r0 = cscale(cadd(z, zr), h), r1 = cscale(cmul_mi(csub(z, zr)), h);
      double2* o = fwd_row(a, set, mi) + ta;
      if (vb && aligned32(o)) st_global_32(o, r0, r1);  // the ring pair: one sector
      else {
        o[0] = r0;
        if (vb) o[1] = r1;
      }
    }
  }
}

template <int T>
__global__ void __launch_bounds__(T, 1) phi_inv_k4_kernel(PhiInvArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;
  double2* part = smem + K4_M;
  uint64_t* mb = reinterpret_cast<uint64_t*>(part + T / 32);
  constexpr int N = K4_N;
  const int tid = threadIdx.x;
  const int per = a.real ? (a.n_rings + 1) / 2 : a.n_rings;
  const int row = blockIdx.x;
  const int set = row / per, p = row - set * per;
  const int ta = a.real ? 2 * p : p;
  const bool vb = a.real && ta + 1 < a.n_rings;
  const int nb = a.n_bins;
  const double2* Ga = a.in + ((size_t)set * a.n_rings + ta) * nb;
  const double2* Gb = Ga + nb;
  const unsigned bytes = (vb ? 2u : 1u) * nb * 16u;
  if (tid == 0) {
    mbar_init(mb, 1);
    mbar_expect_tx(mb, bytes);
    bulk_g2s(buf, Ga, bytes, mb);
    const int nrow = row + a.pfd;
    if (a.pfd && nrow < (int)gridDim.x) {
      const int ns = nrow / per, np = nrow - ns * per;
      const int nta = a.real ? 2 * np : np;
      const bool nvb = a.real && nta + 1 < a.n_rings;
      bulk_prefetch_l2(a.in + ((size_t)ns * a.n_rings + nta) * nb, (nvb ? 2u : 1u) * nb * 16u);
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
  const RaderTabs R = rader_tabs(a.T);
  double2 x0, X0;
  if (a.real) {
    // Hermitian spectra of the two rings (irfft ignores Im of the DC bin),
    // formed in Rader's input gather
    rader8191_from<T, true>(buf, R, part, x0, X0, [&](int n, int) {
      const bool lo = n < nb;
      const int src = lo ? n : N - n;
      double2 X = buf[src], Y = vb ? buf[nb + src] : make_double2(0.0, 0.0);
      if (!lo) {
        X = cconj(X);
        Y = cconj(Y);
      }
      if (n == 0) X.y = Y.y = 0.0;
      return cadd(X, cmul_pi(Y));
    });
  } else {
    rader8191<T, true>(buf, R, part, x0, X0);
  }
  const int pole_ring = (N + 1) / 2 - 1 - a.t_offset;
  const bool pa = a.mw_pole && ta == pole_ring, pb = a.mw_pole && vb && ta + 1 == pole_ring;
  const double2 pva = pa ? __ldg(&Ga[0]) : make_double2(0.0, 0.0);
  const double2 pvb = pb ? __ldg(&Gb[0]) : make_double2(0.0, 0.0);
  const size_t ob = ((size_t)set * a.n_rings + ta) * N;
#pragma unroll 4
  for (int q = tid; q < N; q += T) {
    const double2 v = rader_bin<true>(buf, R, x0, X0, q);
    if (a.real) {
      a.out[ob + q] = hard_thresh(pa ? pva.x : v.x, a.thresh);
      if (vb) a.out[ob + N + q] = hard_thresh(pb ? pvb.x : v.y, a.thresh);
    } else {
      reinterpret_cast<double2*>(a.out)[ob + q] = hard_thresh(pa ? pva : v, a.thresh);
    }
  }
}

// arm the barrier and issue the 8192-point twiddles and a column pair
S2W_DEV void k4_issue(uint64_t* mb, double2* tw, const double2* gtw, double2* dst, const double2* ge,
                      const double2* go) {
  constexpr unsigned col = K4_K * 16u;
  mbar_init(mb, 1);
  mbar_expect_tx(mb, K4_NTW * 16u + (ge ? col : 0u) + (go ? col : 0u));
  bulk_g2s(tw, gtw, K4_NTW * 16u, mb);
  if (ge) bulk_g2s(dst, ge, col, mb);
  if (go) bulk_g2s(dst + K4_K, go, col, mb);
}

template <int T>
__global__ void __launch_bounds__(T, 1) theta_syn_k4_kernel(ThetaSynArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;               // [8192]
  double2* tw = smem + K4_M;         // [546]
  double2* part = tw + K4_NTW;       // [T/32]
  uint64_t* mb = reinterpret_cast<uint64_t*>(part + T / 32);
  constexpr int N = K4_N, k = K4_K, U = K4_M / T;
  const FftTablesDev& F = a.T;
  const int tid = threadIdx.x;
  const ThetaSynRow Rw = theta_syn_row(a, blockIdx.x, true);
  if (tid == 0) k4_issue(mb, tw, F.tw, buf, Rw.ge, Rw.go);
  __syncthreads();
  mbar_wait(mb, 0);
  double2 x[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int n = tid + u * T;
    const bool lo = n < k;
    const int src = lo ? n : 2 * k - 1 - n;
    const double2 e = Rw.ge ? buf[src] : make_double2(0.0, 0.0);
    const double2 o = Rw.go ? buf[k + src] : make_double2(0.0, 0.0);
    x[u] = lo ? cadd(e, o) : csub(e, o);
  }
  __syncthreads();
  // x[u] is element tid + 512 u: the first radix-16 pass runs in registers
  fft_fwd_from_regs<13, T>(buf, tw, x, tid);
  // inverse DFT_N (Rader), its input (bit-reversed source slot, n >= k reads
  // bin n + 1, times phS) formed in Rader's input gather
  const RaderTabs R = rader_tabs(F);
  double2 x0, X0;
  rader8191_from<T, true>(buf, R, part, x0, X0, [&](int n, int g) {
    const int src = n < k ? n : n + 1;
    return cmul(buf[swz(fft_brev<13>(src))], __ldg(&F.phS[g]));
  });
#pragma unroll 4
  for (int t = tid; t < k; t += T)
    theta_syn_store(Rw, a, t, rader_bin<true>(buf, R, x0, X0, t), rader_bin<true>(buf, R, x0, X0, N - 1 - t));
}

template <int T>
__global__ void __launch_bounds__(T, 1) theta_k4_kernel(ThetaArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  double2* buf = smem;               // [8192]
  double2* side = smem + K4_M;       // [4096]
  double2* tw = side + K4_K;         // [546]
  double2* part = tw + K4_NTW;       // [T/32]
  uint64_t* mb = reinterpret_cast<uint64_t*>(part + T / 32);
  constexpr int k = K4_K, U = K4_M / T;
  const FftTablesDev& F = a.T;
  const int tid = threadIdx.x;
  bool has_e, has_o;
  {
    const ThetaPair P = theta_pair(a, blockIdx.x, true);
    has_e = P.ge != nullptr;
    has_o = P.go != nullptr;
    if (tid == 0) k4_issue(mb, tw, F.tw, buf, P.ge, P.go);
  }
  __syncthreads();
  mbar_wait(mb, 0);
  // 1-2. DFT_N (Rader) of the parity extension, formed in Rader's input gather
  double2 x[U];
  const RaderTabs R = rader_tabs(F);
  double2 x0, X0;
  rader8191_from<T, false>(buf, R, part, x0, X0, [&](int n, int) {
    const bool lo = n < k;
    const int src = lo ? n : 2 * k - 2 - n;
    const double2 e = has_e ? buf[src] : make_double2(0.0, 0.0);
    const double2 o = has_o ? buf[k + src] : make_double2(0.0, 0.0);
    return lo ? cadd(e, o) : csub(e, o);
  });
  // 3-8. coefficient split, parity-class convolutions, evaluation FFT
  //      (N2 = 8192), as theta_k2; rings j and N2-1-j, split by parity
  static_assert(U == 16, "theta_classes scratch");
  theta_classes<13, T>(buf, side, tw, F, F.w4s, x,
                       [&](int bin) { return rader_bin<false>(buf, R, x0, X0, bin); });
  const ThetaPair P = theta_pair(a, blockIdx.x, true);
  for (int t = tid; t < k; t += T) {
    const double2 wt = cconj(buf[swz(fft_brev<13>(t))]);
    const double2 wr = cconj(buf[swz(fft_brev<13>(K4_M - 1 - t))]);
    theta_store(P, a, t, wt, wr);
  }
}

// ---------------------------------------------------------------- launchers
static cudaError_t set_smem(const void* fn, size_t smem) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

static int device_sms() {
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Rows per CTA for the shared-memory kernels: the value (<= fft_maxthr threads
// per CTA) that maximises resident threads per SM, given the kernel's registers
// and the shared memory per row.
static int pick_rpc(const void* fn, int logm, int n_rows, size_t& smem) {
  const int M = 1 << logm, gs = fft_gs(logm);
  const size_t tw = (size_t)((fft_ntw(logm) + 7) & ~7) * sizeof(double2);
  cudaFuncAttributes fa;
  int regs = 128;
  if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess && fa.numRegs > 0) regs = fa.numRegs;
  int best = 1, best_occ = -1;
  for (int rpc = 1; rpc * gs <= fft_maxthr(logm) && rpc <= n_rows; rpc *= 2) {
    const int threads = rpc * gs;
    const size_t sm = (size_t)rpc * M * sizeof(double2) + tw;
    if (sm > 227 * 1024) break;
    const int by_smem = (int)((228 * 1024) / (sm + 1024));
    const int by_regs = 65536 / (threads * ((regs + 7) & ~7));
    const int by_thr = 2048 / threads;
    const int ctas = std::min(std::min(by_smem, by_regs), std::min(by_thr, 32));
    const int occ = ctas * threads;
    if (occ > best_occ) {
      best_occ = occ;
      best = rpc;
    }
  }
  smem = (size_t)best * M * sizeof(double2) + tw;
  return best;
}

template <class Args>
static cudaError_t row_launch(void (*kern)(Args), int logm, Args a, int n_rows, cudaStream_t st) {
  size_t smem;
  a.rpc = pick_rpc((const void*)kern, logm, n_rows, smem);
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const int grid = (n_rows + a.rpc - 1) / a.rpc;
  kern<<<grid, a.rpc * fft_gs(logm), smem, st>>>(a);
  return cudaGetLastError();
}

static size_t split_smem(int logM) {
  const int F = 1 << (logM - 1);
  return ((size_t)F + ((fft_ntw(logM - 1) + 7) & ~7) + oct_alloc(logM)) * sizeof(double2);
}

template <class Args>
static cudaError_t split_launch(void (*kern)(Args), Args a, int n_rows, cudaStream_t st) {
  const size_t smem = split_smem(a.T.logM);
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  if (!a.scratch) return cudaErrorInvalidValue;
  kern<<<std::min(n_rows, device_sms()), SPLIT_T, smem, st>>>(a);
  return cudaGetLastError();
}

size_t fft_split_scratch_elems(int logM) {
  if (logM <= FFT_MAX_LOGM_SMEM) return 0;
  return (size_t)device_sms() * 2 * ((size_t)1 << (logM - 1));
}

int fft_tw_elems(int logE) { return fft_ntw(logE); }

// Dispatch on the convolution size: shared-memory kernels for logM <= 13,
// split mode for logM == 14.
#define S2W_FFT_DISPATCH(KERN, SPLIT, ARGS, NROWS, ST)                      \
  switch ((ARGS).T.logM) {                                                   \
    case 3: return row_launch(KERN<3>, 3, ARGS, NROWS, ST);                  \
    case 4: return row_launch(KERN<4>, 4, ARGS, NROWS, ST);                  \
    case 5: return row_launch(KERN<5>, 5, ARGS, NROWS, ST);                  \
    case 6: return row_launch(KERN<6>, 6, ARGS, NROWS, ST);                  \
    case 7: return row_launch(KERN<7>, 7, ARGS, NROWS, ST);                  \
    case 8: return row_launch(KERN<8>, 8, ARGS, NROWS, ST);                  \
    case 9: return row_launch(KERN<9>, 9, ARGS, NROWS, ST);                  \
    case 10: return row_launch(KERN<10>, 10, ARGS, NROWS, ST);               \
    case 11: return row_launch(KERN<11>, 11, ARGS, NROWS, ST);               \
    case 12: return row_launch(KERN<12>, 12, ARGS, NROWS, ST);               \
    case 13: return row_launch(KERN<13>, 13, ARGS, NROWS, ST);               \
    case 14: return split_launch(SPLIT<13>, ARGS, NROWS, ST);                \
    default: return cudaErrorInvalidValue;                                   \
  }

template <class Args>
static cudaError_t pfa_launch(void (*kern)(Args), Args a, int n_rows, cudaStream_t st) {
  const size_t smem = 4096 * sizeof(double2);
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  kern<<<n_rows, PFA_T, smem, st>>>(a);
  return cudaGetLastError();
}

// the prime-factor engine serves N = 4095 (L = 2048) unless S2W_NO_PFA is set
static bool use_pfa(int N) {
  static const bool off = getenv("S2W_NO_PFA") != nullptr;
  return N == PFA_N && !off;
}

// k2 kernels: 64 KiB row buffer + barrier (+ side buffer and twiddles for theta)
static size_t k2_smem(int side, bool tw) {
  return ((size_t)K2_M + side + (tw ? K2_NTW : 0)) * sizeof(double2) + 16;
}
template <class Args>
static cudaError_t k2_launch(void (*kern)(Args), Args a, int n_rows, size_t smem, cudaStream_t st,
                             int threads = K2_T) {
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  static const bool no_pf = getenv("S2W_K2_NOPF") != nullptr;
  int per_sm = 0;
  if (!no_pf && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) == cudaSuccess)
    a.pfd = per_sm * device_sms();
  kern<<<n_rows, threads, smem, st>>>(a);
  return cudaGetLastError();
}
// bulk copies need 16-byte aligned rows: complex buffers always are (if the
// base is); real ring pairs need an even ring count
static bool k2_ok(const void* base, bool real_pairs, int n_rings) {
  static const bool off = getenv("S2W_NO_K2") != nullptr;
  return !off && ((uintptr_t)base & 15) == 0 && (!real_pairs || (n_rings % 2) == 0);
}

static size_t k4_smem(int side, bool tw) {
  return ((size_t)K4_M + side + (tw ? K4_NTW : 0) + K4_T / 32) * sizeof(double2) + 16;
}
static bool use_k4(const FftTablesDev& T) {
  static const bool off = getenv("S2W_NO_K4") != nullptr;
  return !off && T.N == K4_N && T.rD != nullptr;
}

cudaError_t launch_phi_fwd(PhiFwdArgs a, cudaStream_t st) {
  const int n_rows = a.n_sets * (a.real ? (a.n_rings + 1) / 2 : a.n_rings);
  if (n_rows == 0) return cudaSuccess;
  if (use_k4(a.T) && k2_ok(a.in, a.real, a.n_rings))
    return k2_launch(phi_fwd_k4_kernel<K4_T>, a, n_rows, k4_smem(0, false), st, K4_T);
  if (use_pfa(a.T.N) && k2_ok(a.in, a.real, a.n_rings))
    return k2_launch(phi_fwd_k2_kernel<K2_PFT>, a, n_rows, k2_smem(0, false), st, K2_PFT);
  if (use_pfa(a.T.N)) return pfa_launch(phi_fwd_pfa_kernel, a, n_rows, st);
  S2W_FFT_DISPATCH(phi_fwd_kernel, phi_fwd_split_kernel, a, n_rows, st)
}

cudaError_t launch_phi_inv(PhiInvArgs a, cudaStream_t st) {
  const int n_rows = a.n_sets * (a.real ? (a.n_rings + 1) / 2 : a.n_rings);
  if (n_rows == 0) return cudaSuccess;
  if (use_k4(a.T) && k2_ok(a.in, false, a.n_rings) && a.n_bins <= (a.real ? K4_K : K4_N))
    return k2_launch(phi_inv_k4_kernel<K4_T>, a, n_rows, k4_smem(0, false), st, K4_T);
  if (use_pfa(a.T.N) && k2_ok(a.in, false, a.n_rings) && a.n_bins <= (a.real ? K2_K : K2_N))
    return k2_launch(phi_inv_k2_kernel<K2_PIT>, a, n_rows, k2_smem(0, false), st, K2_PIT);
  if (use_pfa(a.T.N)) return pfa_launch(phi_inv_pfa_kernel, a, n_rows, st);
  S2W_FFT_DISPATCH(phi_inv_kernel, phi_inv_split_kernel, a, n_rows, st)
}

void theta_pairs(const int* bins, int n_rows, int k, std::vector<int2>& pairs) {
  const int N = 2 * k - 1;
  std::vector<int> ev, od;
  for (int r = 0; r < n_rows; ++r) {
    const int bin = bins ? bins[r] : r;
    const int m = bin < k ? bin : bin - N;
    ((m & 1) ? od : ev).push_back(r);
  }
  const size_t n = std::max(ev.size(), od.size());
  pairs.resize(n);
  for (size_t i = 0; i < n; ++i)
    pairs[i] = make_int2(i < ev.size() ? ev[i] : -1, i < od.size() ? od[i] : -1);
}

cudaError_t launch_theta_syn(ThetaSynArgs a, cudaStream_t st) {
  const int n_rows = a.n_sets * a.n_pairs;
  if (n_rows == 0) return cudaSuccess;
  if (use_k4(a.T) && k2_ok(a.in, false, 0))
    return k2_launch(theta_syn_k4_kernel<K4_T>, a, n_rows, k4_smem(0, true), st, K4_T);
  if (use_pfa(a.T.N) && a.T.tw12 && k2_ok(a.in, false, 0))
    return k2_launch(theta_syn_k2_kernel<K2_T>, a, n_rows, k2_smem(0, true), st);
  if (use_pfa(a.T.N) && a.T.logM == 13)
    return row_launch(theta_syn_kernel<13, true>, 13, a, n_rows, st);
  S2W_FFT_DISPATCH(theta_syn_kernel, theta_syn_split_kernel, a, n_rows, st)
}

cudaError_t launch_theta(ThetaArgs a, cudaStream_t st) {
  const int n_rows = a.n_sets * a.n_pairs;
  if (n_rows == 0) return cudaSuccess;
  if (use_k4(a.T) && k2_ok(a.in, false, 0))
    return k2_launch(theta_k4_kernel<K4_T>, a, n_rows, k4_smem(K4_K, true), st, K4_T);
  if (use_pfa(a.T.N) && a.T.tw12 && k2_ok(a.in, false, 0))
    return k2_launch(theta_k2_kernel<K2_TT>, a, n_rows, k2_smem(K2_K, true), st, K2_TT);
  if (use_pfa(a.T.N) && a.T.logM == 13) return row_launch(theta_kernel<13, true>, 13, a, n_rows, st);
  S2W_FFT_DISPATCH(theta_kernel, theta_split_kernel, a, n_rows, st)
}

}  // namespace s2w
