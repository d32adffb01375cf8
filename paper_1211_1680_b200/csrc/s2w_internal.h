// Internal (non-ABI) declarations shared by the s2w CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <vector>

namespace s2w {

// Set s2w_last_error() and return `code` (capi.cu).
int io_fail(int code, const char* fmt, ...);

// ------------------------------------------------------------------ FFT tables
// Per grid band k (N = 2k-1, M = 2^logM >= 2N-1).  All spectra are stored in
// bit-reversed order, transposed for the engine's core pass (fft.cuh
// conv_core; capi.cu core_transpose), and carry the 1/M of the unnormalised
// inverse FFT.
constexpr int FFT_MAX_LOGM_SMEM = 13;  // one 128 KiB row per CTA; larger M uses split mode

struct FftTablesDev {
  int N, logM;  // logM of the convolution length M; split mode when logM > 13
  const double2* tw;      // radix-16 pass twiddles of the FFT engine size (M, or M/2 in split mode)
  const double2* octM;    // split mode: octant table of M (for W_M^j)
  const double2* chirp;   // [N]  c_n = exp(-i pi n^2/N)
  const double2* bl_fwd;  // [M]  FFT(conj c, circular)/M
  const double2* bl_inv;  // [M]  FFT(c, circular)/M
  const double2* ph1;     // [N]  c_b exp(-i pi m'(b)/N)/N      (MW theta stage)
  const double2* wconv;   // [M]  FFT(w_hat, circular)/M, w_hat(p)=4/(1-p^2) p even
  // MW theta stage output on the analysis rings theta''_j = (2j+1) pi / N2, N2 = 2k:
  int N2;
  const double2* chirp2;  // [N2] c2_n = exp(-i pi n^2/N2)
  const double2* bl_ev;   // [M]  FFT(c2, circular)/M
  const double2* ph2;     // [N2] exp(i pi q(n)/N2) conj(c2_n), q(n) = n or n - N2 (|q| < k)
  // MW synthesis resampling (analysis rings -> sampling rings, theta_syn_kernel):
  const double2* bl_fwd2; // [M]  FFT(conj c2, circular)/M   (forward DFT_N2)
  const double2* ph4;     // [N]  c2_src e^{-i pi q/N2} e^{i pi q/N} conj(c_n) / N2, q = n or n - N
  // N2 = M/2 (k a power of two; the DFT_N2 steps are direct half-size FFTs):
  const double2* ph2d;    // [N2] exp(-i pi q(n)/N2)  (conjugated evaluation input)
  const double2* ph4d;    // [N]  e^{-i pi q/N2} e^{i pi q/N} conj(c_n) / N2
  // N = 4095 (k = 2048) stage kernels (fft_kernels.cu, "k2"):
  const double2* tw12;    // radix-16 pass twiddles of the 4096-point engine
  const double* w2s;      // [4096] FFT(w_hat(2d), circular)/4096 (real: the kernel is real and even),
                          //        the |sin| series on one parity class, bit-reversed
  const double2* phA;     // [N]  e^{-i pi q/N} / N  (theta: DFT_N bin -> Fourier coefficient)
  const double2* phS;     // [N]  e^{-i pi q/N2} e^{i pi q/N} / N2  (theta_syn: DFT_N2 bin -> DFT_N input);
                          //      N = 4095: in the gather order of the axis-9 prime-factor pass, N = 8191: in
                          //      Rader's gather order (capi.cu)
  // N = 8191 (k = 4096) stage kernels ("k4"; phA / phS above, tw = the 8192-point engine):
  const int* rgpow;       // [8190] Rader gather g^q mod N
  const int* rplog;       // [N]    Rader output map bin g^-p -> p
  const double2* rD;      // [8190] Rader kernel spectrum in prime-factor slot order, / 8190
  const double* w4s;      // [8192] FFT(w_hat(2d), circular)/8192 (real), bit-reversed
};

struct PhiFwdArgs {
  FftTablesDev T;
  int n_sets, n_rings, real;
  const double* in;  // [set][ring][N] real doubles or interleaved complex
  double2* out;      // [set][mi][ring], mi < n_bins
  int n_bins;
  double scale;
  int gsize, rpc;  // filled by the launcher
  double2* scratch;  // split mode: per-CTA scratch (fft_split_scratch_elems)
  int pfd = 0;  // k2 kernels: rows ahead whose input a CTA prefetches into L2 (launcher)
  // optional output row offsets (double2 elements) per (set, bin): the shard
  // plans write each destination rank's bins as one contiguous block
  // (s2w_shard_set_peers); nullptr = [set][mi][ring]
  const long long* ofs = nullptr;
  // fused exchange (s2w_shard_rings_forward_peers): row (set, bin) goes to
  // rank peer_q[.]'s buffer peer[q] at offset ofs[.] -- the destination's own
  // H_local layout, written over peer (NVLink / IPC) pointers
  const int* peer_q = nullptr;
  double2* peer[16] = {};
};

// start of the output row of (set, bin mi) of a forward ring-DFT launch
__device__ __forceinline__ double2* fwd_row(const PhiFwdArgs& a, int set, int mi) {
  const size_t i = (size_t)set * a.n_bins + mi;
  if (a.peer_q) return a.peer[a.peer_q[i]] + a.ofs[i];
  return a.ofs ? a.out + a.ofs[i] : a.out + i * a.n_rings;
}

struct PhiInvArgs {
  FftTablesDev T;
  int n_sets, n_rings, real, mw_pole;
  int t_offset;  // global ring index of local row 0 (ring-sharded maps); pole = ring k-1
  const double2* in;  // [set][ring][n_bins]
  double* out;        // [set][ring][N]
  int n_bins;
  int gsize, rpc;
  double2* scratch;
  double thresh = 0.0;  // > 0: hard threshold: samples with |value| < thresh are zeroed (denoise)
  int pfd = 0;  // k2 kernels: rows ahead whose input a CTA prefetches into L2 (launcher)
};

// The theta operator commutes with the reflection theta -> 2 pi - theta, so an
// even-m row (even extension) and an odd-m row (odd extension) are summed and
// transformed together, then separated by parity (see theta_kernel).
struct ThetaArgs {
  FftTablesDev T;
  int n_sets, k, n_bins;  // n_bins = rows per set
  const int2* pairs;      // [n_pairs] (even-m row, odd-m row) per transform, -1 = none
  int n_pairs;
  const double2* pole_resp;  // [k] response to a unit pole sample (nullptr: no odd rows)
  const double2* in;  // [set][mi][k]
  double2* out;       // [set][mi][k] (may alias in)
  int gsize, rpc;
  double2* scratch;
  int pfd = 0;  // k2 kernels: rows ahead whose input a CTA prefetches into L2 (launcher)
};

// MW synthesis theta stage: G on the analysis rings theta''_j (m-major) ->
// G on the MW rings (ring-major), order pairs by parity as in ThetaArgs.
struct ThetaSynArgs {
  FftTablesDev T;
  int n_sets, k, n_bins;  // n_bins = columns per set
  const int2* pairs;
  int n_pairs;
  const double2* in;  // [set][mi][k]  (analysis rings)
  double2* out;       // [set][t][n_bins] (MW rings), must not alias in
  int rpc;
  double2* scratch;
  int pfd = 0;  // k2 kernels: rows ahead whose input a CTA prefetches into L2 (launcher)
};

cudaError_t launch_phi_fwd(PhiFwdArgs a, cudaStream_t st);
cudaError_t launch_theta_syn(ThetaSynArgs a, cudaStream_t st);
// Scratch (double2 elements) the split-mode kernels need for convolution size 2^logM.
size_t fft_split_scratch_elems(int logM);
// Length of the pass-twiddle table of the FFT engine of size 2^logE.
int fft_tw_elems(int logE);
cudaError_t launch_phi_inv(PhiInvArgs a, cudaStream_t st);
cudaError_t launch_theta(ThetaArgs a, cudaStream_t st);
// Pair storage rows by the parity of their order m (bins[row] = azimuthal bin).
void theta_pairs(const int* bins, int n_rows, int k, std::vector<int2>& pairs);

// ------------------------------------------------------------------ Legendre
struct LegGridDev {
  int k;       // band limit of the grid = number of orders / degrees
  int n_t;     // number of rings
  int n_north; // > 0: rings symmetric about the equator (t <-> n_t-1-t), n_north = ceil(n_t/2)
  int n_bins;  // azimuthal bins stored per ring: 2k-1 (complex) or k (real)
  const double* cos_t;
  const double* omc_t;   // 1 - cos theta to full relative accuracy (symmetric kernels' recursion)
  const double* sin_t;
  const double* ring_w;  // analysis quadrature weight per ring (incl. 2 pi / N factors)
  const int2* act;       // [k] active ring range [lo, hi) per order m
  const int* binmap;     // bin -> local column (synthesis) / row (analysis); nullptr = identity
  int n_cols;            // synthesis output row stride (n_bins unless sharded by order)
  int mmajor;            // synthesis output m-major [col][t] (else ring-major [t][col])
};

// Buffers are addressed as (slot, element offset) into the per-launch base
// table LegSynthArgs::bufs / LegAnaArgs::bufs, so descriptor arrays stay
// device-resident across calls while user pointers change.
constexpr int S2W_NBUF = 4;

struct SynthSet {
  int fb;            // source coefficients: flat l^2+l+m layout, band f_L
  long long foff;
  int f_L;
  const double* w;   // per-degree real weight (tiling factor) or nullptr
  int ob;            // output G, ring-major [t][n_bins]
  long long ooff;
};

struct SynthItem {
  int grid, m, set0, nset;
};

struct AnaSet {
  int hb;            // input H, m-major [mi][t], n_bins rows of n_t
  long long hoff;
  int ob;            // output flat l^2+l+m, accumulated (+=)
  long long ooff;
  const double* w;   // per-degree weight or nullptr
};

struct AnaSeg {
  int grid, set0, nset;
  int combine;  // all sets accumulate (weighted) into the output of set0
};

struct AnaItem {
  int m, seg0, nseg;
};

// The seed table c_m (LegSynthArgs/LegAnaArgs::seed_c) has S2W_SEED_KMAX
// entries and is followed, in the same allocation, by the Reinsch table of
// the low orders: for m < S2W_REIN_M, rein[m * S2W_REIN_STRIDE + l] =
// (lambda'_l, kappa'_l), the x = 1 solution ratios of the normalised
// recursion computed in long double on the host (legendre_kernels.cu,
// ring_step_rein).  The table depends on (l, m) only, not on the rings.
constexpr int S2W_SEED_KMAX = 16384;
constexpr int S2W_REIN_M = 32;
constexpr int S2W_REIN_STRIDE = 4096 + 64;
__host__ __device__ inline const double2* rein_table(const double* seed_c) {
  return reinterpret_cast<const double2*>(seed_c + S2W_SEED_KMAX);
}

struct LegSynthArgs {
  const LegGridDev* grids;
  const SynthSet* sets;
  const SynthItem* items;
  const double* seed_c;  // [S2W_SEED_KMAX] c_m, then the Reinsch table (rein_table)
  int n_items;
  int cplx;
  int ns;  // compile-time set width selected by the launcher
  int win; // degrees per shared-memory window (leg_synth_window)
  int sym; // every grid is equator-symmetric (LegGridDev::n_north > 0)
  int rein; // the items are orders m < S2W_REIN_M (Reinsch recursion; sym only)
  double2* bufs[S2W_NBUF];
};

struct LegAnaArgs {
  const LegGridDev* grids;
  const AnaSet* sets;
  const AnaSeg* segs;
  const AnaItem* items;
  const double* seed_c;
  int n_items;
  int cplx;
  int ns;
  int win;  // degrees per window (leg_ana_window)
  int sym;  // every grid is equator-symmetric (LegGridDev::n_north > 0)
  int rein; // the items are orders m < S2W_REIN_M (Reinsch recursion; sym only)
  double2* bufs[S2W_NBUF];
  // pipelined analysis (leg_ana_pipe_kernel): recursion state between degree
  // passes, [item][ring][3] doubles; nullptr = the reduce-scatter kernels
  double* pipe_scratch = nullptr;
  long long pipe_stride = 0;
};

cudaError_t launch_leg_synth(const LegSynthArgs& a, cudaStream_t st);
cudaError_t launch_leg_ana(const LegAnaArgs& a, cudaStream_t st);
int leg_synth_window(int kmax, int ns, int cplx);
int leg_ana_window(int kmax, int ns, int cplx);
// the pipelined analysis kernel serves this launch shape (symmetric rings, <= 4
// reals per degree, large grids)
bool leg_ana_pipe_ok(int kmax, int ns, int cplx, int sym);
// Per ring: largest order m whose Legendre column reaches the significance
// threshold below degree k (used to build the per-m active ring ranges).
cudaError_t launch_leg_probe(int k, int n_t, const double* cos_t, const double* sin_t,
                             const double* seed_c, int* mmax_out, cudaStream_t st);
// Table of orthonormal P_lm(cos theta) for one theta: out[l*L+m] (assoc_legendre_ring).
cudaError_t launch_leg_table(int L, double cos_t, double sin_t, const double* seed_c,
                             double* out, cudaStream_t st);

// ------------------------------------------------------------------ tiling
constexpr int S2W_MAXK = 64;
struct TileArgs {
  int n_sets, L, n_k;
  const double* fac;        // [n_k][L]  sqrt(4pi/(2l+1)) K_j(l)
  int band[S2W_MAXK];       // coefficient band of each per-kernel set
  double2* ptr[S2W_MAXK];   // analysis: outputs; synthesis: inputs
  const double2* f_in;      // analysis input  [set][L^2]
  double2* f_out;           // synthesis output [set][L^2]
};
// out_j[set][i] = f[set][i] * fac_j[l(i)] for i < band_j^2   (transform.py:117-150)
cudaError_t launch_tile_analysis(const TileArgs& a, cudaStream_t st);
// f[set][i] = sum_j fac_j[l] * in_j[set][i] (i < band_j^2), j ascending (transform.py:153-172)
cudaError_t launch_tile_synthesis(const TileArgs& a, cudaStream_t st);
cudaError_t launch_real_to_complex(const double* in, double2* out, long long n, cudaStream_t st);
cudaError_t launch_complex_real_part(const double2* in, double* out, long long n, cudaStream_t st);

// FP64 FMA throughput microbenchmark (roofline denominator for the Legendre
// stage; MEASURED_PEAKS.json has no FP64 entry).  Synchronises the stream.
cudaError_t measure_fp64_peak(double* tflops, cudaStream_t st);
// FP64 tensor-core (mma.sync m8n8k4 DMMA) throughput in TFLOP/s.
cudaError_t measure_dmma_peak(double* tflops, cudaStream_t st);

// ------------------------------------------------------------------ shard exchange layouts
constexpr int S2W_MAX_RANKS = 16;  // = the PhiFwdArgs::peer table size
struct ShardSrc {
  const double2* p[S2W_MAX_RANKS];  // received block per source rank
};
// blocks [B][n_local][t_q] per source -> H [B][n_local][L]; ring_src[t] = (q, t - t0_q),
// t_len[q] = ring count of q's block
cudaError_t launch_shard_gather_rings(const ShardSrc& src, const int2* ring_src, const int* t_len,
                                      int B, int n_local, int L, double2* H, cudaStream_t st);
// blocks [B][t_r][n_q] per source -> G [B][t_r][n_bins]; bin_src[bin] = (q, index in q's bins),
// n_src[q] = number of q's bins
cudaError_t launch_shard_scatter_bins(const ShardSrc& src, const int2* bin_src, const int* n_src,
                                      int B, int t_r, int n_bins, double2* G, cudaStream_t st);
// push: my G_local [B][k][n_local] -> every ring's owner q, straight into its
// G_ring [B][t_q][n_bins] at (t - t0_q, bins[i]) over peer pointers
struct ShardDst {
  double2* p[S2W_MAX_RANKS];
};
cudaError_t launch_shard_push_rings(const double2* G, const ShardDst& dst, const int2* ring_src,
                                    const int* t_len, const int* bins, int B, int k, int n_local,
                                    int n_bins, cudaStream_t st);

}  // namespace s2w
