// C ABI (include/s2w.h): plans, precomputed tables and the host-side
// orchestration of the hot path.  Host code only; kernels live in
// fft_kernels.cu, legendre_kernels.cu and tiling_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "s2w.h"
#include "s2w_internal.h"

using namespace s2w;

#define S2W_VERSION "s2w-b200 0.1.0"

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// Error reporting for the other translation units (s2wm_io.cu).
int s2w::io_fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? S2W_ENOMEM : S2W_ECUDA, "%s: %s (%s:%d)", \
                  #x, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

#define CHECK(x)            \
  do {                      \
    int r_ = (x);           \
    if (r_ != S2W_OK) return r_; \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Plain device allocation owned by a plan (freed in the plan destructor).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  int ensure(size_t n) {
    if (n <= bytes && p) return S2W_OK;
    release();
    if (n == 0) n = 16;
    CU(cudaMalloc(&p, n));
    bytes = n;
    return S2W_OK;
  }
  template <class T>
  int upload(const std::vector<T>& v) {
    CHECK(ensure(v.size() * sizeof(T)));
    if (!v.empty()) CU(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return S2W_OK;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// ------------------------------------------------------------------ launch accounting
// Every kernel launch made by the library bumps g_launches (reported by
// bench.py as "gpu_launches").  With profiling enabled, each launch is also
// bracketed by CUDA events on its stream and accumulated per stage.
#include <atomic>
static std::atomic<long long> g_launches{0};

enum ProfStage { P_LEG_SYNTH = 0, P_LEG_ANA, P_PHI_FWD, P_THETA, P_PHI_INV, P_TILE, P_XCHG, P_NSTAGE };
static const char* kStageNames[P_NSTAGE] = {"leg_synth", "leg_ana", "phi_fwd",
                                            "theta", "phi_inv", "tile", "xchg_layout"};
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
};
static bool g_prof = false;
static std::vector<ProfRec> g_prof_pending;
static std::vector<cudaEvent_t> g_prof_pool;
static double g_prof_ms[P_NSTAGE] = {0};
static long long g_prof_n[P_NSTAGE] = {0};

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int s, cudaStream_t stream) : stage(s), st(stream) {
    ++g_launches;
    if (g_prof) {
      a = prof_event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, st);
      g_prof_pending.push_back({stage, a, b});
    }
  }
};

// ------------------------------------------------------------------ grids (host)
typedef long double ld;
static const ld PI_L = 3.141592653589793238462643383279502884L;

// Legendre P_n(x) and P_n'(x) in extended precision.
static void legendre_pd(int n, ld x, ld& p, ld& dp) {
  ld p0 = 1.0L, p1 = x;
  if (n == 0) {
    p = 1.0L;
    dp = 0.0L;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    ld p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1.0L);
}

// Gauss-Legendre nodes ordered north -> south (x descending) with weights,
// Newton iteration in 80-bit precision (grid.py:93-124 semantics).
// omc (optional): 1 - x of the 80-bit Newton root, the node the weights belong to.
static void gl_nodes(int L, std::vector<double>& theta, std::vector<double>& w,
                     std::vector<long double>* omc = nullptr) {
  theta.resize(L);
  w.resize(L);
  if (omc) omc->resize(L);
  if (L == 1) {
    theta[0] = std::acos(0.0);
    w[0] = 2.0;
    if (omc) (*omc)[0] = 1.0L;
    return;
  }
  for (int i = 0; i < L; ++i) {
    ld x = std::cos(PI_L * (i + 0.75L) / (L + 0.5L));
    ld p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre_pd(L, x, p, dp);
      ld dx = p / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
    legendre_pd(L, x, p, dp);
    x -= p / dp;
    legendre_pd(L, x, p, dp);
    ld wi = 2.0L / ((1.0L - x * x) * dp * dp);
    theta[i] = std::acos((double)x);
    w[i] = (double)wi;
    if (omc) (*omc)[i] = 1.0L - x;
  }
}

static void mw_nodes(int L, std::vector<double>& theta) {
  theta.resize(L);
  for (int t = 0; t < L; ++t) theta[t] = (double)(2 * t + 1) * M_PI / (double)(2 * L - 1);
}

// ------------------------------------------------------------------ host FFT (tables)
typedef std::complex<ld> cld;

static int ilog2_ceil(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

static unsigned bitrev(unsigned p, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i) r |= ((p >> i) & 1u) << (bits - 1 - i);
  return r;
}

// In-place forward DFT (exp(-2 pi i jk/M)), M a power of two, extended precision.
static void fft_ld(std::vector<cld>& a) {
  const size_t n = a.size();
  const int bits = ilog2_ceil((long long)n);
  for (size_t i = 0; i < n; ++i) {
    size_t j = bitrev((unsigned)i, bits);
    if (j > i) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t h = len / 2;
    std::vector<cld> w(h);
    for (size_t j = 0; j < h; ++j) {
      ld ang = -2.0L * PI_L * (ld)j / (ld)len;
      w[j] = cld(std::cos(ang), std::sin(ang));
    }
    for (size_t i = 0; i < n; i += len)
      for (size_t j = 0; j < h; ++j) {
        cld u = a[i + j], v = a[i + j + h] * w[j];
        a[i + j] = u + v;
        a[i + j + h] = u - v;
      }
  }
}

static double2 d2(cld z) { return make_double2((double)z.real(), (double)z.imag()); }

// spectrum (natural order) / M, stored at bit-reversed positions and then
// transposed for the core pass.  Split mode (M > 2^FFT_MAX_LOGM_SMEM):
// [even half | odd half], each bit-reversed over M/2.
// The table is read only by the engine's core pass (fft.cuh conv_core*),
// whose thread b multiplies the R = 2^CB consecutive elements b R + i: entry
// (b, i) is stored at i (E / R) + b (E the engine size), so the 32 lanes of a
// warp read 32 consecutive entries instead of 32 separate lines.
static void core_transpose(double2* t, int log_e) {
  const int cb = log_e - 4 * ((log_e - 1) / 4);
  const size_t R = (size_t)1 << cb, NB = ((size_t)1 << log_e) / R;
  std::vector<double2> tmp(t, t + R * NB);
  for (size_t b = 0; b < NB; ++b)
    for (size_t i = 0; i < R; ++i) t[i * NB + b] = tmp[b * R + i];
}
static std::vector<double2> spectrum_brev(std::vector<cld> a) {
  const size_t M = a.size();
  const int bits = ilog2_ceil((long long)M);
  fft_ld(a);
  std::vector<double2> out(M);
  if (bits <= FFT_MAX_LOGM_SMEM) {
    for (size_t p = 0; p < M; ++p) out[p] = d2(a[bitrev((unsigned)p, bits)] / (ld)M);
    core_transpose(out.data(), bits);
  } else {
    const size_t F = M / 2;
    for (size_t p = 0; p < F; ++p) {
      const size_t k = bitrev((unsigned)p, bits - 1);
      out[p] = d2(a[2 * k] / (ld)M);
      out[F + p] = d2(a[2 * k + 1] / (ld)M);
    }
    core_transpose(out.data(), bits - 1);
    core_transpose(out.data() + F, bits - 1);
  }
  return out;
}

// Radix-16 pass twiddles of the FFT engine of size 2^logE (fft.cuh): pass p
// (span s = 2^(logE - 4(p+1))) holds W_{16 s}^j, j < s, contiguous.
static std::vector<double2> pass_twiddles(int logE) {
  std::vector<double2> tw;
  for (int p = 0; p < (logE - 1) / 4; ++p) {
    const long long s = 1LL << (logE - 4 * (p + 1));
    for (long long j = 0; j < s; ++j) {
      const ld ang = -2.0L * PI_L * (ld)j / (ld)(16 * s);
      tw.push_back(make_double2((double)std::cos(ang), (double)std::sin(ang)));
    }
  }
  if ((int)tw.size() != fft_tw_elems(logE)) tw.clear();  // cannot happen
  return tw;
}

static std::vector<double2> octant_table(int logM) {
  const int M = 1 << logM;
  std::vector<double2> oct(M / 8 + 1);
  for (int j = 0; j <= M / 8; ++j) {
    ld ang = 2.0L * PI_L * (ld)j / (ld)M;
    oct[j] = make_double2((double)std::cos(ang), (double)std::sin(ang));
  }
  return oct;
}

// ------------------------------------------------------------------ per-device seed table
static const int SEED_KMAX = S2W_SEED_KMAX;
// Largest band limit: ring DFTs of N = 2L-1 need a Bluestein convolution of
// 2^ceil(log2(4L-3)) <= 2^14 points (split mode).
static const int S2W_MAX_L = 4096;
static_assert(S2W_MAX_L + 32 <= S2W_REIN_STRIDE, "Reinsch rows cover every chunk of the largest band");

struct DeviceTables {
  double* seed_c = nullptr;  // c_m, m < SEED_KMAX, then the Reinsch table (rein_table)
};

static std::mutex g_mu;
static std::map<int, DeviceTables> g_dev;

// Reinsch form of the low orders' recursion (legendre_kernels.cu,
// ring_step_rein).  With a_l, b_l of sht.py:146-152 (exact, long double) and
// rho_l the ratio P_l / P_{l-1} of the recursion's solution at x = 1
// (rho_{m+1} = a_{m+1}, rho_l = a_l - b_l / rho_{l-1}):
//   lambda'_l = rho_l / a_l,  kappa'_l = b_l / (a_l rho_{l-1}),
// and the seed degree l = m gets (0, 1).  These are the ratios of the
// normalised state Q_l = P_l / gamma_l whatever the chunking, since gamma
// only rescales both state values by a common factor.
static void rein_rows(std::vector<double2>& tab) {
  tab.assign((size_t)S2W_REIN_M * S2W_REIN_STRIDE, make_double2(1.0, 0.0));
  for (int m = 0; m < S2W_REIN_M; ++m) {
    double2* row = tab.data() + (size_t)m * S2W_REIN_STRIDE;
    row[m] = make_double2(0.0, 1.0);
    ld rho_prev = 0.0L;
    for (int l = m + 1; l < S2W_REIN_STRIDE; ++l) {
      const ld L_ = l, M_ = m, den = L_ * L_ - M_ * M_;
      const ld a = std::sqrt((4.0L * L_ * L_ - 1.0L) / den);
      const ld b = std::sqrt((2.0L * L_ + 1.0L) / (2.0L * L_ - 3.0L) *
                             ((L_ - 1.0L) * (L_ - 1.0L) - M_ * M_) / den);
      const ld rho = (l == m + 1) ? a : a - b / rho_prev;
      const ld kap = (l == m + 1) ? 0.0L : b / (a * rho_prev);
      row[l] = make_double2((double)(rho / a), (double)kap);
      rho_prev = rho;
    }
  }
}

static int device_tables(int dev, DeviceTables** out) {
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) {
    *out = &it->second;
    return S2W_OK;
  }
  std::vector<double> c(SEED_KMAX);
  ld v = 1.0L / std::sqrt(4.0L * PI_L);
  c[0] = (double)v;
  for (int m = 1; m < SEED_KMAX; ++m) {
    v *= std::sqrt((ld)(2 * m + 1) / (ld)(2 * m));
    c[m] = (double)v;
  }
  std::vector<double2> rein;
  rein_rows(rein);
  DeviceTables t;
  const size_t cb = sizeof(double) * SEED_KMAX, rb = sizeof(double2) * rein.size();
  CU(cudaMalloc(&t.seed_c, cb + rb));
  CU(cudaMemcpy(t.seed_c, c.data(), cb, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(t.seed_c + SEED_KMAX, rein.data(), rb, cudaMemcpyHostToDevice));
  g_dev[dev] = t;
  *out = &g_dev[dev];
  return S2W_OK;
}

// ------------------------------------------------------------------ grid resources
// A set of rings for the Legendre stages: nodes, analysis weights, active
// ring range per order.  n_north > 0 marks an equator-symmetric set.
struct RingSet {
  double *cos_t = nullptr, *omc_t = nullptr, *sin_t = nullptr, *ring_w = nullptr;
  int2* act = nullptr;
  std::vector<int2> act_host;
  int n_north = 0;
};

struct GridRes {
  int device, scheme, k, N, logM;
  // syn: the sampling rings (synthesis output, GL analysis);
  // ana: the analysis rings (GL: the GL rings; MW: theta''_j = (2j+1) pi / 2k, see theta_kernel)
  RingSet syn, ana;
  double2 *tw = nullptr, *octM = nullptr, *chirp = nullptr, *bl_fwd = nullptr, *bl_inv = nullptr,
          *ph1 = nullptr, *ph2 = nullptr, *wconv = nullptr, *chirp2 = nullptr, *bl_ev = nullptr,
          *bl_fwd2 = nullptr, *ph4 = nullptr, *ph2d = nullptr, *ph4d = nullptr, *tw12 = nullptr,
          *phA = nullptr, *phS = nullptr, *rD = nullptr;
  double* w2s = nullptr;
  double* w4s = nullptr;
  int *rgpow = nullptr, *rplog = nullptr;
  double* seed_c = nullptr;
  // MW theta stage: parity pairs of the full real / complex bin layouts, pole response
  int2 *pairs_r = nullptr, *pairs_c = nullptr;
  int np_r = 0, np_c = 0;
  double2* pole_resp = nullptr;

  ThetaArgs theta(bool cplx) const {
    ThetaArgs t;
    t.T = fft();
    t.k = k;
    t.n_bins = n_bins(cplx);
    t.pairs = cplx ? pairs_c : pairs_r;
    t.n_pairs = cplx ? np_c : np_r;
    t.pole_resp = pole_resp;
    return t;
  }

  FftTablesDev fft() const {
    FftTablesDev t;
    t.N = N;
    t.logM = logM;
    t.tw = tw;
    t.octM = octM;
    t.chirp = chirp;
    t.bl_fwd = bl_fwd;
    t.bl_inv = bl_inv;
    t.ph1 = ph1;
    t.ph2 = ph2;
    t.wconv = wconv;
    t.N2 = 2 * k;
    t.chirp2 = chirp2;
    t.bl_ev = bl_ev;
    t.bl_fwd2 = bl_fwd2;
    t.ph4 = ph4;
    t.ph2d = ph2d;
    t.ph4d = ph4d;
    t.tw12 = tw12;
    t.w2s = w2s;
    t.phA = phA;
    t.phS = phS;
    t.rgpow = rgpow;
    t.rplog = rplog;
    t.rD = rD;
    t.w4s = w4s;
    return t;
  }
  // MW synthesis runs on the (symmetric) analysis rings and is resampled to
  // the MW rings by theta_syn_kernel; GL synthesis runs on its own rings.
  // Small MW grids synthesise on their own rings directly: there the
  // resampling (O(k^2 log k)) costs more than the halved recursion saves.
  bool syn_on_ana() const { return scheme == S2W_SCHEME_MW && k >= syn_resample_min(); }
  static int syn_resample_min() {
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("S2W_SYN_RESAMPLE_MIN");
      v = e ? atoi(e) : 1024;
    }
    return v;
  }
  LegGridDev leg(bool cplx, bool analysis) const {
    const RingSet& rs = (analysis || syn_on_ana()) ? ana : syn;
    LegGridDev g;
    g.k = k;
    g.n_t = k;
    g.n_north = rs.n_north;
    g.n_bins = cplx ? N : k;
    g.cos_t = rs.cos_t;
    g.omc_t = rs.omc_t;
    g.sin_t = rs.sin_t;
    g.ring_w = rs.ring_w;
    g.act = rs.act;
    g.binmap = nullptr;
    g.n_cols = cplx ? N : k;
    g.mmajor = (!analysis && syn_on_ana()) ? 1 : 0;
    return g;
  }
  int n_bins(bool cplx) const { return cplx ? N : k; }
  // Free every device table (a half-built grid on a setup failure).  GL
  // grids alias ana to syn.
  void release() {
    auto fr = [](auto*& p) {
      if (p) cudaFree((void*)p);
      p = nullptr;
    };
    const bool alias = ana.cos_t == syn.cos_t;
    for (RingSet* rs : {&syn, &ana}) {
      if (rs == &ana && alias) break;
      fr(rs->cos_t), fr(rs->omc_t), fr(rs->sin_t), fr(rs->ring_w), fr(rs->act);
    }
    fr(tw), fr(octM), fr(chirp), fr(bl_fwd), fr(bl_inv), fr(ph1), fr(ph2), fr(wconv), fr(chirp2);
    fr(bl_ev), fr(bl_fwd2), fr(ph4), fr(ph2d), fr(ph4d), fr(tw12), fr(phA), fr(phS), fr(rD);
    fr(w2s), fr(w4s), fr(rgpow), fr(rplog), fr(pairs_r), fr(pairs_c), fr(pole_resp);
  }
  // rough cost of the Legendre work for order m (ring-steps)
  double cost(int m, bool analysis) const {
    const RingSet& rs = (analysis || syn_on_ana()) ? ana : syn;
    const int2 a = rs.act_host[m];
    const int n = rs.n_north ? std::max(0, std::min(a.y, rs.n_north) - a.x) : std::max(0, a.y - a.x);
    return (double)(k - m) * (double)n + 64.0;
  }
};

static std::map<std::tuple<int, int, int>, GridRes*> g_grids;
// Private non-blocking stream for grid setup (uploads, probe and pole-response
// launches), created and destroyed by get_grid under g_mu: setup never orders
// against, or stalls, the caller's streams through the legacy stream 0.
static cudaStream_t g_setup = nullptr;

template <class T>
static int upload_new(T** dst, const std::vector<T>& v) {
  CU(cudaMalloc(dst, std::max<size_t>(16, v.size() * sizeof(T))));
  if (!v.empty())
    CU(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, g_setup));
  return S2W_OK;
}

// Upload a ring set and find its active ring range per order (probe kernel).
// Symmetric sets (n_north > 0) get exactly mirrored nodes: cos(pi - x) = -cos x.
// omc_exact (optional): 1 - cos of the exact nodes in long double (else from theta).
static int ring_set(RingSet& rs, const std::vector<double>& theta, const std::vector<double>& w,
                    int k, const double* seed_c, int n_north,
                    const std::vector<long double>* omc_exact = nullptr) {
  const int n = (int)theta.size();
  std::vector<double> c(n), s(n);
  for (int t = 0; t < n; ++t) {
    c[t] = std::cos(theta[t]);
    s[t] = std::sin(theta[t]);
  }
  if (n_north)
    for (int t = n - n_north; t < n; ++t) {
      const int tm = n - 1 - t;
      if (tm == t) {
        c[t] = 0.0;
        continue;
      }
      c[t] = -c[tm];
      s[t] = s[tm];
    }
  // 1 - cos theta with full relative accuracy (2 sin^2(theta/2) in the north,
  // 1 + |cos theta| in the south): the symmetric kernels step the recursion
  // with x Q = Q - (1 - x) Q, so polar nodes keep their exact position (a
  // rounded cos theta moves 1 - x by up to 1e-9 relative at L = 4096).
  std::vector<double> omc(n);
  for (int t = 0; t < n; ++t) {
    if (omc_exact) {
      omc[t] = (double)(*omc_exact)[t];
    } else if (c[t] >= 0.0) {
      const ld h = std::sin((ld)theta[t] / 2);
      omc[t] = (double)(2 * h * h);
    } else {
      omc[t] = (double)(1.0L - (ld)c[t]);
    }
  }
  rs.n_north = n_north;
  CHECK(upload_new(&rs.cos_t, c));
  CHECK(upload_new(&rs.omc_t, omc));
  CHECK(upload_new(&rs.sin_t, s));
  CHECK(upload_new(&rs.ring_w, w));
  int* d_mmax = nullptr;
  CU(cudaMalloc(&d_mmax, sizeof(int) * n));
  CU(launch_leg_probe(k, n, rs.cos_t, rs.sin_t, seed_c, d_mmax, g_setup));
  std::vector<int> mmax(n);
  CU(cudaMemcpyAsync(mmax.data(), d_mmax, sizeof(int) * n, cudaMemcpyDeviceToHost, g_setup));
  CU(cudaStreamSynchronize(g_setup));
  cudaFree(d_mmax);
  rs.act_host.assign(k, make_int2(0, 0));
  for (int m = 0; m < k; ++m) {
    int lo = -1, hi = -1;
    for (int t = 0; t < n; ++t)
      if (mmax[t] >= m) {
        if (lo < 0) lo = t;
        hi = t;
      }
    rs.act_host[m] = (lo < 0) ? make_int2(0, 0) : make_int2(lo, hi + 1);
  }
  CHECK(upload_new(&rs.act, rs.act_host));
  return S2W_OK;
}

// Parity pairs for the theta stage and its response to a unit pole sample
// (one even-row transform of e_{k-1}, run once per grid).
static int theta_setup(GridRes* g) {
  const int k = g->k;
  std::vector<int2> pr;
  theta_pairs(nullptr, k, k, pr);
  g->np_r = (int)pr.size();
  CHECK(upload_new(&g->pairs_r, pr));
  theta_pairs(nullptr, g->N, k, pr);
  g->np_c = (int)pr.size();
  CHECK(upload_new(&g->pairs_c, pr));
  std::vector<double2> imp(k, make_double2(0.0, 0.0));
  imp[k - 1] = make_double2(1.0, 0.0);
  double2 *d_imp = nullptr, *scratch = nullptr;
  int2* one = nullptr;
  CHECK(upload_new(&d_imp, imp));
  CHECK(upload_new(&one, std::vector<int2>{make_int2(0, -1)}));
  CU(cudaMalloc(&g->pole_resp, sizeof(double2) * k));
  const size_t se = fft_split_scratch_elems(g->logM);
  if (se) CU(cudaMalloc(&scratch, sizeof(double2) * se));
  ThetaArgs ta = g->theta(false);
  ta.n_sets = 1;
  ta.n_bins = 1;
  ta.pairs = one;
  ta.n_pairs = 1;
  ta.pole_resp = nullptr;
  ta.in = d_imp;
  ta.out = g->pole_resp;
  ta.scratch = scratch;
  CU(launch_theta(ta, g_setup));
  CU(cudaStreamSynchronize(g_setup));
  cudaFree(d_imp);
  cudaFree(one);
  if (scratch) cudaFree(scratch);
  return S2W_OK;
}

static int build_grid(GridRes* g, int dev, int scheme, int k);

static int get_grid(int dev, int scheme, int k, GridRes** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, scheme, k);
  auto it = g_grids.find(key);
  if (it != g_grids.end()) {
    *out = it->second;
    return S2W_OK;
  }
  if (k < 1 || k > S2W_MAX_L) return fail(S2W_EPARAM, "band-limit %d out of range [1, %d]", k, S2W_MAX_L);
  CU(cudaStreamCreateWithFlags(&g_setup, cudaStreamNonBlocking));
  std::unique_ptr<GridRes> g(new GridRes());
  int r = build_grid(g.get(), dev, scheme, k);
  if (r == S2W_OK) r = cudaStreamSynchronize(g_setup) == cudaSuccess ? S2W_OK : fail(S2W_ECUDA, "grid setup");
  cudaStreamDestroy(g_setup);
  g_setup = nullptr;
  if (r != S2W_OK) {
    g->release();  // no half-built grid leaks its tables
    return r;
  }
  *out = g_grids[key] = g.release();
  return S2W_OK;
}

static int build_grid(GridRes* g, int dev, int scheme, int k) {
  DeviceTables* dt;
  CHECK(device_tables(dev, &dt));
  g->device = dev;
  g->scheme = scheme;
  g->k = k;
  g->N = 2 * k - 1;
  g->logM = std::max(3, ilog2_ceil(2LL * g->N - 1));
  g->seed_c = dt->seed_c;
  const int N = g->N, M = 1 << g->logM;

  // exact nodes' 1 - cos theta in long double (recursion in the symmetric kernels)
  std::vector<double> theta, wq;
  std::vector<long double> omc_syn(k), omc_ana(k);
  if (scheme == S2W_SCHEME_GL) {
    gl_nodes(k, theta, wq, &omc_syn);
  } else {
    mw_nodes(k, theta);
    for (int t = 0; t < k; ++t) {
      const ld th = (ld)(2 * t + 1) * PI_L / (ld)(2 * k - 1);
      omc_syn[t] = th <= PI_L / 2 ? 2 * std::sin(th / 2) * std::sin(th / 2) : 1.0L - std::cos(th);
    }
    for (int j = 0; j < k; ++j) {
      const ld th = (ld)(2 * j + 1) * PI_L / (ld)(2 * k);
      omc_ana[j] = th <= PI_L / 2 ? 2 * std::sin(th / 2) * std::sin(th / 2) : 1.0L - std::cos(th);
    }
  }
  std::vector<double> rw(k);
  for (int t = 0; t < k; ++t) {
    if (scheme == S2W_SCHEME_GL) rw[t] = 2.0 * M_PI * wq[t];
    else rw[t] = (2.0 * M_PI / (double)N) * (t == k - 1 ? 0.5 : 1.0);
  }
  CHECK(ring_set(g->syn, theta, rw, k, g->seed_c, 0, &omc_syn));
  if (scheme == S2W_SCHEME_GL) {
    g->syn.n_north = (k + 1) / 2;  // GL nodes are symmetric about the equator
    g->ana = g->syn;                // same device tables
  } else {
    // analysis rings of the MW theta stage: theta''_j = (2j+1) pi / 2k, weight pi / k
    std::vector<double> th2(k), w2(k, M_PI / (double)k);
    for (int j = 0; j < k; ++j) th2[j] = (double)((ld)(2 * j + 1) * PI_L / (ld)(2 * k));
    CHECK(ring_set(g->ana, th2, w2, k, g->seed_c, (k + 1) / 2, &omc_ana));
  }

  // FFT / Bluestein / theta-stage tables
  const int N2 = 2 * k;
  std::vector<double2> chirp(N), ph1(N), ph2(N2), chirp2(N2);
  const bool split = g->logM > FFT_MAX_LOGM_SMEM;
  std::vector<cld> cl(N);
  for (int n = 0; n < N; ++n) {
    long long r = ((long long)n * n) % (2LL * N);
    ld ang = -PI_L * (ld)r / (ld)N;
    cl[n] = cld(std::cos(ang), std::sin(ang));
    chirp[n] = d2(cl[n]);
  }
  std::vector<cld> b(M, cld(0, 0)), cc(M, cld(0, 0)), w(M, cld(0, 0));
  for (int j = 0; j < N; ++j) {
    b[j] = std::conj(cl[j]);
    cc[j] = cl[j];
    if (j > 0) {
      b[M - j] = std::conj(cl[j]);
      cc[M - j] = cl[j];
    }
  }
  for (int p = -(2 * k - 2); p <= 2 * k - 2; ++p) {
    if (p & 1) continue;
    w[(p % M + M) % M] = cld(4.0L / (1.0L - (ld)p * (ld)p), 0);
  }
  for (int bin = 0; bin < N; ++bin) {
    const int q = bin < k ? bin : bin - N;
    ld a1 = -PI_L * (ld)q / (ld)N;
    ph1[bin] = d2(cl[bin] * cld(std::cos(a1), std::sin(a1)) / (ld)N);
  }
  // evaluation on the analysis rings: inverse DFT of length N2 = 2k (Bluestein)
  std::vector<cld> c2(N2), cc2(M, cld(0, 0));
  for (int n = 0; n < N2; ++n) {
    const long long r = ((long long)n * n) % (2LL * N2);
    const ld ang = -PI_L * (ld)r / (ld)N2;
    c2[n] = cld(std::cos(ang), std::sin(ang));
    chirp2[n] = d2(c2[n]);
    cc2[n] = c2[n];
    if (n > 0) cc2[M - n] = c2[n];
  }
  std::vector<cld> b2(M, cld(0, 0));
  for (int n = 0; n < N2; ++n) {
    b2[n] = std::conj(c2[n]);
    if (n > 0) b2[M - n] = std::conj(c2[n]);
  }
  // synthesis resampling: X_n = DFT_N2[src] ph4[n], n < N (see theta_syn_kernel)
  std::vector<double2> ph4(N), ph4d(N), ph2d(N2);
  for (int n = 0; n < N; ++n) {
    const int q = n < k ? n : n - N;
    const int src = q >= 0 ? q : N2 + q;
    const ld a2 = -PI_L * (ld)q / (ld)N2, a1 = PI_L * (ld)q / (ld)N;
    const cld base = cld(std::cos(a2), std::sin(a2)) * cld(std::cos(a1), std::sin(a1)) *
                     std::conj(cl[n]) / (ld)N2;
    ph4[n] = d2(c2[src] * base);
    ph4d[n] = d2(base);
  }
  for (int n = 0; n < N2; ++n) {
    const int q = n < k ? n : n - N2;
    const ld a2 = -PI_L * (ld)q / (ld)N2;
    ph2d[n] = (n >= k && n <= N2 - k) ? make_double2(0.0, 0.0)
                                      : d2(cld(std::cos(a2), std::sin(a2)));
  }
  for (int n = 0; n < N2; ++n) {
    const int q = n < k ? n : n - N2;
    if (n >= k && n <= N2 - k) {
      ph2[n] = make_double2(0.0, 0.0);
      continue;
    }
    const ld a2 = PI_L * (ld)q / (ld)N2;
    ph2[n] = d2(cld(std::cos(a2), std::sin(a2)) * std::conj(c2[n]));
  }
  CHECK(upload_new(&g->tw, pass_twiddles(split ? g->logM - 1 : g->logM)));
  if (split) CHECK(upload_new(&g->octM, octant_table(g->logM)));
  CHECK(upload_new(&g->chirp, chirp));
  CHECK(upload_new(&g->bl_fwd, spectrum_brev(b)));
  CHECK(upload_new(&g->bl_inv, spectrum_brev(cc)));
  CHECK(upload_new(&g->wconv, spectrum_brev(w)));
  CHECK(upload_new(&g->ph1, ph1));
  CHECK(upload_new(&g->ph2, ph2));
  CHECK(upload_new(&g->chirp2, chirp2));
  CHECK(upload_new(&g->bl_ev, spectrum_brev(cc2)));
  CHECK(upload_new(&g->bl_fwd2, spectrum_brev(b2)));
  CHECK(upload_new(&g->ph4, ph4));
  CHECK(upload_new(&g->ph2d, ph2d));
  CHECK(upload_new(&g->ph4d, ph4d));
  if (N == 4095) {
    // k2 stage kernels (fft_kernels.cu): 4096-point engine twiddles, the |sin|
    // series on one parity class w_hat(2d) = 4/(1 - 4d^2), |d| <= 2047, and the
    // bin phases of the theta / theta_syn stages with the chirps folded out
    const int M2 = 4096;
    std::vector<cld> w2(M2, cld(0, 0));
    for (int d = -(M2 / 2 - 1); d <= M2 / 2 - 1; ++d)
      w2[(d + M2) % M2] = cld(4.0L / (1.0L - 4.0L * (ld)d * (ld)d), 0);
    std::vector<double2> phA(N), phS(N);
    for (int n = 0; n < N; ++n) {
      const int q = n < k ? n : n - N;
      const ld a1 = -PI_L * (ld)q / (ld)N;
      phA[n] = d2(cld(std::cos(a1), std::sin(a1)) / (ld)N);
      const ld a2 = -PI_L * (ld)q / (ld)N2 + PI_L * (ld)q / (ld)N;
      phS[n] = d2(cld(std::cos(a2), std::sin(a2)) / (ld)N2);
    }
    CHECK(upload_new(&g->tw12, pass_twiddles(12)));
    std::vector<double> w2r;
    for (const double2& z : spectrum_brev(w2)) w2r.push_back(z.x);  // Im ~ 1e-19: exact zero
    CHECK(upload_new(&g->w2s, w2r));
    CHECK(upload_new(&g->phA, phA));
    // theta_syn_k2 applies phS in the gather of the axis-9 prime-factor pass
    // (pfa_pass_gather: line r, element j is sample (9 r + 455 j) mod N, read
    // as entry j * 455 + r): stored in that order, a warp's loads are contiguous
    std::vector<double2> phS9(N);
    for (int r = 0; r < N / 9; ++r)
      for (int j = 0; j < 9; ++j) phS9[(size_t)j * (N / 9) + r] = phS[(9 * r + j * (N / 9)) % N];
    CHECK(upload_new(&g->phS, phS9));
  }
  if (N == 8191) {
    // k4 stage kernels: Rader's DFT_8191 over the prime-factor DFT_8190
    // (pfa.cuh), the |sin| series on one parity class at M = 8192, and the
    // theta / theta_syn bin phases
    const int R = 8190, G = 17, STEP = 253, M4 = 8192;
    std::vector<int> gpow(R), plog(N, 0);
    long long gq = 1;
    for (int q = 0; q < R; ++q) {
      gpow[q] = (int)gq;
      gq = gq * G % N;
    }
    long long ginv = 1;  // G^(N-2) mod N
    for (int e = 0; e < N - 2; ++e) ginv = ginv * G % N;
    std::vector<cld> dd(R);
    long long gi = 1;  // g^-j
    for (int j = 0; j < R; ++j) {
      plog[gi] = j;
      const ld ang = -2.0L * PI_L * (ld)gi / (ld)N;
      dd[j] = cld(std::cos(ang), std::sin(ang));
      gi = gi * ginv % N;
    }
    // DFT_8190 of d in long double by the same prime-factor passes as the
    // kernels (pfa.cuh): natural order in, bin k at slot 253 k mod 8190 out,
    // which is exactly the slot order the kernels multiply in
    std::vector<double2> Dslot(R);
    {
      std::vector<cld> b(dd);
      for (int P : {13, 7, 5, 9, 2}) {
        const int A = R / P;
        std::vector<cld> W(P * P);
        for (int u = 0; u < P; ++u)
          for (int v = 0; v < P; ++v) {
            const ld ang = -2.0L * PI_L * (ld)((u * v) % P) / (ld)P;
            W[u * P + v] = cld(std::cos(ang), std::sin(ang));
          }
        std::vector<cld> x(P), y(P);
        for (int r = 0; r < A; ++r) {
          for (int j = 0; j < P; ++j) x[j] = b[(P * r + j * A) % R];
          for (int u = 0; u < P; ++u) {
            cld acc(0, 0);
            for (int v = 0; v < P; ++v) acc += W[u * P + v] * x[v];
            y[u] = acc;
          }
          for (int j = 0; j < P; ++j) b[(P * r + j * A) % R] = y[j];
        }
      }
      for (int i = 0; i < R; ++i) Dslot[i] = d2(b[i] / (ld)R);
      (void)STEP;
    }
    std::vector<cld> w4(M4, cld(0, 0));
    for (int d = -(M4 / 2 - 1); d <= M4 / 2 - 1; ++d)
      w4[(d + M4) % M4] = cld(4.0L / (1.0L - 4.0L * (ld)d * (ld)d), 0);
    std::vector<double> w4r;
    for (const double2& z : spectrum_brev(w4)) w4r.push_back(z.x);  // Im ~ 1e-19: exact zero
    std::vector<double2> phA(N), phS(N);
    for (int n = 0; n < N; ++n) {
      const int q = n < k ? n : n - N;
      const ld a1 = -PI_L * (ld)q / (ld)N;
      phA[n] = d2(cld(std::cos(a1), std::sin(a1)) / (ld)N);
      const ld a2 = -PI_L * (ld)q / (ld)N2 + PI_L * (ld)q / (ld)N;
      phS[n] = d2(cld(std::cos(a2), std::sin(a2)) / (ld)N2);
    }
    CHECK(upload_new(&g->rgpow, gpow));
    CHECK(upload_new(&g->rplog, plog));
    CHECK(upload_new(&g->rD, Dslot));
    CHECK(upload_new(&g->w4s, w4r));
    CHECK(upload_new(&g->phA, phA));
    // theta_syn_k4 applies phS in Rader's input gather (rader8191_from: entry q
    // is sample g^q, entry 8190 sample 0): stored in that order
    std::vector<double2> phSg(N);
    for (int q = 0; q < N - 1; ++q) phSg[q] = phS[gpow[q]];
    phSg[N - 1] = phS[0];
    CHECK(upload_new(&g->phS, phSg));
  }
  if (scheme == S2W_SCHEME_MW) CHECK(theta_setup(g));
  return S2W_OK;
}

// ------------------------------------------------------------------ Legendre launch configs
static int pick_ns(int n, bool cplx) {
  const int cap = cplx ? 8 : 16;
  int ns = 1;
  while (ns < n && ns < cap) ns *= 2;
  return ns;
}

// Side stream for the Reinsch launch of the low orders (legendre_kernels.cu,
// REIN): forked from and joined back into the caller's stream with events,
// so it runs beside the plain launch (and CUDA-graph capture follows it).
struct SideLane {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  SideLane() = default;
  SideLane(const SideLane&) = delete;
  SideLane& operator=(const SideLane&) = delete;
  ~SideLane() {
    if (s) cudaStreamDestroy(s);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
  }
  int ensure() {
    if (s) return S2W_OK;
    // highest priority: the low orders are the heaviest items, so their CTAs
    // should take SMs before the plain launch's
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
    CU(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    return S2W_OK;
  }
  // launch `side_fn` on the lane and `main_fn` on st, joined back into st on
  // every exit path
  template <class F, class G>
  int fork_join(cudaStream_t st, F&& side_fn, G&& main_fn) {
    CHECK(ensure());
    CU(cudaEventRecord(fork, st));
    CU(cudaStreamWaitEvent(s, fork, 0));
    const cudaError_t e1 = side_fn(s);
    const cudaError_t e2 = e1 == cudaSuccess ? main_fn(st) : cudaSuccess;
    CU(cudaEventRecord(join, s));
    CU(cudaStreamWaitEvent(st, join, 0));
    CU(e1);
    CU(e2);
    return S2W_OK;
  }
};

static int item_grid(const SynthItem& it) { return it.grid; }
static int item_grid(const AnaItem&) { return 0; }  // analysis grids are all symmetric when sym

// Items of the low orders on equator-symmetric ring sets go first (Reinsch
// launch; the symmetric kernels sweep only their northern rings, x >= 0, where
// the Reinsch form applies); returns their count.  Cost order is kept within
// each part.  Asymmetric grids of a symmetric launch keep the plain recursion.
template <class It>
static int rein_partition(std::vector<It>& items, bool sym, const std::vector<LegGridDev>& grids,
                          bool per_item_grid) {
  if (!sym) return 0;
  auto mid = std::stable_partition(items.begin(), items.end(), [&](const It& i) {
    if (i.it.m >= S2W_REIN_M) return false;
    return !per_item_grid || grids[item_grid(i.it)].n_north > 0;
  });
  return (int)(mid - items.begin());
}

struct SynthCfg {
  bool built = false;
  int n_rein = 0;
  mutable SideLane lane;
  int key[4] = {0, 0, 0, 0};
  DevBuf grids, sets, items;
  int n_items = 0, ns = 1, cplx = 1, win = 32, sym = 0;
};

struct AnaCfg {
  bool built = false;
  int n_rein = 0;
  mutable SideLane lane;
  DevBuf pipe;  // leg_ana_pipe_kernel's inter-pass ring states ([item][ring][3])
  long long pipe_stride = 0;
  int key[4] = {0, 0, 0, 0};
  DevBuf grids, sets, segs, items;
  int n_items = 0, ns = 1, cplx = 1, win = 32, sym = 0;
};

// A synthesis "group": sets sharing one grid.
struct SynthGroupSpec {
  const GridRes* g;
  std::vector<SynthSet> sets;
};

static int build_synth(SynthCfg& cfg, const std::vector<SynthGroupSpec>& groups, bool cplx) {
  std::vector<LegGridDev> grids;
  std::vector<SynthSet> sets;
  struct It {
    SynthItem it;
    double cost;
  };
  std::vector<It> items;
  int maxn = 1;
  for (auto& gr : groups) maxn = std::max<int>(maxn, (int)gr.sets.size());
  // the symmetric kernel also runs asymmetric grids (n_north == 0) as such
  cfg.sym = 0;
  for (auto& gr : groups) cfg.sym |= gr.g->leg(cplx, false).n_north > 0 ? 1 : 0;
  // symmetric rings keep two accumulator sets: at most 4 complex / 8 real sets per CTA
  int ns = cfg.sym ? std::min(pick_ns(maxn, cplx), cplx ? 4 : 8) : pick_ns(maxn, cplx);
  {
    static const int cap = getenv("S2W_SYN_NS_CAP") ? atoi(getenv("S2W_SYN_NS_CAP")) : 0;
    if (cap > 0) ns = std::min(ns, cap);
    // two complex sets on symmetric rings: two one-set items per order run
    // faster than one two-set item (the one-set kernel keeps two CTAs per SM)
    else if (cap == 0 && cfg.sym && cplx && ns == 2) ns = 1;
  }
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const auto& gr = groups[gi];
    grids.push_back(gr.g->leg(cplx, false));
    const int base = (int)sets.size();
    for (auto& s : gr.sets) sets.push_back(s);
    const int n = (int)gr.sets.size();
    for (int m = 0; m < gr.g->k; ++m)
      for (int s0 = 0; s0 < n; s0 += ns) {
        const int nset = std::min(ns, n - s0);
        SynthItem it{(int)gi, m, base + s0, nset};
        items.push_back({it, gr.g->cost(m, false) * (3.0 + 4.0 * ns)});
      }
  }
  std::stable_sort(items.begin(), items.end(),
                   [](const It& a, const It& b) { return a.cost > b.cost; });
  cfg.n_rein = rein_partition(items, cfg.sym != 0, grids, true);
  std::vector<SynthItem> its;
  for (auto& i : items) its.push_back(i.it);
  CHECK(cfg.grids.upload(grids));
  CHECK(cfg.sets.upload(sets));
  CHECK(cfg.items.upload(its));
  cfg.n_items = (int)its.size();
  cfg.ns = ns;
  cfg.cplx = cplx;
  int kmax = 1;
  for (auto& gr : groups) kmax = std::max(kmax, gr.g->k);
  cfg.win = leg_synth_window(kmax, ns, cplx);
  cfg.built = true;
  return S2W_OK;
}

// Analysis: a segment = sets of one grid processed together.  combine != 0
// means all sets of the segment accumulate into the same output (weighted).
struct AnaSegSpec {
  const GridRes* g;
  std::vector<AnaSet> sets;
  int combine;
};

// Scratch of the pipelined analysis kernel when it serves this launch.
static int ana_pipe_setup(AnaCfg& cfg, const std::vector<LegGridDev>& grids, int kmax) {
  cfg.pipe_stride = 0;
  if (!leg_ana_pipe_ok(kmax, cfg.ns, cfg.cplx, cfg.sym)) return S2W_OK;
  int nn = 1;
  for (auto& g : grids) nn = std::max(nn, g.n_north);
  cfg.pipe_stride = 3LL * nn;
  CHECK(cfg.pipe.ensure(sizeof(double) * (size_t)std::max(1, cfg.n_items) * cfg.pipe_stride));
  return S2W_OK;
}

static int build_ana(AnaCfg& cfg, const std::vector<AnaSegSpec>& segspecs, bool cplx) {
  // distinct grids
  std::vector<const GridRes*> gl;
  for (auto& s : segspecs)
    if (std::find(gl.begin(), gl.end(), s.g) == gl.end()) gl.push_back(s.g);
  std::vector<LegGridDev> grids;
  for (auto* g : gl) grids.push_back(g->leg(cplx, true));
  cfg.sym = 1;
  for (auto& gd : grids) cfg.sym &= gd.n_north > 0 ? 1 : 0;
  int maxn = 1, kmax = 0;
  for (auto& s : segspecs) maxn = std::max<int>(maxn, (int)s.sets.size());
  for (auto* g : gl) kmax = std::max(kmax, g->k);
  // symmetric rings: at most 16 reals per degree (the symmetric DMMA kernel's
  // two operand sets must fit the registers); wider batches become segments
  const int ns = cfg.sym ? std::min(pick_ns(maxn, cplx), cplx ? 4 : 8) : pick_ns(maxn, cplx);
  // split segments wider than ns
  std::vector<AnaSet> sets;
  std::vector<AnaSeg> segs0;
  std::vector<int> seg_grid_k;
  for (auto& sp : segspecs) {
    const int gi = (int)(std::find(gl.begin(), gl.end(), sp.g) - gl.begin());
    const int n = (int)sp.sets.size();
    for (int s0 = 0; s0 < n; s0 += ns) {
      AnaSeg sg;
      sg.grid = gi;
      sg.set0 = (int)sets.size();
      sg.nset = std::min(ns, n - s0);
      sg.combine = sp.combine;
      for (int i = 0; i < sg.nset; ++i) sets.push_back(sp.sets[s0 + i]);
      segs0.push_back(sg);
    }
  }
  // items: one per order m, listing every segment whose grid has k > m
  struct It {
    AnaItem it;
    double cost;
  };
  std::vector<AnaSeg> segs;
  std::vector<It> items;
  // Segments that accumulate into a common output share an item (their folds
  // run in order inside one CTA); segments with disjoint outputs get an item
  // (CTA) each.  Components by union-find over shared outputs.
  const int nsg = (int)segs0.size();
  std::vector<int> comp(nsg);
  for (int i = 0; i < nsg; ++i) comp[i] = i;
  std::function<int(int)> root = [&](int i) { return comp[i] == i ? i : comp[i] = root(comp[i]); };
  std::map<std::pair<int, long long>, int> owner;
  for (int i = 0; i < nsg; ++i)
    for (int q = 0; q < segs0[i].nset; ++q) {
      const AnaSet& S = sets[segs0[i].set0 + q];
      auto key = std::make_pair(S.ob, S.ooff);
      auto f = owner.find(key);
      if (f == owner.end()) owner[key] = i;
      else comp[root(i)] = root(f->second);
    }
  for (int m = 0; m < kmax; ++m) {
    for (int c0 = 0; c0 < nsg; ++c0) {
      if (root(c0) != c0) continue;
      AnaItem it{m, (int)segs.size(), 0};
      double cost = 0;
      for (int i = 0; i < nsg; ++i) {
        const GridRes* g = gl[segs0[i].grid];
        if (root(i) != c0 || m >= g->k) continue;
        segs.push_back(segs0[i]);
        ++it.nseg;
        cost += g->cost(m, true) * (3.0 + 4.0 * ns);
      }
      if (it.nseg) items.push_back({it, cost});
    }
  }
  std::stable_sort(items.begin(), items.end(),
                   [](const It& a, const It& b) { return a.cost > b.cost; });
  cfg.n_rein = rein_partition(items, cfg.sym != 0, grids, false);
  std::vector<AnaItem> its;
  for (auto& i : items) its.push_back(i.it);
  CHECK(cfg.grids.upload(grids));
  CHECK(cfg.sets.upload(sets));
  CHECK(cfg.segs.upload(segs));
  CHECK(cfg.items.upload(its));
  cfg.n_items = (int)its.size();
  cfg.ns = ns;
  cfg.cplx = cplx;
  cfg.win = leg_ana_window(kmax, ns, cplx);
  CHECK(ana_pipe_setup(cfg, grids, kmax));
  cfg.built = true;
  return S2W_OK;
}

static int run_synth(const SynthCfg& cfg, const double* seed_c, double2* const* bufs,
                     cudaStream_t st) {
  LegSynthArgs a;
  a.grids = cfg.grids.as<LegGridDev>();
  a.sets = cfg.sets.as<SynthSet>();
  a.items = cfg.items.as<SynthItem>();
  a.seed_c = seed_c;
  a.n_items = cfg.n_items;
  a.cplx = cfg.cplx;
  a.ns = cfg.ns;
  a.win = cfg.win;
  a.sym = cfg.sym;
  a.rein = 0;
  for (int i = 0; i < S2W_NBUF; ++i) a.bufs[i] = bufs[i];
  ProfScope ps(P_LEG_SYNTH, st);
  if (cfg.n_rein == 0) {
    CU(launch_leg_synth(a, st));
    return S2W_OK;
  }
  LegSynthArgs r = a;
  r.n_items = cfg.n_rein;
  r.rein = 1;
  a.items += cfg.n_rein;
  a.n_items -= cfg.n_rein;
  ++g_launches;
  return cfg.lane.fork_join(st, [&](cudaStream_t s) { return launch_leg_synth(r, s); },
                            [&](cudaStream_t s) { return launch_leg_synth(a, s); });
}

static int run_ana(const AnaCfg& cfg, const double* seed_c, double2* const* bufs,
                   cudaStream_t st) {
  LegAnaArgs a;
  a.grids = cfg.grids.as<LegGridDev>();
  a.sets = cfg.sets.as<AnaSet>();
  a.segs = cfg.segs.as<AnaSeg>();
  a.items = cfg.items.as<AnaItem>();
  a.seed_c = seed_c;
  a.n_items = cfg.n_items;
  a.cplx = cfg.cplx;
  a.ns = cfg.ns;
  a.win = cfg.win;
  a.sym = cfg.sym;
  a.rein = 0;
  a.pipe_scratch = cfg.pipe_stride ? cfg.pipe.as<double>() : nullptr;
  a.pipe_stride = cfg.pipe_stride;
  for (int i = 0; i < S2W_NBUF; ++i) a.bufs[i] = bufs[i];
  ProfScope ps(P_LEG_ANA, st);
  if (cfg.n_rein == 0) {
    CU(launch_leg_ana(a, st));
    return S2W_OK;
  }
  LegAnaArgs r = a;
  r.n_items = cfg.n_rein;
  r.rein = 1;
  a.items += cfg.n_rein;
  a.n_items -= cfg.n_rein;
  ++g_launches;
  return cfg.lane.fork_join(st, [&](cudaStream_t s) { return launch_leg_ana(r, s); },
                            [&](cudaStream_t s) { return launch_leg_ana(a, s); });
}

// ------------------------------------------------------------------ shared pipeline steps
// map [n_sets][k][N] -> H [n_sets][mi][k] (m-major; MW: theta stage applied)
static int forward_rings(const GridRes* g, int n_sets, bool real, const double* map,
                         double2* G, double2* scratch, cudaStream_t st) {
  PhiFwdArgs pa;
  pa.scratch = scratch;
  pa.T = g->fft();
  pa.n_sets = n_sets;
  pa.n_rings = g->k;
  pa.real = real ? 1 : 0;
  pa.in = map;
  pa.out = G;
  pa.n_bins = g->n_bins(!real);
  pa.scale = 1.0 / (double)g->N;
  {
    ProfScope ps(P_PHI_FWD, st);
    CU(launch_phi_fwd(pa, st));
  }
  if (g->scheme == S2W_SCHEME_MW) {
    ThetaArgs ta = g->theta(!real);
    ta.n_sets = n_sets;
    ta.in = G;
    ta.out = G;
    ta.scratch = scratch;
    ProfScope ps(P_THETA, st);
    CU(launch_theta(ta, st));
  }
  return S2W_OK;
}

// G ring-major [n_sets][k][n_bins] -> map [n_sets][k][N]
// Resample synthesis output from the analysis rings (m-major) to the MW rings
// (ring-major): theta_syn_kernel.
static int theta_resample(const GridRes* g, int n_sets, bool real, const double2* Gm,
                          double2* Gr, double2* scratch, cudaStream_t st) {
  ThetaSynArgs ta;
  ta.T = g->fft();
  ta.n_sets = n_sets;
  ta.k = g->k;
  ta.n_bins = g->n_bins(!real);
  ta.pairs = real ? g->pairs_r : g->pairs_c;
  ta.n_pairs = real ? g->np_r : g->np_c;
  ta.in = Gm;
  ta.out = Gr;
  ta.scratch = scratch;
  ProfScope ps(P_THETA, st);
  CU(launch_theta_syn(ta, st));
  return S2W_OK;
}

// Ring-major G on the sampling rings -> maps (ring DFTs, MW pole pin).
static int phi_inverse(const GridRes* g, int n_sets, bool real, const double2* G, double* map,
                       double2* scratch, cudaStream_t st, double thresh = 0.0) {
  PhiInvArgs pa;
  pa.thresh = thresh;
  pa.scratch = scratch;
  pa.T = g->fft();
  pa.n_sets = n_sets;
  pa.n_rings = g->k;
  pa.real = real ? 1 : 0;
  pa.mw_pole = g->scheme == S2W_SCHEME_MW;
  pa.t_offset = 0;
  pa.in = G;
  pa.out = map;
  pa.n_bins = g->n_bins(!real);
  ProfScope ps(P_PHI_INV, st);
  CU(launch_phi_inv(pa, st));
  return S2W_OK;
}

// Legendre synthesis output G -> maps.  MW: G is m-major on the analysis
// rings and is first resampled into tmp (ring-major, MW rings).
static int inverse_rings(const GridRes* g, int n_sets, bool real, const double2* G, double* map,
                         double2* scratch, double2* tmp, cudaStream_t st, double thresh = 0.0) {
  if (g->syn_on_ana()) {
    CHECK(theta_resample(g, n_sets, real, G, tmp, scratch, st));
    G = tmp;
  }
  return phi_inverse(g, n_sets, real, G, map, scratch, st, thresh);
}

// ------------------------------------------------------------------ SHT plan
struct s2w_sht_plan {
  int device, scheme, L;
  GridRes* g;
  DevBuf G, G2, scratch;  // G2: MW resampling target
  SynthCfg syn;
  AnaCfg ana;
};

extern "C" {

const char* s2w_version(void) { return S2W_VERSION; }
const char* s2w_last_error(void) { return g_err.c_str(); }

int s2w_grid_nodes(int scheme, int L, double* theta, double* weights) {
  if (L < 1) return fail(S2W_EPARAM, "band-limit must be >= 1, got %d", L);
  if (scheme != S2W_SCHEME_GL && scheme != S2W_SCHEME_MW)
    return fail(S2W_EPARAM, "unknown sampling scheme %d", scheme);
  std::vector<double> th, w;
  if (scheme == S2W_SCHEME_GL) gl_nodes(L, th, w);
  else mw_nodes(L, th);
  if (theta) std::memcpy(theta, th.data(), sizeof(double) * L);
  if (weights && scheme == S2W_SCHEME_GL) std::memcpy(weights, w.data(), sizeof(double) * L);
  return S2W_OK;
}

int s2w_assoc_legendre_ring(int L, double theta, double* table, void* stream) {
  if (L < 1) return fail(S2W_EPARAM, "band-limit must be >= 1, got %d", L);
  if (L >= SEED_KMAX) return fail(S2W_EPARAM, "band-limit %d too large", L);
  if (!(theta >= 0.0 && theta <= M_PI))
    return fail(S2W_EPARAM, "colatitude must lie in [0, pi], got %g", theta);
  int dev;
  CU(cudaGetDevice(&dev));
  DeviceTables* dt;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    CHECK(device_tables(dev, &dt));
  }
  CU(launch_leg_table(L, std::cos(theta), std::sin(theta), dt->seed_c, table,
                      (cudaStream_t)stream));
  return S2W_OK;
}

int s2w_sht_plan_create(int scheme, int L, int device, s2w_sht_plan** plan) {
  if (!plan) return fail(S2W_EPARAM, "null plan pointer");
  if (L < 1) return fail(S2W_EPARAM, "band-limit must be >= 1, got %d", L);
  if (scheme != S2W_SCHEME_GL && scheme != S2W_SCHEME_MW)
    return fail(S2W_EPARAM, "unknown sampling scheme %d", scheme);
  DeviceGuard dg(device);
  CU(dg.err);
  s2w_sht_plan* p = new s2w_sht_plan();
  p->device = device;
  p->scheme = scheme;
  p->L = L;
  int r = get_grid(device, scheme, L, &p->g);
  if (r == S2W_OK) r = p->scratch.ensure(sizeof(double2) * fft_split_scratch_elems(p->g->logM));
  if (r != S2W_OK) {
    delete p;
    return r;
  }
  *plan = p;
  return S2W_OK;
}

int s2w_sht_plan_destroy(s2w_sht_plan* plan) {
  if (!plan) return S2W_OK;
  DeviceGuard dg(plan->device);
  delete plan;
  return S2W_OK;
}

int s2w_sh_synthesis(s2w_sht_plan* p, int n_sets, int L_coef, int is_real, const double* flm,
                     double* map, void* stream) {
  if (!p) return fail(S2W_EPARAM, "null plan");
  if (n_sets < 0) return fail(S2W_EPARAM, "negative set count");
  if (L_coef < 1 || L_coef > p->L)
    return fail(S2W_EPARAM, "coefficient band-limit %d exceeds the grid band-limit %d", L_coef,
                p->L);
  if (n_sets == 0) return S2W_OK;
  DeviceGuard dg(p->device);
  CU(dg.err);
  cudaStream_t st = (cudaStream_t)stream;
  const bool cplx = !is_real;
  const GridRes* g = p->g;
  const int k = g->k, nb = g->n_bins(cplx);
  CHECK(p->G.ensure(sizeof(double2) * (size_t)n_sets * nb * k));
  SynthCfg& c = p->syn;
  if (!c.built || c.key[0] != n_sets || c.key[1] != is_real || c.key[2] != L_coef) {
    SynthGroupSpec gs;
    gs.g = g;
    for (int s = 0; s < n_sets; ++s) {
      SynthSet ss;
      ss.fb = 0;
      ss.foff = (long long)s * L_coef * L_coef;
      ss.f_L = L_coef;
      ss.w = nullptr;
      ss.ob = 1;
      ss.ooff = (long long)s * nb * k;
      gs.sets.push_back(ss);
    }
    CHECK(build_synth(c, {gs}, cplx));
    c.key[0] = n_sets;
    c.key[1] = is_real;
    c.key[2] = L_coef;
  }
  double2* bufs[S2W_NBUF] = {(double2*)flm, p->G.as<double2>(), nullptr, nullptr};
  CHECK(run_synth(c, g->seed_c, bufs, st));
  if (g->syn_on_ana()) CHECK(p->G2.ensure(sizeof(double2) * (size_t)n_sets * nb * k));
  CHECK(inverse_rings(g, n_sets, !cplx, p->G.as<double2>(), map, p->scratch.as<double2>(),
                      p->G2.as<double2>(), st));
  return S2W_OK;
}

int s2w_sh_analysis(s2w_sht_plan* p, int n_sets, int is_real, const double* map, double* flm,
                    void* stream) {
  if (!p) return fail(S2W_EPARAM, "null plan");
  if (n_sets < 0) return fail(S2W_EPARAM, "negative set count");
  if (n_sets == 0) return S2W_OK;
  DeviceGuard dg(p->device);
  CU(dg.err);
  cudaStream_t st = (cudaStream_t)stream;
  const bool cplx = !is_real;
  const GridRes* g = p->g;
  const int k = g->k, nb = g->n_bins(cplx);
  CHECK(p->G.ensure(sizeof(double2) * (size_t)n_sets * nb * k));
  AnaCfg& c = p->ana;
  if (!c.built || c.key[0] != n_sets || c.key[1] != is_real) {
    AnaSegSpec sp;
    sp.g = g;
    sp.combine = 0;
    for (int s = 0; s < n_sets; ++s) {
      AnaSet as;
      as.hb = 1;
      as.hoff = (long long)s * nb * k;
      as.ob = 0;
      as.ooff = (long long)s * k * k;
      as.w = nullptr;
      sp.sets.push_back(as);
    }
    CHECK(build_ana(c, {sp}, cplx));
    c.key[0] = n_sets;
    c.key[1] = is_real;
  }
  CHECK(forward_rings(g, n_sets, !cplx, map, p->G.as<double2>(), p->scratch.as<double2>(), st));
  CU(cudaMemsetAsync(flm, 0, sizeof(double2) * (size_t)n_sets * k * k, st));
  double2* bufs[S2W_NBUF] = {(double2*)flm, p->G.as<double2>(), nullptr, nullptr};
  CHECK(run_ana(c, g->seed_c, bufs, st));
  return S2W_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ wavelet plan
struct s2w_wav_plan {
  int device, scheme, L, B, real, nk;
  std::vector<int> bands;
  DevBuf fac;                         // [nk][L]
  GridRes* top = nullptr;             // grid at L
  std::vector<GridRes*> kgrid;        // grid per kernel index
  std::vector<long long> goff;        // offset (double2) of scale j's G block in Gs
  DevBuf f, Gtop, Gs, Gr, scratch;  // Gr: MW resampling target (one scale at a time)
  SynthCfg syn_top, syn_scales;
  AnaCfg ana_top, ana_scales;
  double2* bufs() const { return nullptr; }
  // Per-scale ring stages (phi / theta of each scale map) are independent:
  // they run on side streams forked from and joined back into the caller's
  // stream (event fork/join, so CUDA-graph capture follows them), largest
  // band first, each scale with its own resampling target and each side
  // stream with its own split-mode scratch.
  static constexpr int NSIDE = 4;
  bool concurrent = true;
  cudaStream_t side[NSIDE] = {};
  cudaEvent_t fork = nullptr, join[NSIDE] = {};
  std::vector<int> order;                 // scales by descending band
  std::vector<std::unique_ptr<DevBuf>> Grj;  // per scale resampling target (MW, k >= 1024)
  DevBuf sscratch[NSIDE];
  ~s2w_wav_plan() {
    for (int i = 0; i < NSIDE; ++i) {
      if (side[i]) cudaStreamDestroy(side[i]);
      if (join[i]) cudaEventDestroy(join[i]);
    }
    if (fork) cudaEventDestroy(fork);
  }
  // run f(j, stream, scratch, Gr_j) for every scale on the side streams
  template <class F>
  int per_scale(cudaStream_t st, F&& f) {
    if (!concurrent) {
      for (int j : order) CHECK(f(j, st, sscratch[0].as<double2>(), Grj[j] ? Grj[j]->as<double2>() : nullptr));
      return S2W_OK;
    }
    CU(cudaEventRecord(fork, st));
    const int ns = std::min<int>(NSIDE, (int)order.size());
    int r = S2W_OK, forked = 0;
    for (; forked < ns && r == S2W_OK; ++forked)
      if (cudaStreamWaitEvent(side[forked], fork, 0) != cudaSuccess)
        r = fail(S2W_ECUDA, "side stream fork failed");
    for (size_t i = 0; i < order.size() && r == S2W_OK; ++i) {
      const int j = order[i], q = (int)(i % NSIDE);
      r = f(j, side[q], sscratch[q].as<double2>(), Grj[j] ? Grj[j]->as<double2>() : nullptr);
    }
    // join every forked side stream on every exit path: a capture must end
    // with all branches joined, and eager callers must stay ordered after
    // side work that reuses sscratch
    for (int i = 0; i < forked; ++i) {
      const bool ok = cudaEventRecord(join[i], side[i]) == cudaSuccess &&
                      cudaStreamWaitEvent(st, join[i], 0) == cudaSuccess;
      if (!ok && r == S2W_OK) r = fail(S2W_ECUDA, "side stream join failed");
    }
    return r;
  }
};

extern "C" {

int s2w_wav_plan_create(int scheme, int L, int batch, int is_real, int n_kern,
                        const double* kernels, const int* bands, int device,
                        s2w_wav_plan** plan) {
  if (!plan || !kernels || !bands) return fail(S2W_EPARAM, "null argument");
  if (L < 2) return fail(S2W_EPARAM, "band-limit must be >= 2 for a wavelet tiling, got %d", L);
  if (batch < 1) return fail(S2W_EPARAM, "batch must be >= 1");
  if (n_kern < 1 || n_kern > S2W_MAXK)
    return fail(S2W_EPARAM, "kernel count %d out of range [1, %d]", n_kern, S2W_MAXK);
  if (scheme != S2W_SCHEME_GL && scheme != S2W_SCHEME_MW)
    return fail(S2W_EPARAM, "unknown sampling scheme %d", scheme);
  for (int j = 0; j < n_kern; ++j)
    if (bands[j] < 1 || bands[j] > L)
      return fail(S2W_EPARAM, "scale band-limit %d outside [1, %d]", bands[j], L);
  DeviceGuard dg(device);
  CU(dg.err);
  s2w_wav_plan* p = new s2w_wav_plan();
  p->device = device;
  p->scheme = scheme;
  p->L = L;
  p->B = batch;
  p->real = is_real ? 1 : 0;
  p->nk = n_kern;
  p->bands.assign(bands, bands + n_kern);
  auto bail = [&](int r) {
    delete p;
    return r;
  };
  // tiling factors sqrt(4 pi / (2l+1)) * K_j(l)  (transform.py:117-126)
  std::vector<double> fac((size_t)n_kern * L);
  for (int j = 0; j < n_kern; ++j)
    for (int l = 0; l < L; ++l)
      fac[(size_t)j * L + l] = std::sqrt(4.0 * M_PI / (2.0 * l + 1.0)) * kernels[(size_t)j * L + l];
  int r;
  if ((r = p->fac.upload(fac)) != S2W_OK) return bail(r);
  if ((r = get_grid(device, scheme, L, &p->top)) != S2W_OK) return bail(r);
  const bool cplx = !is_real;
  long long off = 0;
  for (int j = 0; j < n_kern; ++j) {
    GridRes* g;
    if ((r = get_grid(device, scheme, bands[j], &g)) != S2W_OK) return bail(r);
    p->kgrid.push_back(g);
    p->goff.push_back(off);
    off += (long long)batch * g->n_bins(cplx) * g->k;
  }
  if ((r = p->f.ensure(sizeof(double2) * (size_t)batch * L * L)) != S2W_OK) return bail(r);
  if ((r = p->Gtop.ensure(sizeof(double2) * (size_t)batch * p->top->n_bins(cplx) * L)) != S2W_OK)
    return bail(r);
  if ((r = p->Gs.ensure(sizeof(double2) * (size_t)off)) != S2W_OK) return bail(r);
  if (p->top->syn_on_ana() &&
      (r = p->Gr.ensure(sizeof(double2) * (size_t)batch * p->top->n_bins(cplx) * L)) != S2W_OK)
    return bail(r);
  if ((r = p->scratch.ensure(sizeof(double2) * fft_split_scratch_elems(p->top->logM))) != S2W_OK)
    return bail(r);
  // side streams, per-scale resampling targets and per-stream scratch
  for (int i = 0; i < s2w_wav_plan::NSIDE; ++i) {
    if (cudaStreamCreateWithFlags(&p->side[i], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->join[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(S2W_ECUDA, "side stream / event creation failed"));
    if ((r = p->sscratch[i].ensure(sizeof(double2) * fft_split_scratch_elems(p->top->logM))) != S2W_OK)
      return bail(r);
  }
  if (cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(S2W_ECUDA, "event creation failed"));
  for (int j = 0; j < n_kern; ++j) p->order.push_back(j);
  std::stable_sort(p->order.begin(), p->order.end(),
                   [&](int a, int b) { return p->bands[a] > p->bands[b]; });
  p->Grj.resize(n_kern);
  for (int j = 0; j < n_kern; ++j) {
    const GridRes* g = p->kgrid[j];
    if (!g->syn_on_ana()) continue;
    p->Grj[j].reset(new DevBuf());
    if ((r = p->Grj[j]->ensure(sizeof(double2) * (size_t)batch * g->n_bins(cplx) * g->k)) != S2W_OK)
      return bail(r);
  }

  // slots: 0 = f, 1 = Gtop, 2 = Gs
  const int nbL = p->top->n_bins(cplx);
  // (a) analysis at L into f (plain)
  {
    AnaSegSpec sp;
    sp.g = p->top;
    sp.combine = 0;
    for (int b = 0; b < batch; ++b)
      sp.sets.push_back(AnaSet{1, (long long)b * nbL * L, 0, (long long)b * L * L, nullptr});
    if ((r = build_ana(p->ana_top, {sp}, cplx)) != S2W_OK) return bail(r);
  }
  // (b) synthesis at L from f (plain)
  {
    SynthGroupSpec gs;
    gs.g = p->top;
    for (int b = 0; b < batch; ++b)
      gs.sets.push_back(SynthSet{0, (long long)b * L * L, L, nullptr, 1, (long long)b * nbL * L});
    if ((r = build_synth(p->syn_top, {gs}, cplx)) != S2W_OK) return bail(r);
  }
  // distinct scale grids (ascending band)
  std::vector<int> distinct(p->bands);
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  // (c) grouped per-scale synthesis: f * fac_j, truncated to band_j
  {
    std::vector<SynthGroupSpec> groups;
    for (int kb : distinct) {
      SynthGroupSpec gs;
      for (int j = 0; j < n_kern; ++j) {
        if (p->bands[j] != kb) continue;
        gs.g = p->kgrid[j];
        const int nb = gs.g->n_bins(cplx);
        for (int b = 0; b < batch; ++b)
          gs.sets.push_back(SynthSet{0, (long long)b * L * L, L, p->fac.as<double>() + (size_t)j * L,
                                     2, p->goff[j] + (long long)b * nb * kb});
      }
      groups.push_back(gs);
    }
    if ((r = build_synth(p->syn_scales, groups, cplx)) != S2W_OK) return bail(r);
  }
  // (d) grouped per-scale analysis recombined into f (weighted by fac_j)
  {
    std::vector<AnaSegSpec> segs;
    for (int kb : distinct) {
      std::vector<int> js;
      for (int j = 0; j < n_kern; ++j)
        if (p->bands[j] == kb) js.push_back(j);
      const GridRes* g = p->kgrid[js[0]];
      const int nb = g->n_bins(cplx);
      if ((int)js.size() > 1 && batch == 1) {
        // one output, several weighted scales: share the recursion
        AnaSegSpec sp;
        sp.g = g;
        sp.combine = 1;
        for (int j : js)
          sp.sets.push_back(AnaSet{2, p->goff[j], 0, 0, p->fac.as<double>() + (size_t)j * L});
        segs.push_back(sp);
      } else {
        for (int j : js) {
          AnaSegSpec sp;
          sp.g = g;
          sp.combine = 0;
          for (int b = 0; b < batch; ++b)
            sp.sets.push_back(AnaSet{2, p->goff[j] + (long long)b * nb * kb, 0, (long long)b * L * L,
                                     p->fac.as<double>() + (size_t)j * L});
          segs.push_back(sp);
        }
      }
    }
    if ((r = build_ana(p->ana_scales, segs, cplx)) != S2W_OK) return bail(r);
  }
  *plan = p;
  return S2W_OK;
}

int s2w_wav_plan_destroy(s2w_wav_plan* plan) {
  if (!plan) return S2W_OK;
  DeviceGuard dg(plan->device);
  delete plan;
  return S2W_OK;
}

int s2w_wav_plan_set_concurrency(s2w_wav_plan* p, int on) {
  if (!p) return fail(S2W_EPARAM, "null argument");
  p->concurrent = on != 0;
  return S2W_OK;
}

int s2w_wav_plan_flm(s2w_wav_plan* p, double** flm) {
  if (!p || !flm) return fail(S2W_EPARAM, "null argument");
  *flm = p->f.as<double>();
  return S2W_OK;
}

int s2w_wav_analysis_harmonic(s2w_wav_plan* p, int truncate, const double* flm,
                              double* const* outs, void* stream) {
  if (!p || !flm || !outs) return fail(S2W_EPARAM, "null argument");
  DeviceGuard dg(p->device);
  CU(dg.err);
  TileArgs a;
  a.n_sets = p->B;
  a.L = p->L;
  a.n_k = p->nk;
  a.fac = p->fac.as<double>();
  for (int j = 0; j < p->nk; ++j) {
    a.band[j] = truncate ? p->bands[j] : p->L;
    a.ptr[j] = (double2*)outs[j];
  }
  a.f_in = (const double2*)flm;
  a.f_out = nullptr;
  ProfScope ps(P_TILE, (cudaStream_t)stream);
  CU(launch_tile_analysis(a, (cudaStream_t)stream));
  return S2W_OK;
}

int s2w_wav_synthesis_harmonic(s2w_wav_plan* p, int full_band, const double* const* ins,
                               double* flm, void* stream) {
  if (!p || !flm || !ins) return fail(S2W_EPARAM, "null argument");
  DeviceGuard dg(p->device);
  CU(dg.err);
  TileArgs a;
  a.n_sets = p->B;
  a.L = p->L;
  a.n_k = p->nk;
  a.fac = p->fac.as<double>();
  for (int j = 0; j < p->nk; ++j) {
    a.band[j] = full_band ? p->L : p->bands[j];
    a.ptr[j] = (double2*)ins[j];
  }
  a.f_in = nullptr;
  a.f_out = (double2*)flm;
  ProfScope ps(P_TILE, (cudaStream_t)stream);
  CU(launch_tile_synthesis(a, (cudaStream_t)stream));
  return S2W_OK;
}

static int wav_analysis_pixel_impl(s2w_wav_plan* p, const double* map, const double* thresholds,
                                   double* const* scale_maps, void* stream);

int s2w_wav_analysis_pixel(s2w_wav_plan* p, const double* map, double* const* scale_maps,
                           void* stream) {
  return wav_analysis_pixel_impl(p, map, nullptr, scale_maps, stream);
}

int s2w_wav_analysis_pixel_threshold(s2w_wav_plan* p, const double* map, const double* thresholds,
                                     double* const* scale_maps, void* stream) {
  if (!thresholds) return fail(S2W_EPARAM, "null threshold table");
  return wav_analysis_pixel_impl(p, map, thresholds, scale_maps, stream);
}

int s2w_wav_denoise_pixel(s2w_wav_plan* p, const double* map, const double* thresholds,
                          double* const* scale_maps, double* map_out, void* stream) {
  if (!thresholds || !map_out) return fail(S2W_EPARAM, "null argument");
  CHECK(wav_analysis_pixel_impl(p, map, thresholds, scale_maps, stream));
  return s2w_wav_synthesis_pixel(p, (const double* const*)scale_maps, map_out, stream);
}

static int wav_analysis_pixel_impl(s2w_wav_plan* p, const double* map, const double* thresholds,
                                   double* const* scale_maps, void* stream) {
  if (!p || !map || !scale_maps) return fail(S2W_EPARAM, "null argument");
  if (thresholds)
    for (int j = 1; j < p->nk; ++j)
      if (!(thresholds[j] >= 0.0)) return fail(S2W_EPARAM, "threshold %d must be >= 0", j);
  DeviceGuard dg(p->device);
  CU(dg.err);
  cudaStream_t st = (cudaStream_t)stream;
  const bool cplx = !p->real;
  double2* bufs[S2W_NBUF] = {p->f.as<double2>(), p->Gtop.as<double2>(), p->Gs.as<double2>(),
                             nullptr};
  // sh_analysis at L (transform.py:186)
  CHECK(forward_rings(p->top, p->B, !cplx, map, p->Gtop.as<double2>(), p->scratch.as<double2>(),
                      st));
  CU(cudaMemsetAsync(p->f.p, 0, sizeof(double2) * (size_t)p->B * p->L * p->L, st));
  CHECK(run_ana(p->ana_top, p->top->seed_c, bufs, st));
  // tiling + truncation fused into the grouped per-scale synthesis (transform.py:187-190)
  CHECK(run_synth(p->syn_scales, p->top->seed_c, bufs, st));
  // hard thresholding of the wavelet maps (not the scaling map) fused into
  // the ring-DFT epilogue (denoise.py:78-96)
  return p->per_scale(st, [&](int j, cudaStream_t s, double2* scratch, double2* Gr) {
    return inverse_rings(p->kgrid[j], p->B, !cplx, p->Gs.as<double2>() + p->goff[j], scale_maps[j],
                         scratch, Gr, s, (thresholds && j > 0) ? thresholds[j] : 0.0);
  });
}

int s2w_wav_synthesis_pixel(s2w_wav_plan* p, const double* const* scale_maps, double* map,
                            void* stream) {
  if (!p || !map || !scale_maps) return fail(S2W_EPARAM, "null argument");
  DeviceGuard dg(p->device);
  CU(dg.err);
  cudaStream_t st = (cudaStream_t)stream;
  const bool cplx = !p->real;
  double2* bufs[S2W_NBUF] = {p->f.as<double2>(), p->Gtop.as<double2>(), p->Gs.as<double2>(),
                             nullptr};
  // per-scale analysis (transform.py:196)
  CHECK(p->per_scale(st, [&](int j, cudaStream_t s, double2* scratch, double2*) {
    return forward_rings(p->kgrid[j], p->B, !cplx, scale_maps[j], p->Gs.as<double2>() + p->goff[j],
                         scratch, s);
  }));
  CU(cudaMemsetAsync(p->f.p, 0, sizeof(double2) * (size_t)p->B * p->L * p->L, st));
  // recombination (transform.py:197-199) fused into the analysis reduction
  CHECK(run_ana(p->ana_scales, p->top->seed_c, bufs, st));
  // sh_synthesis at L (transform.py:200)
  CHECK(run_synth(p->syn_top, p->top->seed_c, bufs, st));
  CHECK(inverse_rings(p->top, p->B, !cplx, p->Gtop.as<double2>(), map, p->scratch.as<double2>(),
                      p->Gr.as<double2>(), st));
  return S2W_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ accounting / probes
extern "C" {

long long s2w_kernel_launches(void) { return g_launches.load(); }

int s2w_real_to_complex(const double* in, double* out, long long n, void* stream) {
  if ((!in || !out) && n > 0) return fail(S2W_EPARAM, "null argument");
  CU(launch_real_to_complex(in, (double2*)out, n, (cudaStream_t)stream));
  return S2W_OK;
}

int s2w_complex_real_part(const double* in, double* out, long long n, void* stream) {
  if ((!in || !out) && n > 0) return fail(S2W_EPARAM, "null argument");
  CU(launch_complex_real_part((const double2*)in, out, n, (cudaStream_t)stream));
  return S2W_OK;
}

int s2w_profile_enable(int on) {
  g_prof = on != 0;
  return S2W_OK;
}

// Synchronises on the recorded events, accumulates per-stage milliseconds and
// launch counts since the last reset, and writes them in stage order
// (leg_synth, leg_ana, phi_fwd, theta, phi_inv, tile).  n = capacity.
int s2w_profile_read(int n, double* ms, long long* count, int reset) {
  for (auto& r : g_prof_pending) {
    float t = 0.f;
    CU(cudaEventSynchronize(r.b));
    CU(cudaEventElapsedTime(&t, r.a, r.b));
    g_prof_ms[r.stage] += t;
    g_prof_n[r.stage] += 1;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_pending.clear();
  for (int i = 0; i < n && i < P_NSTAGE; ++i) {
    if (ms) ms[i] = g_prof_ms[i];
    if (count) count[i] = g_prof_n[i];
  }
  if (reset)
    for (int i = 0; i < P_NSTAGE; ++i) {
      g_prof_ms[i] = 0;
      g_prof_n[i] = 0;
    }
  return S2W_OK;
}

const char* s2w_profile_stage_name(int i) { return (i >= 0 && i < P_NSTAGE) ? kStageNames[i] : ""; }

int s2w_fp64_peak(double* tflops, void* stream) {
  CU(s2w::measure_fp64_peak(tflops, (cudaStream_t)stream));
  return S2W_OK;
}

int s2w_dmma_peak(double* tflops, void* stream) {
  CU(s2w::measure_dmma_peak(tflops, (cudaStream_t)stream));
  return S2W_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ stage hooks (tests)
// Individual pipeline stages on one grid, for stage-level parity tests
// (include/s2w_testing.h).  Same kernels as the transforms above.
extern "C" {

static DevBuf g_test_scratch;

int s2w_test_rings_inverse(int scheme, int L, int n_sets, int is_real, const double* G,
                           double* map, void* stream) {
  int dev;
  CU(cudaGetDevice(&dev));
  GridRes* g;
  CHECK(get_grid(dev, scheme, L, &g));
  CHECK(g_test_scratch.ensure(sizeof(double2) * fft_split_scratch_elems(g->logM)));
  return phi_inverse(g, n_sets, is_real != 0, (const double2*)G, map,
                     g_test_scratch.as<double2>(), (cudaStream_t)stream);
}

int s2w_test_rings_forward(int scheme, int L, int n_sets, int is_real, int theta_stage,
                           const double* map, double* G, void* stream) {
  int dev;
  CU(cudaGetDevice(&dev));
  GridRes* g;
  CHECK(get_grid(dev, scheme, L, &g));
  PhiFwdArgs pa;
  pa.T = g->fft();
  pa.n_sets = n_sets;
  pa.n_rings = g->k;
  pa.real = is_real ? 1 : 0;
  pa.in = map;
  pa.out = (double2*)G;
  pa.n_bins = g->n_bins(!is_real);
  pa.scale = 1.0 / (double)g->N;
  CHECK(g_test_scratch.ensure(sizeof(double2) * fft_split_scratch_elems(g->logM)));
  pa.scratch = g_test_scratch.as<double2>();
  {
    ProfScope ps(P_PHI_FWD, (cudaStream_t)stream);
    CU(launch_phi_fwd(pa, (cudaStream_t)stream));
  }
  if (theta_stage) {
    ThetaArgs ta = g->theta(!is_real);
    ta.n_sets = n_sets;
    ta.in = (double2*)G;
    ta.out = (double2*)G;
    ta.scratch = g_test_scratch.as<double2>();
    ProfScope ps(P_THETA, (cudaStream_t)stream);
    CU(launch_theta(ta, (cudaStream_t)stream));
  }
  return S2W_OK;
}

}  // extern "C"
#include "capi_shard.inc"
