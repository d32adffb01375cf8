/*
 * s2w.h -- C ABI of the B200-native spherical-wavelet hot path.
 *
 * Drop-in boundary for the reference package `sphwav` (arXiv 1211.1680,
 * /root/reference/pkg/src/sphwav).  The reference exposes this path only as
 * Python functions; every entry point below replaces one of them and keeps its
 * argument meaning, layout and error behaviour:
 *
 *   s2w_grid_nodes            <- grid.py:112-131   (_cached_grid / make_grid)
 *   s2w_assoc_legendre_ring   <- sht.py:190-206    (assoc_legendre_ring)
 *   s2w_sh_synthesis          <- sht.py:222-290    (sh_synthesis_stack / sh_synthesis)
 *   s2w_sh_analysis           <- sht.py:293-355    (sh_analysis_stack / sh_analysis;
 *                                                   additionally supports MW grids)
 *   s2w_wav_analysis_harmonic <- transform.py:129-150 (wav_analysis_harmonic)
 *   s2w_wav_synthesis_harmonic<- transform.py:153-172 (wav_synthesis_harmonic)
 *   s2w_wav_analysis_pixel    <- transform.py:175-191 (wav_analysis_pixel)
 *   s2w_wav_synthesis_pixel   <- transform.py:194-202 (wav_synthesis_pixel)
 *   s2w_s2wm_read_header, s2w_s2wm_read_payload, s2w_s2wm_write
 *                             <- mapio.py:83-168 (write_map/read_map/write_flm/read_flm)
 *   s2w_wav_analysis_pixel_threshold, s2w_wav_denoise_pixel
 *                             <- denoise.py:78-103 (hard_threshold / denoise_pipeline),
 *                                threshold fused into the scale maps' ring-DFT epilogue
 *
 * Conventions ("contiguous 64-bit float buffers plus scalar
 * parameters; no object graphs cross the boundary"):
 *   - harmonic coefficients: complex128 interleaved (re, im) doubles, flat index
 *     l*l + l + m (sht.py:50-52), L*L entries per set; sets are contiguous;
 *   - maps: theta-major rows (grid.py:143), n_theta = L rings of n_phi = 2L-1
 *     samples; complex maps are interleaved (re, im) doubles, real maps
 *     (is_real = 1) are plain doubles (the imaginary part is exactly zero by
 *     construction, grid.py:160);
 *   - all data pointers are DEVICE pointers (CUDA global memory) except where a
 *     parameter says "host"; `stream` is a cudaStream_t (NULL = legacy default);
 *   - every call is asynchronous on `stream` and returns a status code; a plan is
 *     used by one host thread at a time; distinct plans are independent.
 *
 * Status codes map onto the reference's exception hierarchy (errors.py:4-13):
 *   S2W_EPARAM -> ParameterError, everything else -> SphwavError/RuntimeError.
 */
#ifndef S2W_H
#define S2W_H

#ifdef __cplusplus
extern "C" {
#endif

#define S2W_OK 0
#define S2W_EPARAM 1    /* domain violation: ParameterError (errors.py:8)       */
#define S2W_ECUDA 2     /* CUDA runtime failure                                 */
#define S2W_ENOMEM 3    /* device allocation failure                            */
#define S2W_EINTERNAL 4 /* invariant broken inside the library                  */
/* S2WM files (mapio.py:48-63): FormatError subclasses, and OSError */
#define S2W_EFORMAT_MAGIC 5     /* NotS2wmFileError        */
#define S2W_EFORMAT_VERSION 6   /* UnsupportedVersionError */
#define S2W_EFORMAT_TRUNCATED 7 /* TruncatedFileError      */
#define S2W_EFORMAT_PAYLOAD 8   /* PayloadMismatchError    */
#define S2W_EIO 9               /* OSError                 */

#define S2W_SCHEME_GL 0 /* SamplingScheme.GL (grid.py:33-35)                   */
#define S2W_SCHEME_MW 1 /* SamplingScheme.MW                                   */

typedef struct s2w_sht_plan s2w_sht_plan;
typedef struct s2w_wav_plan s2w_wav_plan;

/* Library version string ("s2w-b200 x.y.z"). */
const char* s2w_version(void);
/* Message of the last failing call on this host thread ("" if none). */
const char* s2w_last_error(void);

/* Host-only: ring colatitudes theta[L] and, for GL, the Gauss-Legendre weights
 * over cos(theta) (weights may be NULL; for MW they are not defined and the
 * array is left untouched).  grid.py:93-124.  No GPU needed. */
int s2w_grid_nodes(int scheme, int L, double* theta, double* weights);

/* table[l*L + m] = orthonormal P_lm(cos theta) for 0 <= m <= l < L, zero above
 * the diagonal (sht.py:190-206, without the reference's 1e-280 flush).
 * `table` is a device buffer of L*L doubles. */
int s2w_assoc_legendre_ring(int L, double theta, double* table, void* stream);

/* ---------------------------------------------------------------- SHT */
/* Plan for spherical harmonic transforms on one grid (scheme, L) of `device`. */
int s2w_sht_plan_create(int scheme, int L, int device, s2w_sht_plan** plan);
int s2w_sht_plan_destroy(s2w_sht_plan* plan);

/* map[s] = synthesis of flm[s] (band L_coef <= plan L, zero-padded above it)
 * for s < n_sets.  is_real: coefficient sets carry the real-signal symmetry;
 * the output map is then real (n_sets*L*(2L-1) doubles).  MW: the south-pole
 * ring is pinned to its m = 0 value (sht.py:274-279). */
int s2w_sh_synthesis(s2w_sht_plan* plan, int n_sets, int L_coef, int is_real,
                     const double* flm, double* map, void* stream);

/* flm[s] (n_sets*L*L complex) = exact analysis of map[s].  GL: Gauss-Legendre
 * quadrature (sht.py:308-346).  MW: McEwen-Wiaux sampling theorem (theta
 * extension + |sin| convolution), which the reference lacks (sht.py:300-303).
 * is_real: map is real; negative orders are written as (-1)^m conj(f_lm)
 * exactly (sht.py:328-331). */
int s2w_sh_analysis(s2w_sht_plan* plan, int n_sets, int is_real, const double* map,
                    double* flm, void* stream);

/* ---------------------------------------------------------------- wavelets */
/* Plan for the axisymmetric wavelet transform of `batch` maps at band L.
 *   n_kern   = 1 + number of wavelet scales (scaling kernel first, then j0..J)
 *   kernels  = HOST array [n_kern][L]: Phi_l0 then Psi^j_l0 (tiling.py:219-245)
 *   bands    = HOST array [n_kern]: band limit of each coefficient map
 *              (multires: scaling_bandlimit, scale_bandlimits; full-res: all L;
 *               transform.py:108-114)
 * The plan precomputes sqrt(4 pi/(2l+1)) * K_j(l) (transform.py:117-126). */
int s2w_wav_plan_create(int scheme, int L, int batch, int is_real, int n_kern,
                        const double* kernels, const int* bands, int device,
                        s2w_wav_plan** plan);
int s2w_wav_plan_destroy(s2w_wav_plan* plan);

/* Harmonic tiling.  outs[j] receives batch sets of band_j^2 coefficients
 * (truncate != 0) or L^2 coefficients (truncate == 0). */
int s2w_wav_analysis_harmonic(s2w_wav_plan* plan, int truncate, const double* flm,
                              double* const* outs, void* stream);
/* flm (batch*L*L) = sum_j sqrt(4pi/(2l+1)) K_j(l) pad(ins[j]); ins[j] has
 * band_j^2 (or L^2 when full_band != 0) coefficients per set. */
int s2w_wav_synthesis_harmonic(s2w_wav_plan* plan, int full_band, const double* const* ins,
                               double* flm, void* stream);

/* map (batch maps at L) -> scale_maps[j] (batch maps at band_j), j < n_kern. */
int s2w_wav_analysis_pixel(s2w_wav_plan* plan, const double* map, double* const* scale_maps,
                           void* stream);
/* scale_maps[j] -> map (exact inverse of s2w_wav_analysis_pixel). */
int s2w_wav_synthesis_pixel(s2w_wav_plan* plan, const double* const* scale_maps, double* map,
                            void* stream);

/* Wavelet analysis with the denoiser's hard threshold fused in (denoise.py:78-96):
 * samples of wavelet map j (1 <= j < n_kern) with |value| < thresholds[j] are
 * zeroed as they are written; the scaling map (j = 0, thresholds[0] ignored)
 * passes unchanged.  thresholds: HOST array of n_kern doubles, each >= 0. */
int s2w_wav_analysis_pixel_threshold(s2w_wav_plan* plan, const double* map,
                                     const double* thresholds, double* const* scale_maps,
                                     void* stream);
/* denoise_pipeline (denoise.py:99-103): thresholded analysis into the caller's
 * scale_maps workspace, then wavelet synthesis into map_out. */
int s2w_wav_denoise_pixel(s2w_wav_plan* plan, const double* map, const double* thresholds,
                          double* const* scale_maps, double* map_out, void* stream);

/* Coefficient workspace of the plan (batch*L*L complex, device): after
 * s2w_wav_analysis_pixel it holds f_lm of the input map; after
 * s2w_wav_synthesis_pixel the recombined f_lm (transform.py:196-200). */
int s2w_wav_plan_flm(s2w_wav_plan* plan, double** flm);

/* Per-scale ring stages (phi and theta of each scale map) run concurrently on
 * plan-owned side streams forked from and joined back into the caller's
 * stream (default, on != 0), or in order on the caller's stream (on == 0:
 * serial per-stage profiling).  Results are bit-identical either way. */
int s2w_wav_plan_set_concurrency(s2w_wav_plan* plan, int on);

/* ---------------------------------------------------------------- S2WM files (mapio.py) */
/* 22-byte little-endian header (mapio.py:1-15): magic, version, scheme, L, kind, count.
 * Validates length, magic and version (mapio.py:110-119); the caller checks kind,
 * scheme, L and count against what it expects (mapio.py:133-145, 163-168). */
int s2w_s2wm_read_header(const char* path, int* scheme, int* L, int* kind, long long* count);
/* Payload of `count` float64 (or (re, im) pairs when complex_payload) into dst
 * (device memory when dst_device, through pinned double-buffered staging on
 * `stream`, complete on return; else host).  S2W_EFORMAT_TRUNCATED when the file
 * holds a different number of bytes (mapio.py:122-130). */
int s2w_s2wm_read_payload(const char* path, long long count, int complex_payload, void* dst,
                          int dst_device, void* stream);
/* Header + payload from src (device or host); byte-identical for equal input
 * (mapio.py:83-106).  kind: 0 real map, 1 complex map, 2 coefficients. */
int s2w_s2wm_write(const char* path, int scheme, int L, int kind, long long count,
                   int complex_payload, const void* src, int src_device, void* stream);

/* ---------------------------------------------------------------- shards (multi-GPU) */
/* One grid restricted to a rank's share of the work: the orders m in `orders`
 * (Legendre and theta stages) and the ring block [t0, t1) (ring FFT stages).
 * The exchange between the two (an all-to-all of per-ring Fourier modes) is
 * the caller's (torch.distributed / NCCL); paper_1211_1680_b200/distributed.py
 * drives it.  Layouts (B = batch, n_local = number of my bins: per listed order
 * m, bin m then, for complex data and m > 0, bin 2L-1-m):
 *   map rows [B][t1-t0][2L-1]  G_col [B][n_bins][t1-t0]  G_ring [B][t1-t0][n_bins]
 *   G_local [B][L][n_local]    H_local [B][n_local][L]
 * weights: optional HOST table [n_w][L] of per-degree factors (tiling). */
typedef struct s2w_shard_plan s2w_shard_plan;
int s2w_shard_plan_create(int scheme, int L, int batch, int is_real, int n_orders,
                          const int* orders, int t0, int t1, int n_w, const double* weights,
                          int device, s2w_shard_plan** plan);
int s2w_shard_plan_destroy(s2w_shard_plan* plan);
/* Number (and list, if bins != NULL) of my bins, in local order. */
int s2w_shard_bins(s2w_shard_plan* plan, int* n_bins, int* bins);
/* map rows -> G_col = DFT_phi / N (all bins, my rings). */
int s2w_shard_rings_forward(s2w_shard_plan* plan, const double* map_rows, double* G, void* stream);
/* G_ring -> map rows (my rings; MW pole ring pinned if it is mine). */
int s2w_shard_rings_inverse(s2w_shard_plan* plan, const double* G, double* map_rows, void* stream);
/* H_local in place: MW theta stage for my bins (no-op on GL grids). */
int s2w_shard_theta(s2w_shard_plan* plan, double* H, void* stream);
/* flm [B][flm_L^2] (x weight row w_index, -1 = none) -> G_local for my orders. */
int s2w_shard_legendre_synthesis(s2w_shard_plan* plan, const double* flm, int flm_L, int w_index,
                                 double* G, void* stream);
/* H_local -> flm [B][flm_L^2] at my orders (x weight row w_index); accumulate != 0
 * adds into flm, otherwise flm is zeroed first. */
int s2w_shard_legendre_analysis(s2w_shard_plan* plan, const double* H, double* flm, int flm_L,
                                int w_index, int accumulate, void* stream);

/* Several weighted sets of one grid in one launch (the scales that share
 * it): synthesis writes G[s] from weight row w_index[s]; analysis folds
 * sum_s w[s] x analysis(H[s]) into flm in set order.  n <= 3. */
int s2w_shard_legendre_synthesis_sets(s2w_shard_plan* plan, const double* flm, int flm_L, int n,
                                      const int* w_index, double* const* G, void* stream);
int s2w_shard_legendre_analysis_sets(s2w_shard_plan* plan, int n, const double* const* H,
                                     const int* w_index, double* flm, int flm_L, int accumulate,
                                     void* stream);
/* Exchange layout: the P ranks' ring blocks (ring_t0t1[2q], [2q+1], tiling
 * [0, L) in rank order) and bin lists (n_bins[q] entries each, concatenated in
 * rank order; `rank`'s must equal this plan's).  Afterwards rings_forward
 * writes G_col grouped by destination: for q in rank order, [B][n_q][t1-t0]
 * (one contiguous block per destination, sent as is).  Replaces the
 * all-to-all packing of distributed.py (round 1). */
int s2w_shard_set_peers(s2w_shard_plan* plan, int P, int rank, const int* ring_t0t1,
                        const int* n_bins, const int* bins);
/* Fused exchange over peer memory (NVLink / CUDA IPC pointers, HOST array of P
 * device pointers, peer_*[q] = rank q's buffer).  rings_forward_peers: the
 * forward ring DFTs of my rings store each bin row straight into its owner's
 * H_local [B][n_q][L] (my ring columns), no send buffer and no gather.
 * push_rings: my G_local [B][L][n_local] (Legendre synthesis output) is
 * stored straight into every ring owner's G_ring [B][t_q][n_bins].  The
 * caller orders them against the peers' readers (a barrier before and after). */
int s2w_shard_rings_forward_peers(s2w_shard_plan* plan, const double* map_rows,
                                  double* const* peer_H, void* stream);
int s2w_shard_push_rings(s2w_shard_plan* plan, const double* G, double* const* peer_G, void* stream);
/* Received blocks [B][n_local][t_q] (src[q], device pointers, HOST array of P)
 * -> H_local [B][n_local][L]. */
int s2w_shard_gather_rings(s2w_shard_plan* plan, const double* const* src, double* H, void* stream);
/* Received blocks [B][t1-t0][n_q] of rank q's bins -> G_ring [B][t1-t0][n_bins]. */
int s2w_shard_scatter_bins(s2w_shard_plan* plan, const double* const* src, double* G, void* stream);

/* ---------------------------------------------------------------- layouts */
/* n real doubles -> n complex128 (zero imaginary parts), and back (real parts):
 * the numpy drop-in's real maps are complex128 arrays (reference grid.py:155-160). */
int s2w_real_to_complex(const double* in, double* out, long long n, void* stream);
int s2w_complex_real_part(const double* in, double* out, long long n, void* stream);

/* ---------------------------------------------------------------- accounting */
/* Number of kernels launched by this library since load (bench "gpu_launches"). */
long long s2w_kernel_launches(void);
/* Per-stage CUDA-event timing of every launch (off by default). */
int s2w_profile_enable(int on);
/* ms[i], count[i] for stage i < n in the order of s2w_profile_stage_name(i);
 * synchronises on the recorded events; reset != 0 clears the accumulators. */
int s2w_profile_read(int n, double* ms, long long* count, int reset);
const char* s2w_profile_stage_name(int i);
/* Measured FP64 FMA throughput of the current device in TFLOP/s (synchronous). */
int s2w_fp64_peak(double* tflops, void* stream);
/* Measured FP64 tensor-core (DMMA m8n8k4) throughput in TFLOP/s (synchronous). */
int s2w_dmma_peak(double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* S2W_H */
