// Exchange-side layout kernels of the sharded transform (capi_shard.inc).
//
// The forward ring DFTs of a shard plan already write every destination
// rank's bins as one contiguous block (PhiFwdArgs::ofs), and the Legendre
// synthesis writes ring-major rows whose ring blocks are contiguous, so the
// send side needs no packing.  What arrives from the P ranks is one block per
// source; these kernels place the blocks where the next stage reads them:
//   gather_rings: blocks [B][n_local][t_q] from each source q -> H_local
//                 [B][n_local][L] (ring t of H at block q(t), offset t - t0_q);
//   scatter_bins: blocks [B][t_r][n_q] of the source's bins -> G_ring
//                 [B][t_r][n_bins] (bin b at block q(b), index i(b)).
// Both are one pass of HBM traffic (read + write of the received bytes),
// coalesced on the write side; the sources are read through a table of P
// device pointers (a rank's own block is read straight from its send buffer).
#include <algorithm>
#include "common.cuh"
#include "s2w_internal.h"

namespace s2w {

__global__ void shard_gather_rings_kernel(ShardSrc src, const int2* ring_src, const int* t_len,
                                          int B, int n_local, int L, double2* H) {
  const long long total = (long long)B * n_local * L;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(e % L);
    const long long row = e / L;  // b * n_local + i
    const int2 qs = __ldg(&ring_src[t]);
    const double2* s = src.p[qs.x];
    H[e] = __ldg(&s[row * __ldg(&t_len[qs.x]) + qs.y]);
  }
}

__global__ void shard_scatter_bins_kernel(ShardSrc src, const int2* bin_src, const int* n_src,
                                          int B, int t_r, int n_bins, double2* G) {
  const long long total = (long long)B * t_r * n_bins;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int bin = (int)(e % n_bins);
    const long long row = e / n_bins;  // b * t_r + t
    const int2 qi = __ldg(&bin_src[bin]);
    const double2* s = src.p[qi.x];
    G[e] = __ldg(&s[row * __ldg(&n_src[qi.x]) + qi.y]);
  }
}

static int grid_for(long long n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long want = (n + 255) / 256;
  return (int)std::min<long long>(want, 8LL * sms);
}

cudaError_t launch_shard_gather_rings(const ShardSrc& src, const int2* ring_src, const int* t_len,
                                      int B, int n_local, int L, double2* H, cudaStream_t st) {
  const long long n = (long long)B * n_local * L;
  if (n == 0) return cudaSuccess;
  shard_gather_rings_kernel<<<grid_for(n), 256, 0, st>>>(src, ring_src, t_len, B, n_local, L, H);
  return cudaGetLastError();
}

cudaError_t launch_shard_scatter_bins(const ShardSrc& src, const int2* bin_src, const int* n_src,
                                      int B, int t_r, int n_bins, double2* G, cudaStream_t st) {
  const long long n = (long long)B * t_r * n_bins;
  if (n == 0) return cudaSuccess;
  shard_scatter_bins_kernel<<<grid_for(n), 256, 0, st>>>(src, bin_src, n_src, B, t_r, n_bins, G);
  return cudaGetLastError();
}

// Fused synthesis-direction exchange: each element of my G_local goes
// straight to the owner of its ring, into that rank's G_ring row (a store over
// NVLink when the owner is another GPU).  Reads coalesced along my bins.
__global__ void shard_push_rings_kernel(const double2* G, ShardDst dst, const int2* ring_src,
                                        const int* t_len, const int* bins, int B, int k, int nl,
                                        int nb) {
  const long long total = (long long)B * k * nl;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nl);
    const long long bt = e / nl;  // b * k + t
    const int t = (int)(bt % k), b = (int)(bt / k);
    const int2 qs = __ldg(&ring_src[t]);
    dst.p[qs.x][((long long)b * __ldg(&t_len[qs.x]) + qs.y) * nb + __ldg(&bins[i])] = G[e];
  }
}

cudaError_t launch_shard_push_rings(const double2* G, const ShardDst& dst, const int2* ring_src,
                                    const int* t_len, const int* bins, int B, int k, int n_local,
                                    int n_bins, cudaStream_t st) {
  const long long n = (long long)B * k * n_local;
  if (n == 0) return cudaSuccess;
  shard_push_rings_kernel<<<grid_for(n), 256, 0, st>>>(G, dst, ring_src, t_len, bins, B, k, n_local,
                                                        n_bins);
  return cudaGetLastError();
}

}  // namespace s2w
