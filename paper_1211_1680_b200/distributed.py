"""Multi-GPU wavelet transform of one large map.

Partition (one process per GPU, torch.distributed over NCCL):

* the Legendre and MW theta stages are split **by order m**: every rank owns
  a fixed, load-balanced set of orders (snake assignment by decreasing cost
  (L - m)), the same set for every scale grid, so the harmonic tiling between
  the SHTs of a wavelet transform is rank-local;
* the ring FFT stages are split **by ring**: every rank owns a contiguous
  block of rings of each grid (its slice of the input / output maps);
* between the two, one all-to-all per grid moves the per-ring Fourier modes
  G_m(theta_t): analysis ring-block x all-orders -> all-rings x my-orders;
  synthesis the reverse.  Message size per SHT is k (2k-1) 16 B in total
  (134 MB for C4's L = 2048), i.e. ~20 us over NVLink 5 against milliseconds
  of FP64 work.

All arithmetic runs in libs2w.so (C ABI ``s2w_shard_*``); this module only
builds the partition, packs / unpacks exchange buffers with torch indexing
and calls the exchanger.  Two exchangers exist: ``TorchExchange``
(torch.distributed ``all_to_all_single``; NCCL on GPUs, gloo on CPU) and
``VirtualExchange`` (several ranks in one process, for single-GPU testing:
ranks run stage by stage and never wait on one another).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _device, _native
from .errors import ParameterError
from .grid import SamplingScheme, scheme_code
from .transform import TransformConfig, kernels_for, scale_bands

__all__ = [
    "order_owner",
    "ring_blocks",
    "shard_bins",
    "TorchExchange",
    "VirtualExchange",
    "ShardedWaveletTransform",
]


# ---------------------------------------------------------------- partition (pure host logic)
def order_owner(L: int, P: int) -> np.ndarray:
    """owner[m] for m < L: snake assignment of orders sorted by cost (L - m)."""
    if P < 1:
        raise ParameterError("world size must be >= 1")
    owner = np.empty(L, dtype=np.int64)
    for i, m in enumerate(range(L)):  # cost decreases with m: already sorted
        rnd, pos = divmod(i, P)
        owner[m] = pos if rnd % 2 == 0 else P - 1 - pos
    return owner


def ring_blocks(k: int, P: int) -> list[tuple[int, int]]:
    """Contiguous, near-equal ring blocks [t0, t1) of a k-ring grid."""
    base, extra = divmod(k, P)
    out, t = [], 0
    for r in range(P):
        n = base + (1 if r < extra else 0)
        out.append((t, t + n))
        t += n
    return out


def shard_bins(k: int, orders, real: bool) -> np.ndarray:
    """Local bin list of an order set: m, then 2k-1-m (complex, m > 0)."""
    N = 2 * k - 1
    bins = []
    for m in orders:
        bins.append(m)
        if not real and m > 0:
            bins.append(N - m)
    return np.asarray(bins, dtype=np.int64)


# ---------------------------------------------------------------- exchangers
class TorchExchange:
    """all-to-all through torch.distributed (one rank per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.P = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def all_to_all(self, sends: dict, recv_sizes: dict) -> dict:
        """sends[rank][dst] -> tensors; recv_sizes[rank][src] element counts
        (known from the partition); returns recvs[rank][src] (flat)."""
        th = _device.torch()
        (me,) = self.ranks
        out = sends[me]
        cplx = out[0].is_complex()
        # complex payloads travel as interleaved float64 (NCCL / gloo have no complex type)
        flat = [th.view_as_real(t).reshape(-1) if cplx else t.reshape(-1) for t in out]
        w = 2 if cplx else 1
        in_splits = [int(t.numel()) for t in flat]
        send = th.cat(flat)
        out_splits = [w * int(x) for x in recv_sizes[me]]
        recv = th.empty(sum(out_splits), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)
        parts = th.split(recv, out_splits)
        if cplx:
            parts = [th.view_as_complex(p.view(-1, 2)) for p in parts]
        return {me: list(parts)}


class VirtualExchange:
    """P ranks in one process (single-GPU testing): delivery by reference."""

    def __init__(self, P: int):
        self.P = P
        self.ranks = list(range(P))

    def all_to_all(self, sends: dict, recv_sizes: dict = None) -> dict:
        return {r: [sends[q][r].reshape(-1) for q in range(self.P)] for r in self.ranks}


# ---------------------------------------------------------------- GPU backend
class _GpuShard:
    """C-ABI shard plan of one grid for one rank."""

    def __init__(self, scheme, k, batch, real, orders, t0, t1, weights):
        lib = _native.load()
        orders = np.ascontiguousarray(orders, dtype=np.int32)
        oc = orders.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) if orders.size else None
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        wp = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if w is not None else None
        h = ctypes.c_void_p()
        _native.check(lib.s2w_shard_plan_create(
            scheme_code(scheme), k, batch, int(real), int(orders.size), oc, t0, t1,
            0 if w is None else w.shape[0], wp, _device.device_index(), ctypes.byref(h)))
        self.h, self.lib = h, lib

    def __del__(self):
        try:
            self.lib.s2w_shard_plan_destroy(self.h)
        except Exception:
            pass

    def call(self, name, *args):
        _native.check(getattr(self.lib, name)(self.h, *args))


@dataclass
class _Grid:
    k: int
    blocks: list            # ring block per rank
    orders: list            # np.ndarray of orders per rank
    bins: list              # local bins per rank
    plans: dict             # rank -> _GpuShard (unweighted)
    wplans: dict            # (rank, scale j) -> _GpuShard with weight row 0 = fac_j


class ShardedWaveletTransform:
    """Wavelet analysis / synthesis of one map sharded over P ranks.

    Inputs and outputs are the rank-local ring blocks of the maps:
    ``analysis({rank: x_rows})`` with x_rows of shape (batch, t1 - t0, 2L-1)
    returns ``{rank: [rows of scale map j]}``; ``synthesis`` is the inverse.
    """

    def __init__(self, config: TransformConfig, exchange, batch: int = 1, real: bool = False):
        _device.require_cuda()
        self.cfg, self.ex, self.B, self.real = config, exchange, batch, bool(real)
        self.P = exchange.P
        kern = kernels_for(config)
        self.bands = scale_bands(config, kern)
        L = config.L
        ell = np.arange(L, dtype=np.float64)
        self.fac = np.sqrt(4.0 * np.pi / (2.0 * ell + 1.0))[None, :] * kern.table()
        owner = order_owner(L, self.P)
        self.owner = owner
        self.grids = {}
        for k in sorted(set([L, *self.bands])):
            blocks = ring_blocks(k, self.P)
            orders = [np.nonzero(owner[:k] == r)[0] for r in range(self.P)]
            bins = [shard_bins(k, o, self.real) for o in orders]
            self.grids[k] = _Grid(k, blocks, orders, bins, {}, {})
            for r in exchange.ranks:
                t0, t1 = blocks[r]
                self.grids[k].plans[r] = _GpuShard(config.scheme, k, batch, real, orders[r], t0, t1,
                                                    None)
        for j, k in enumerate(self.bands):
            g = self.grids[k]
            for r in exchange.ranks:
                t0, t1 = g.blocks[r]
                g.wplans[(r, j)] = _GpuShard(config.scheme, k, batch, real, g.orders[r], t0, t1,
                                             self.fac[j:j + 1, :k])
        th = _device.torch()
        self.dev = f"cuda:{_device.device_index()}"
        self._bins_t = {k: [th.as_tensor(b, device=self.dev) for b in g.bins]
                        for k, g in self.grids.items()}
        self.f = {r: th.zeros((batch, L * L), dtype=th.complex128, device=self.dev)
                  for r in exchange.ranks}

    # -- helpers
    def _nb(self, k):
        return k if self.real else 2 * k - 1

    def _stream(self):
        return _device.stream_handle()

    def _cols_to_local(self, k, gcol: dict) -> dict:
        """G_col[r] (B, n_bins, t_r) -> H_local[r] (B, n_local_r, k) via all-to-all."""
        th = _device.torch()
        g = self.grids[k]
        sends = {r: [gcol[r][:, self._bins_t[k][q], :].contiguous() for q in range(self.P)]
                 for r in self.ex.ranks}
        sizes = {r: [self.B * len(g.bins[r]) * (g.blocks[q][1] - g.blocks[q][0])
                     for q in range(self.P)] for r in self.ex.ranks}
        recv = self.ex.all_to_all(sends, sizes)
        out = {}
        for r in self.ex.ranks:
            nl = len(g.bins[r])
            parts = [recv[r][q].view(self.B, nl, g.blocks[q][1] - g.blocks[q][0])
                     for q in range(self.P)]
            out[r] = th.cat(parts, dim=2).contiguous()
        return out

    def _local_to_rings(self, k, glocal: dict) -> dict:
        """G_local[r] (B, k, n_local_r) -> G_ring[r] (B, t_r, n_bins) via all-to-all."""
        th = _device.torch()
        g = self.grids[k]
        sends = {r: [glocal[r][:, g.blocks[q][0]:g.blocks[q][1], :].contiguous()
                     for q in range(self.P)] for r in self.ex.ranks}
        sizes = {r: [self.B * (g.blocks[r][1] - g.blocks[r][0]) * len(g.bins[q])
                     for q in range(self.P)] for r in self.ex.ranks}
        recv = self.ex.all_to_all(sends, sizes)
        out = {}
        for r in self.ex.ranks:
            t = g.blocks[r][1] - g.blocks[r][0]
            ring = th.zeros((self.B, t, self._nb(k)), dtype=th.complex128, device=self.dev)
            for q in range(self.P):
                nl = len(g.bins[q])
                if nl:
                    ring[:, :, self._bins_t[k][q]] = recv[r][q].view(self.B, t, nl)
            out[r] = ring
        return out

    def _forward(self, k, rows: dict) -> dict:
        """map rows -> H_local (theta stage applied on MW)."""
        th = _device.torch()
        g = self.grids[k]
        gcol = {}
        for r in self.ex.ranks:
            t = g.blocks[r][1] - g.blocks[r][0]
            gc = th.empty((self.B, self._nb(k), t), dtype=th.complex128, device=self.dev)
            g.plans[r].call("s2w_shard_rings_forward", _device.ptr(rows[r]), _device.ptr(gc),
                            self._stream())
            gcol[r] = gc
        H = self._cols_to_local(k, gcol)
        for r in self.ex.ranks:
            if len(g.bins[r]):
                g.plans[r].call("s2w_shard_theta", _device.ptr(H[r]), self._stream())
        return H

    def _inverse(self, k, glocal: dict) -> dict:
        th = _device.torch()
        g = self.grids[k]
        ring = self._local_to_rings(k, glocal)
        out = {}
        for r in self.ex.ranks:
            t = g.blocks[r][1] - g.blocks[r][0]
            x = th.empty((self.B, t, 2 * k - 1), dtype=th.float64 if self.real else th.complex128,
                         device=self.dev)
            g.plans[r].call("s2w_shard_rings_inverse", _device.ptr(ring[r]), _device.ptr(x),
                            self._stream())
            out[r] = x
        return out

    # -- public
    def analysis(self, x_rows: dict) -> dict:
        th = _device.torch()
        L = self.cfg.L
        H = self._forward(L, x_rows)
        top = self.grids[L]
        for r in self.ex.ranks:
            top.plans[r].call("s2w_shard_legendre_analysis", _device.ptr(H[r]),
                              _device.ptr(self.f[r]), L, -1, 0, self._stream())
        out = {r: [] for r in self.ex.ranks}
        for j, k in enumerate(self.bands):
            g = self.grids[k]
            gl = {}
            for r in self.ex.ranks:
                G = th.empty((self.B, k, len(g.bins[r])), dtype=th.complex128, device=self.dev)
                if len(g.bins[r]):
                    g.wplans[(r, j)].call("s2w_shard_legendre_synthesis", _device.ptr(self.f[r]),
                                          L, 0, _device.ptr(G), self._stream())
                gl[r] = G
            maps = self._inverse(k, gl)
            for r in self.ex.ranks:
                out[r].append(maps[r])
        return out

    def synthesis(self, scale_rows: dict) -> dict:
        th = _device.torch()
        L = self.cfg.L
        for j, k in enumerate(self.bands):
            g = self.grids[k]
            H = self._forward(k, {r: scale_rows[r][j] for r in self.ex.ranks})
            for r in self.ex.ranks:
                g.wplans[(r, j)].call("s2w_shard_legendre_analysis", _device.ptr(H[r]),
                                      _device.ptr(self.f[r]), L, 0, int(j > 0), self._stream())
        top = self.grids[L]
        gl = {}
        for r in self.ex.ranks:
            G = th.empty((self.B, L, len(top.bins[r])), dtype=th.complex128, device=self.dev)
            if len(top.bins[r]):
                top.plans[r].call("s2w_shard_legendre_synthesis", _device.ptr(self.f[r]), L, -1,
                                  _device.ptr(G), self._stream())
            gl[r] = G
        return self._inverse(L, gl)

    def round_trip(self, x_rows: dict) -> dict:
        return self.synthesis(self.analysis(x_rows))

    def ring_block(self, k: int, rank: int) -> tuple[int, int]:
        return self.grids[k].blocks[rank]
