"""Multi-GPU wavelet transform of one large map.

Partition (one process per GPU, torch.distributed over NCCL):

* the Legendre and MW theta stages are split **by order m**: every rank owns
  a fixed, load-balanced set of orders (snake assignment by decreasing cost
  (L - m)), the same set for every scale grid, so the harmonic tiling between
  the SHTs of a wavelet transform is rank-local;
* the ring FFT stages are split **by ring**: every rank owns a contiguous
  block of rings of each grid (its slice of the input / output maps);
* between the two, an all-to-all exchange of the per-ring Fourier modes
  G_m(theta_t): analysis ring-block x all-orders -> all-rings x my-orders;
  synthesis the reverse.  Message size per SHT is k (2k-1) 16 B in total
  (134 MB for C4's L = 2048), i.e. ~20 us over NVLink 5 against milliseconds
  of FP64 work (DESIGN.md section 7 tabulates the bytes per rank).

Small scales are not sharded: a scale whose band is at most ``whole_max``
(256) runs whole on one rank (owners dealt by cost, largest first), on the
low-degree block of f_lm that one all-reduce (B k_s^2 16 B, k_s the largest
such band: 1 MB at C4) makes complete on every rank.  Their maps live whole on
the owner; the synthesis folds them back with a second all-reduce.  The large
scales and the map itself are order/ring sharded, and all large scales of a
direction share ONE grouped exchange (per destination, one message per
scale, in a single NCCL group): per round trip 4 exchanges + 2 small
all-reduces, whatever the number of scales.

All arithmetic runs in libs2w.so (C ABI ``s2w_shard_*``).  No packing: the
forward ring DFTs write each destination's bins as one contiguous block
(``s2w_shard_set_peers``), the Legendre synthesis writes ring-major rows whose
ring blocks are contiguous, and the receive side places the blocks with
``s2w_shard_gather_rings`` / ``s2w_shard_scatter_bins`` (a rank's own block is
read straight from its send buffer).  Exchangers: ``TorchExchange``
(torch.distributed grouped P2P, ``batch_isend_irecv``: NCCL on GPUs, gloo on
CPU) and ``VirtualExchange`` (several ranks in one process, for single-GPU
testing: delivery by reference, ranks never wait on one another).
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
    "TorchPeerExchange",
    "VirtualPeerExchange",
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
    """Grouped point-to-point exchange through torch.distributed (one rank per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.P = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def exchange(self, sends: dict, recv_shapes: dict) -> dict:
        """sends[rank][key][dst] -> contiguous tensor for dst (None: nothing);
        recv_shapes[rank][key][src] -> shape of what src sends (None: nothing).
        Returns got[rank][key][src]: the received tensor (a rank's own block is
        its send tensor, not copied).  All messages of the call form one group
        (one NCCL launch); messages between a pair match in key order."""
        th = _device.torch()
        (me,) = self.ranks
        ops, got = [], {}
        for key in sorted(sends[me]):
            out, shapes = sends[me][key], recv_shapes[me][key]
            row = []
            for q in range(self.P):
                if q == me:
                    row.append(out[q])
                    continue
                if out[q] is not None and out[q].numel():
                    ops.append(self.dist.P2POp(self.dist.isend, _real_view(out[q]), q, self.group))
                rb = None
                if shapes[q] is not None and math.prod(shapes[q]):
                    rb = th.empty(shapes[q], dtype=out_dtype(sends[me][key]), device=_dev_of(sends[me][key]))
                    ops.append(self.dist.P2POp(self.dist.irecv, _real_view(rb), q, self.group))
                row.append(rb)
            got[key] = row
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return {me: got}

    def all_reduce(self, bufs: dict) -> None:
        """In-place sum over ranks."""
        (me,) = self.ranks
        t = bufs[me]
        if t.numel():
            self.dist.all_reduce(_real_view(t), group=self.group)

    def all_to_all(self, sends: dict, recv_sizes: dict) -> dict:
        """Flat all-to-all (sends[rank][dst] -> tensors; recv_sizes[rank][src]
        element counts); returns recvs[rank][src] (flat).  Kept for callers
        that exchange host-computed blocks."""
        th = _device.torch()
        (me,) = self.ranks
        out = sends[me]
        cplx = out[0].is_complex()
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


def _real_view(t):
    """NCCL / gloo have no complex type: complex payloads travel as float64 pairs."""
    th = _device.torch()
    return th.view_as_real(t) if t.is_complex() else t


def out_dtype(row):
    for t in row:
        if t is not None:
            return t.dtype
    raise ParameterError("exchange row without any tensor")


def _dev_of(row):
    for t in row:
        if t is not None:
            return t.device
    raise ParameterError("exchange row without any tensor")


class VirtualExchange:
    """P ranks in one process (single-GPU testing): delivery by reference."""

    def __init__(self, P: int):
        self.P = P
        self.ranks = list(range(P))

    def exchange(self, sends: dict, recv_shapes: dict = None) -> dict:
        return {r: {key: [sends[q][key][r] for q in range(self.P)] for key in sends[r]}
                for r in self.ranks}

    def all_reduce(self, bufs: dict) -> None:
        total = None
        for r in self.ranks:
            total = bufs[r].clone() if total is None else total + bufs[r]
        for r in self.ranks:
            bufs[r].copy_(total)

    def all_to_all(self, sends: dict, recv_sizes: dict = None) -> dict:
        return {r: [sends[q][r].reshape(-1) for q in range(self.P)] for r in self.ranks}


class VirtualPeerExchange(VirtualExchange):
    """Fused exchange over peer memory, P virtual ranks in one process: every
    rank's receive buffers are plain device tensors, and a rank's kernels store
    straight into the other ranks' buffers (on one GPU the "peer" pointers are
    local; the same kernels take NVLink pointers across GPUs)."""

    peer = True

    def __init__(self, P: int):
        super().__init__(P)
        self._bufs = {}

    def alloc_shared(self, key, shapes: dict, dtype):
        """{rank: tensor} receive buffers (persistent per key) and, per writing
        rank, the table of every rank's buffer pointer."""
        th = _device.torch()
        if key not in self._bufs:
            dev = f"cuda:{_device.device_index()}"
            bufs = {q: th.empty(shapes[q], dtype=dtype, device=dev) for q in range(self.P)}
            self._bufs[key] = (bufs, {r: [bufs[q] for q in range(self.P)] for r in self.ranks})
        return self._bufs[key]

    def barrier(self):
        pass  # one stream: the writers precede the readers in stream order


class TorchPeerExchange(TorchExchange):
    """Fused exchange over peer memory between processes of one node: each
    rank allocates its receive buffers, shares them by CUDA IPC handles
    (all_gather_object) and opens its peers' -- the exchanging kernels then
    store over NVLink.  barrier(): NCCL all-reduce of a flag, stream-ordered
    (all ranks' writes complete before any reader starts); on gloo (tests) a
    host-side synchronize + barrier."""

    peer = True

    def __init__(self, group=None):
        super().__init__(group)
        th = _device.torch()
        self._bufs = {}
        self._flag = th.zeros(1, device=f"cuda:{_device.device_index()}")
        self._nccl = self.dist.get_backend(group) == "nccl"

    def alloc_shared(self, key, shapes: dict, dtype):
        th = _device.torch()
        if key not in self._bufs:
            (me,) = self.ranks
            dev = f"cuda:{_device.device_index()}"
            mine = th.empty(shapes[me], dtype=dtype, device=dev)
            if mine.numel() == 0:
                mine = th.empty(1, dtype=dtype, device=dev)  # a handle even for an empty block
            handle = mine.untyped_storage()._share_cuda_()
            handles = [None] * self.P
            self.dist.all_gather_object(handles, handle, group=self.group)
            table = []
            for q in range(self.P):
                if q == me:
                    table.append(mine)
                else:
                    st = th.UntypedStorage._new_shared_cuda(*handles[q])
                    table.append(th.empty(0, dtype=dtype, device=dev).set_(st))
            self._bufs[key] = ({me: mine.view(shapes[me]) if mine.numel() else mine}, {me: table})
        return self._bufs[key]

    def barrier(self):
        if self._nccl:
            self.dist.all_reduce(self._flag, group=self.group)
        else:
            _device.torch().cuda.synchronize()
            self.dist.barrier(group=self.group)


# ---------------------------------------------------------------- GPU backend
def _ptrs(tensors):
    arr = (ctypes.c_void_p * len(tensors))(
        *[(t.data_ptr() if t is not None and t.numel() else 0) for t in tensors])
    return arr


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

    def set_peers(self, rank, blocks, bins):
        t = np.ascontiguousarray(np.asarray(blocks, dtype=np.int32).reshape(-1))
        n = np.ascontiguousarray([len(b) for b in bins], dtype=np.int32)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype=np.int32) for b in bins])
                                   if sum(n) else np.zeros(1, np.int32))
        ip = ctypes.POINTER(ctypes.c_int)
        _native.check(self.lib.s2w_shard_set_peers(
            self.h, len(bins), rank, t.ctypes.data_as(ip), n.ctypes.data_as(ip),
            cat.ctypes.data_as(ip)))

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
    wplans: dict            # rank -> _GpuShard, weight row i = fac of the grid's i-th large scale


_SETS_MAX = 3  # weighted sets per shard Legendre launch (s2w_shard_legendre_*_sets)


def whole_scale_owners(bands, P: int, whole_max: int = 256) -> dict:
    """Scales with band <= whole_max, dealt whole to ranks: largest band first,
    each to the least loaded rank (cost ~ k^3).  {scale j: rank}."""
    load = np.zeros(P)
    own = {}
    for j in sorted((j for j, k in enumerate(bands) if k <= whole_max), key=lambda j: (-bands[j], j)):
        r = int(np.argmin(load))
        own[j] = r
        load[r] += float(bands[j]) ** 3
    return own


class ShardedWaveletTransform:
    """Wavelet analysis / synthesis of one map sharded over P ranks.

    The map and the large scale maps are ring-sharded: ``analysis({rank:
    x_rows})`` with x_rows of shape (batch, t1 - t0, 2L-1) (``ring_block``)
    returns ``{rank: [scale map j]}`` where a large scale's entry is the rank's
    ring block and a whole scale's (band <= whole_max, ``whole_owner``) is the
    full map on its owner and an empty (batch, 0, 2k-1) tensor elsewhere;
    ``synthesis`` takes the same layout back.
    """

    def __init__(self, config: TransformConfig, exchange, batch: int = 1, real: bool = False,
                 whole_max: int = 256):
        _device.require_cuda()
        self.cfg, self.ex, self.B, self.real = config, exchange, batch, bool(real)
        self.P = exchange.P
        self.whole_max = whole_max
        kern = kernels_for(config)
        self.bands = scale_bands(config, kern)
        L = config.L
        ell = np.arange(L, dtype=np.float64)
        self.fac = np.sqrt(4.0 * np.pi / (2.0 * ell + 1.0))[None, :] * kern.table()
        owner = order_owner(L, self.P)
        self.owner = owner
        self.whole_owner = whole_scale_owners(self.bands, self.P, whole_max)
        self.large = [j for j in range(len(self.bands)) if j not in self.whole_owner]
        self.ks = max([self.bands[j] for j in self.whole_owner], default=0)
        self.grids = {}
        for k in sorted(set([L] + [self.bands[j] for j in self.large])):
            blocks = ring_blocks(k, self.P)
            orders = [np.nonzero(owner[:k] == r)[0] for r in range(self.P)]
            bins = [shard_bins(k, o, self.real) for o in orders]
            g = _Grid(k, blocks, orders, bins, {}, {})
            self.grids[k] = g
            for r in exchange.ranks:
                t0, t1 = blocks[r]
                g.plans[r] = _GpuShard(config.scheme, k, batch, real, orders[r], t0, t1, None)
                g.plans[r].set_peers(r, blocks, bins)
        # one weighted plan per (rank, large grid): weight row i = fac of the
        # grid's i-th scale, so the scales sharing a grid run as one launch
        self.large_groups = {}
        for j in self.large:
            self.large_groups.setdefault(self.bands[j], []).append(j)
        for k, js in self.large_groups.items():
            g = self.grids[k]
            for r in exchange.ranks:
                t0, t1 = g.blocks[r]
                p = _GpuShard(config.scheme, k, batch, real, g.orders[r], t0, t1,
                              self.fac[js, :k])
                p.set_peers(r, g.blocks, g.bins)
                g.wplans[r] = p
        # whole scales: the owner's plan holds every order and every ring
        self.wholeplans = {}
        for j, r in self.whole_owner.items():
            if r in exchange.ranks:
                k = self.bands[j]
                p = _GpuShard(config.scheme, k, batch, real, np.arange(k), 0, k,
                              self.fac[j:j + 1, :k])
                # one "rank" holding everything: local bin order for the ring DFTs,
                # natural order back through scatter_bins
                p.set_peers(0, [(0, k)], [shard_bins(k, np.arange(k), self.real)])
                self.wholeplans[j] = p
        th = _device.torch()
        self.dev = f"cuda:{_device.device_index()}"
        self.f = {r: th.zeros((batch, L * L), dtype=th.complex128, device=self.dev)
                  for r in exchange.ranks}
        self.flow = {r: th.zeros((batch, self.ks * self.ks), dtype=th.complex128, device=self.dev)
                     for r in exchange.ranks}

    # -- helpers
    def _nb(self, k):
        return k if self.real else 2 * k - 1

    def _stream(self):
        return _device.stream_handle()

    def _map_dtype(self):
        th = _device.torch()
        return th.float64 if self.real else th.complex128

    def _forward_peers(self, items: list) -> dict:
        """Fused analysis-direction exchange: the ring DFTs of every rank store
        their bins straight into the owners' H_local (s2w_shard_rings_forward_peers)."""
        th = _device.torch()
        self.ex.barrier()  # the owners have finished reading their previous H
        bufs = {}
        for key, k, plan_of, rows in items:
            g = self.grids[k]
            shapes = {q: (self.B, len(g.bins[q]), k) for q in range(self.P)}
            own, tables = self.ex.alloc_shared(("H", key), shapes, th.complex128)
            bufs[key] = own
            for r in self.ex.ranks:
                plan_of(r).call("s2w_shard_rings_forward_peers", _device.ptr(rows[r]),
                                _ptrs(tables[r]), self._stream())
        self.ex.barrier()  # every rank's stores have landed
        out = {}
        for r in self.ex.ranks:
            out[r] = {}
            for key, k, plan_of, _ in items:
                H = bufs[key][r]
                if len(self.grids[k].bins[r]):
                    plan_of(r).call("s2w_shard_theta", _device.ptr(H), self._stream())
                out[r][key] = H
        return out

    def _inverse_peers(self, items: list) -> dict:
        """Fused synthesis-direction exchange: every rank pushes its G_local
        straight into the ring owners' G_ring (s2w_shard_push_rings)."""
        th = _device.torch()
        self.ex.barrier()  # the owners have finished reading their previous G_ring
        bufs = {}
        for key, k, plan_of, gl in items:
            g = self.grids[k]
            shapes = {q: (self.B, g.blocks[q][1] - g.blocks[q][0], self._nb(k)) for q in range(self.P)}
            own, tables = self.ex.alloc_shared(("G", key), shapes, th.complex128)
            bufs[key] = own
            for r in self.ex.ranks:
                plan_of(r).call("s2w_shard_push_rings", _device.ptr(gl[r]), _ptrs(tables[r]),
                                self._stream())
        self.ex.barrier()
        out = {}
        for r in self.ex.ranks:
            out[r] = {}
            for key, k, plan_of, _ in items:
                g = self.grids[k]
                t = g.blocks[r][1] - g.blocks[r][0]
                x = th.empty((self.B, t, 2 * k - 1), dtype=self._map_dtype(), device=self.dev)
                if t:
                    plan_of(r).call("s2w_shard_rings_inverse", _device.ptr(bufs[key][r]),
                                    _device.ptr(x), self._stream())
                out[r][key] = x
        return out

    def _forward_many(self, items: list) -> dict:
        """items: [(key, k, plan_of(r), {rank: map rows})] -> {rank: {key: H_local}}
        (ring DFTs of my rings, ONE grouped exchange, MW theta stage)."""
        if getattr(self.ex, "peer", False):
            return self._forward_peers(items)
        th = _device.torch()
        sends, shapes, gcols = {}, {}, {}
        for r in self.ex.ranks:
            sends[r], shapes[r], gcols[r] = {}, {}, {}
            for key, k, plan_of, rows in items:
                g = self.grids[k]
                t = g.blocks[r][1] - g.blocks[r][0]
                gc = th.empty(self.B * self._nb(k) * t, dtype=th.complex128, device=self.dev)
                plan_of(r).call("s2w_shard_rings_forward", _device.ptr(rows[r]), _device.ptr(gc),
                                self._stream())
                gcols[r][key] = gc
                # destination-grouped blocks [B][n_q][t_r]: views, no packing
                parts, o = [], 0
                for q in range(self.P):
                    n = self.B * len(g.bins[q]) * t
                    parts.append(gc[o:o + n].view(self.B, len(g.bins[q]), t))
                    o += n
                sends[r][key] = parts
                shapes[r][key] = [(self.B, len(g.bins[r]), g.blocks[q][1] - g.blocks[q][0])
                                  for q in range(self.P)]
        got = self.ex.exchange(sends, shapes)
        out = {}
        for r in self.ex.ranks:
            out[r] = {}
            for key, k, plan_of, _ in items:
                g = self.grids[k]
                if self.P == 1:
                    # one rank: its destination block [B][n_local][k] is H itself
                    H = got[r][key][0]
                else:
                    H = th.empty((self.B, len(g.bins[r]), k), dtype=th.complex128, device=self.dev)
                    if len(g.bins[r]):
                        plan_of(r).call("s2w_shard_gather_rings", _ptrs(got[r][key]),
                                        _device.ptr(H), self._stream())
                if len(g.bins[r]):
                    plan_of(r).call("s2w_shard_theta", _device.ptr(H), self._stream())
                out[r][key] = H
        return out

    def _inverse_many(self, items: list) -> dict:
        """items: [(key, k, plan_of(r), {rank: G_local [B][k][n_local]})] ->
        {rank: {key: map rows}} (ONE grouped exchange, ring inverse DFTs)."""
        if getattr(self.ex, "peer", False):
            return self._inverse_peers(items)
        th = _device.torch()
        sends, shapes = {}, {}
        for r in self.ex.ranks:
            sends[r], shapes[r] = {}, {}
            for key, k, _, gl in items:
                g = self.grids[k]
                G = gl[r]
                # ring-major rows: each destination's ring block is contiguous per set
                if self.B == 1:
                    sends[r][key] = [G[:, g.blocks[q][0]:g.blocks[q][1], :] for q in range(self.P)]
                else:
                    sends[r][key] = [G[:, g.blocks[q][0]:g.blocks[q][1], :].contiguous()
                                     for q in range(self.P)]
                t = g.blocks[r][1] - g.blocks[r][0]
                shapes[r][key] = [(self.B, t, len(g.bins[q])) for q in range(self.P)]
        got = self.ex.exchange(sends, shapes)
        out = {}
        for r in self.ex.ranks:
            out[r] = {}
            for key, k, plan_of, _ in items:
                g = self.grids[k]
                t = g.blocks[r][1] - g.blocks[r][0]
                ring = th.empty((self.B, t, self._nb(k)), dtype=th.complex128, device=self.dev)
                x = th.empty((self.B, t, 2 * k - 1), dtype=self._map_dtype(), device=self.dev)
                if t:
                    plan_of(r).call("s2w_shard_scatter_bins", _ptrs(got[r][key]), _device.ptr(ring),
                                    self._stream())
                    plan_of(r).call("s2w_shard_rings_inverse", _device.ptr(ring), _device.ptr(x),
                                    self._stream())
                out[r][key] = x
        return out

    def _empty_map(self, k):
        th = _device.torch()
        return th.empty((self.B, 0, 2 * k - 1), dtype=self._map_dtype(), device=self.dev)

    # -- public
    def analysis(self, x_rows: dict) -> dict:
        th = _device.torch()
        L = self.cfg.L
        top = self.grids[L]
        H = self._forward_many([("top", L, lambda r: top.plans[r], x_rows)])
        for r in self.ex.ranks:
            top.plans[r].call("s2w_shard_legendre_analysis", _device.ptr(H[r]["top"]),
                              _device.ptr(self.f[r]), L, -1, 0, self._stream())
        out = {r: [None] * len(self.bands) for r in self.ex.ranks}
        # whole scales: complete low-degree f on every rank (one all-reduce)
        if self.whole_owner:
            ks = self.ks
            for r in self.ex.ranks:
                self.flow[r].copy_(self.f[r][:, :ks * ks])
            self.ex.all_reduce(self.flow)
            for j, k in enumerate(self.bands):
                if j not in self.whole_owner:
                    continue
                for r in self.ex.ranks:
                    if self.whole_owner[j] != r:
                        out[r][j] = self._empty_map(k)
                        continue
                    p = self.wholeplans[j]
                    G = th.empty((self.B, k, self._nb(k)), dtype=th.complex128, device=self.dev)
                    p.call("s2w_shard_legendre_synthesis", _device.ptr(self.flow[r]), ks, 0,
                           _device.ptr(G), self._stream())
                    ring = th.empty_like(G)
                    p.call("s2w_shard_scatter_bins", _ptrs([G]), _device.ptr(ring), self._stream())
                    x = th.empty((self.B, k, 2 * k - 1), dtype=self._map_dtype(), device=self.dev)
                    p.call("s2w_shard_rings_inverse", _device.ptr(ring), _device.ptr(x),
                           self._stream())
                    out[r][j] = x
        # large scales: order-sharded synthesis, ONE grouped exchange, ring inverse
        items = []
        for k, js in self.large_groups.items():
            g = self.grids[k]
            gls = {j: {} for j in js}
            for r in self.ex.ranks:
                Gs = [th.empty((self.B, k, len(g.bins[r])), dtype=th.complex128, device=self.dev)
                      for _ in js]
                if len(g.bins[r]):
                    for c0 in range(0, len(js), _SETS_MAX):  # <= 3 sets per launch
                        n = min(_SETS_MAX, len(js) - c0)
                        w = (ctypes.c_int * n)(*range(c0, c0 + n))
                        g.wplans[r].call("s2w_shard_legendre_synthesis_sets",
                                         _device.ptr(self.f[r]), L, n, w, _ptrs(Gs[c0:c0 + n]),
                                         self._stream())
                for j, G in zip(js, Gs):
                    gls[j][r] = G
            for j in js:
                items.append((f"s{j:03d}", k, (lambda g_: lambda r: g_.wplans[r])(g), gls[j]))
        maps = self._inverse_many(items) if items else {r: {} for r in self.ex.ranks}
        for j in self.large:
            for r in self.ex.ranks:
                out[r][j] = maps[r][f"s{j:03d}"]
        return out

    def synthesis(self, scale_rows: dict) -> dict:
        th = _device.torch()
        L = self.cfg.L
        # whole scales on their owners, folded in scale order, then one all-reduce
        for r in self.ex.ranks:
            self.f[r].zero_()
        if self.whole_owner:
            ks = self.ks
            for r in self.ex.ranks:
                self.flow[r].zero_()
            for j in sorted(self.whole_owner):
                r = self.whole_owner[j]
                if r not in self.ex.ranks:
                    continue
                k = self.bands[j]
                p = self.wholeplans[j]
                H = th.empty((self.B, self._nb(k), k), dtype=th.complex128, device=self.dev)
                p.call("s2w_shard_rings_forward", _device.ptr(scale_rows[r][j]), _device.ptr(H),
                       self._stream())
                p.call("s2w_shard_theta", _device.ptr(H), self._stream())
                p.call("s2w_shard_legendre_analysis", _device.ptr(H), _device.ptr(self.flow[r]),
                       ks, 0, 1, self._stream())
            self.ex.all_reduce(self.flow)
            for r in self.ex.ranks:
                self.f[r][:, :ks * ks].copy_(self.flow[r])
        # large scales: ring DFTs, ONE grouped exchange, order-sharded analysis
        items = []
        for j in self.large:
            k = self.bands[j]
            g = self.grids[k]
            items.append((f"s{j:03d}", k, (lambda g_: lambda r: g_.wplans[r])(g),
                          {r: scale_rows[r][j] for r in self.ex.ranks}))
        H = self._forward_many(items) if items else {r: {} for r in self.ex.ranks}
        # grids in increasing band = scale order; a grid's scales fold in one launch
        for k, js in self.large_groups.items():
            g = self.grids[k]
            for r in self.ex.ranks:
                for c0 in range(0, len(js), _SETS_MAX):  # <= 3 sets per launch, in order
                    n = min(_SETS_MAX, len(js) - c0)
                    w = (ctypes.c_int * n)(*range(c0, c0 + n))
                    g.wplans[r].call("s2w_shard_legendre_analysis_sets", n,
                                     _ptrs([H[r][f"s{j:03d}"] for j in js[c0:c0 + n]]), w,
                                     _device.ptr(self.f[r]), L, 1, self._stream())
        top = self.grids[L]
        gl = {}
        for r in self.ex.ranks:
            G = th.empty((self.B, L, len(top.bins[r])), dtype=th.complex128, device=self.dev)
            if len(top.bins[r]):
                top.plans[r].call("s2w_shard_legendre_synthesis", _device.ptr(self.f[r]), L, -1,
                                  _device.ptr(G), self._stream())
            gl[r] = G
        rows = self._inverse_many([("top", L, lambda r: top.plans[r], gl)])
        return {r: rows[r]["top"] for r in self.ex.ranks}

    def round_trip(self, x_rows: dict) -> dict:
        return self.synthesis(self.analysis(x_rows))

    def ring_block(self, k: int, rank: int) -> tuple[int, int]:
        return ring_blocks(k, self.P)[rank]

    def exchange_bytes(self) -> dict:
        return exchange_bytes(self.cfg, self.P, self.B, self.real, self.whole_max)


def exchange_bytes(config: TransformConfig, P: int, batch: int = 1, real: bool = False,
                   whole_max: int = 256) -> dict:
    """Bytes that leave the busiest rank per exchange of one round trip (pure
    host arithmetic): the exchanges move G / H blocks of complex128, a rank's
    own block stays local; the all-reduces move B k_s^2 complex128."""
    L, B = config.L, batch
    bands = scale_bands(config, kernels_for(config))
    owner = order_owner(L, P)
    whole = whole_scale_owners(bands, P, whole_max)
    ks = max([bands[j] for j in whole], default=0)

    def a2a(k):
        g = ring_blocks(k, P)
        orders = [np.nonzero(owner[:k] == r)[0] for r in range(P)]
        nb = [len(shard_bins(k, o, real)) for o in orders]
        return max(sum(B * nb[q] * (g[r][1] - g[r][0]) * 16 for q in range(P) if q != r)
                   for r in range(P))

    large = sum(a2a(k) for j, k in enumerate(bands) if j not in whole)
    ar = B * ks * ks * 16
    return {"top_a2a": a2a(L), "large_scales_a2a": large, "whole_allreduce": ar,
            "per_round_trip_max_rank": 2 * a2a(L) + 2 * large + 2 * ar}
