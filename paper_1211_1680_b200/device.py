"""Device-resident public API (torch tensors in, torch tensors out).

The numpy drop-in (``sht``/``transform``) copies host arrays in and out on every
call.  These classes keep maps and coefficients in HBM and expose the same
transforms on torch tensors; host tensors (ideally pinned) are copied to the
device inside the call, which is what bench.py's end-to-end figure times.

Layouts: complex maps are complex128 tensors (batch, L, 2L-1); real maps are
float64 tensors of the same shape; coefficients are complex128 (batch, L*L).
"""
from __future__ import annotations

import numpy as np

from . import _device, _native
from .errors import ParameterError
from .grid import make_grid, scheme_code
from .transform import TransformConfig, kernels_for, scale_bands

__all__ = ["WaveletTransform", "SphericalHarmonicTransform"]


def _on_device(t):
    if t.is_cuda:
        return t.contiguous()
    return t.to(device=f"cuda:{_device.device_index()}", non_blocking=True)


def _checked(t, shape, dtype, what):
    """The C ABI trusts its pointers: refuse anything whose extent, element
    type, device or layout differs from what the kernels will address."""
    th = _device.torch()
    if not isinstance(t, th.Tensor):
        raise ParameterError(f"{what}: expected a torch tensor, got {type(t).__name__}")
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype:
        raise ParameterError(f"{what}: expected {dtype} of shape {tuple(shape)}, "
                             f"got {t.dtype} of shape {tuple(t.shape)}")
    if not t.is_cuda or t.device.index != _device.device_index():
        raise ParameterError(f"{what}: must live on cuda:{_device.device_index()}, got {t.device}")
    if not t.is_contiguous():
        raise ParameterError(f"{what}: must be contiguous")
    return t


class SphericalHarmonicTransform:
    """SHT on one grid for batches of device tensors."""

    def __init__(self, scheme, L: int):
        _device.require_cuda()
        self.grid = make_grid(scheme, L)
        self.plan = _device.sht_plan(scheme_code(scheme), L)

    def synthesis(self, flm, real: bool = False):
        th = _device.torch()
        flm = _on_device(flm)
        if flm.dim() != 2 or flm.shape[0] < 1:
            raise ParameterError(f"flm: expected (batch, Lc*Lc), got shape {tuple(flm.shape)}")
        n = flm.shape[0]
        Lc = int(round(np.sqrt(flm.shape[1])))
        if Lc * Lc != flm.shape[1] or not 1 <= Lc <= self.grid.L:
            raise ParameterError(f"flm: {flm.shape[1]} coefficients is not Lc*Lc with "
                                 f"1 <= Lc <= {self.grid.L}")
        _checked(flm, (n, Lc * Lc), th.complex128, "flm")
        g = self.grid
        dt = th.float64 if real else th.complex128
        out = th.empty((n, g.n_theta, g.n_phi), dtype=dt, device=flm.device)
        _native.check(_native.load().s2w_sh_synthesis(
            self.plan.handle, n, Lc, int(real), _device.ptr(flm), _device.ptr(out),
            _device.stream_handle()))
        return out

    def analysis(self, maps):
        th = _device.torch()
        maps = _on_device(maps)
        real = not maps.is_complex()
        if maps.dim() != 3 or maps.shape[0] < 1:
            raise ParameterError(f"maps: expected (batch, n_theta, n_phi), got {tuple(maps.shape)}")
        n = maps.shape[0]
        g = self.grid
        _checked(maps, (n, g.n_theta, g.n_phi), th.float64 if real else th.complex128, "maps")
        L = g.L
        out = th.empty((n, L * L), dtype=th.complex128, device=maps.device)
        _native.check(_native.load().s2w_sh_analysis(
            self.plan.handle, n, int(real), _device.ptr(maps), _device.ptr(out),
            _device.stream_handle()))
        return out


class WaveletTransform:
    """Wavelet analysis/synthesis of ``batch`` maps sharing one TransformConfig."""

    def __init__(self, config: TransformConfig, batch: int = 1, real: bool = False):
        _device.require_cuda()
        if batch < 1:
            raise ParameterError("batch must be >= 1")
        self.config, self.batch, self.real = config, batch, bool(real)
        kern = kernels_for(config)
        self.bands = scale_bands(config, kern)
        self.plan = _device.wav_plan(scheme_code(config.scheme), config.L, batch, real,
                                     kern.table(), self.bands)
        self.grids = [make_grid(config.scheme, k) for k in self.bands]
        self.map_shape = (batch, config.L, 2 * config.L - 1)

    def _dtype(self):
        th = _device.torch()
        return th.float64 if self.real else th.complex128

    def set_concurrency(self, on: bool) -> None:
        """Per-scale ring stages on forked side streams (default) or serially on
        the caller's stream (per-stage profiling); results are identical."""
        _native.check(_native.load().s2w_wav_plan_set_concurrency(self.plan.handle, int(bool(on))))

    def _check_scale_maps(self, maps, what):
        if len(maps) != len(self.grids):
            raise ParameterError(f"{what}: expected {len(self.grids)} scale maps "
                                 f"(scaling + wavelets), got {len(maps)}")
        for j, (m, g) in enumerate(zip(maps, self.grids)):
            _checked(m, (self.batch, g.n_theta, g.n_phi), self._dtype(), f"{what}[{j}]")

    def alloc_scale_maps(self):
        th = _device.torch()
        return [th.empty((self.batch, g.n_theta, g.n_phi), dtype=self._dtype(),
                         device=f"cuda:{_device.device_index()}") for g in self.grids]

    def analysis(self, x, outs=None):
        """x: (batch, L, 2L-1) map tensor -> [scaling, j0..J] map tensors."""
        x = _checked(_on_device(x), self.map_shape, self._dtype(), "x")
        outs = self.alloc_scale_maps() if outs is None else list(outs)
        self._check_scale_maps(outs, "outs")
        _native.check(_native.load().s2w_wav_analysis_pixel(
            self.plan.handle, _device.ptr(x), _device.ptr_array(outs), _device.stream_handle()))
        return outs

    def synthesis(self, maps, out=None):
        th = _device.torch()
        maps = [_on_device(m) for m in maps]
        self._check_scale_maps(maps, "maps")
        if out is None:
            out = th.empty(self.map_shape, dtype=self._dtype(), device=maps[0].device)
        _checked(out, self.map_shape, self._dtype(), "out")
        _native.check(_native.load().s2w_wav_synthesis_pixel(
            self.plan.handle, _device.ptr_array(maps), _device.ptr(out), _device.stream_handle()))
        return out

    def round_trip(self, x, scale_maps=None, out=None):
        return self.synthesis(self.analysis(x, scale_maps), out)

    def round_trip_graph(self, x, scale_maps, out):
        """round_trip(x, scale_maps, out) replayed from a CUDA graph captured on
        first use for these buffers (small maps are launch-bound: the graph
        removes the host launch cost of the ~30 kernels per round trip)."""
        th = _device.torch()
        graphs = self.__dict__.setdefault("_graphs", {})
        key = (x.data_ptr(), out.data_ptr(), tuple(m.data_ptr() for m in scale_maps))
        g = graphs.get(key)
        if g is None:
            self.round_trip(x, scale_maps, out)  # allocates the plan's workspaces
            th.cuda.synchronize()
            was = _native.profile_enabled()
            _native.profile_enable(False)
            g = th.cuda.CUDAGraph()
            s = th.cuda.Stream()
            s.wait_stream(th.cuda.current_stream())
            with th.cuda.stream(s):
                with th.cuda.graph(g, stream=s):
                    self.round_trip(x, scale_maps, out)
            th.cuda.current_stream().wait_stream(s)
            _native.profile_enable(was)
            graphs[key] = g
        g.replay()
        return out

    def round_trip_stream(self, inputs, outputs):
        """Round trips of a sequence of host maps (pinned tensors of map_shape)
        into host tensors, double-buffered: the host-to-device copy of map i+1
        and the device-to-host copy of map i-1 run on their own streams while
        map i is transformed, so the transfers hide behind the transforms.
        Same results as ``outputs[i].copy_(round_trip(inputs[i]))``."""
        th = _device.torch()
        if len(inputs) != len(outputs):
            raise ParameterError("inputs and outputs must have the same length")
        n = len(inputs)
        if n == 0:
            return outputs
        for t in (*inputs, *outputs):
            if tuple(t.shape) != self.map_shape or t.dtype != self._dtype() or t.is_cuda:
                raise ParameterError(f"expected host {self._dtype()} tensors of shape {self.map_shape}")
        dev = f"cuda:{_device.device_index()}"
        comp = th.cuda.current_stream()
        h2d, d2h = th.cuda.Stream(), th.cuda.Stream()
        bufs = self.__dict__.get("_stream_bufs")
        if bufs is None:  # kept across calls (the graphs below are keyed on them)
            bufs = ([th.empty(self.map_shape, dtype=self._dtype(), device=dev) for _ in range(2)],
                    [th.empty(self.map_shape, dtype=self._dtype(), device=dev) for _ in range(2)],
                    self.alloc_scale_maps())
            self._stream_bufs = bufs
        xin, xout, scale = bufs
        # small maps are launch-bound: replay the transforms from CUDA graphs
        # (at L = 2048 graph replays slowed this overlapped stream: 82 vs 91 rt/s)
        use_graph = self.config.L <= 512
        if use_graph:
            for b in range(2):
                self.round_trip_graph(xin[b], scale, xout[b])  # capture outside the pipeline
            th.cuda.synchronize()
        in_ready = [th.cuda.Event() for _ in range(2)]
        in_free = [th.cuda.Event() for _ in range(2)]
        out_ready = [th.cuda.Event() for _ in range(2)]
        out_free = [th.cuda.Event() for _ in range(2)]
        # the buffers are fresh: nothing to wait for before their first use
        for e in (*in_free, *out_free):
            e.record(comp)
        with th.cuda.stream(h2d):
            h2d.wait_event(in_free[0])
            xin[0].copy_(inputs[0], non_blocking=True)
            in_ready[0].record(h2d)
        for i in range(n):
            b = i & 1
            if i + 1 < n:
                nb = b ^ 1
                with th.cuda.stream(h2d):
                    h2d.wait_event(in_free[nb])
                    xin[nb].copy_(inputs[i + 1], non_blocking=True)
                    in_ready[nb].record(h2d)
            comp.wait_event(in_ready[b])
            comp.wait_event(out_free[b])
            if use_graph:
                self.round_trip_graph(xin[b], scale, xout[b])
            else:
                self.synthesis(self.analysis(xin[b], scale), xout[b])
            in_free[b].record(comp)
            out_ready[b].record(comp)
            with th.cuda.stream(d2h):
                d2h.wait_event(out_ready[b])
                outputs[i].copy_(xout[b], non_blocking=True)
                out_free[b].record(d2h)
        comp.wait_stream(d2h)
        comp.wait_stream(h2d)
        # host outputs are complete when this returns, like the synchronous
        # outputs[i].copy_(round_trip(inputs[i])) it stands for
        d2h.synchronize()
        return outputs

    def flm(self):
        """View of the plan's f_lm workspace (batch, L*L) complex128."""
        import ctypes

        th = _device.torch()
        p = ctypes.c_void_p()
        _native.check(_native.load().s2w_wav_plan_flm(self.plan.handle, ctypes.byref(p)))
        L = self.config.L
        # wrap the device pointer through __cuda_array_interface__
        class _Wrap:
            __cuda_array_interface__ = {
                "shape": (self.batch, L * L, 2), "typestr": "<f8", "data": (p.value, False),
                "version": 3, "strides": None,
            }
        return th.view_as_complex(th.as_tensor(_Wrap(), device=f"cuda:{_device.device_index()}"))
