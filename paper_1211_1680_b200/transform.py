"""Axisymmetric wavelet transforms (drop-in for sphwav/transform.py).

Same names and semantics as the reference (transform.py:34-245).  The pixel
transforms run as one device pipeline per call (C-ABI s2w_wav_*_pixel):

  analysis : ring DFTs -> [MW theta stage] -> Legendre analysis at L
             -> ONE grouped Legendre synthesis over every scale grid with the
                tiling factor and multiresolution truncation fused into the
                coefficient staging -> ring inverse DFTs per scale map
  synthesis: per-scale ring DFTs -> [MW theta stage] -> ONE grouped Legendre
             analysis whose reduction epilogue applies the tiling factors and
             recombines all scales into f_lm -> Legendre synthesis at L
             -> ring inverse DFT

Batched entry points (``wav_analysis_pixel_batch`` etc.) transform several
maps sharing one config in one launch sequence.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _device, _native
from .errors import ParameterError
from .grid import GridSpec, SamplingScheme, SphereMap, make_grid, scheme_code
from .sht import (
    HarmonicCoeffs,
    maps_from_device,
    maps_to_device,
    pad_coeffs,
    sh_analysis,
    sh_synthesis,
)
from .tiling import KernelFamily, TilingParams, WaveletKernels, build_kernels

__all__ = [
    "TransformConfig",
    "WaveletDecomposition",
    "HarmonicWaveletCoeffs",
    "kernels_for",
    "wav_analysis_harmonic",
    "wav_synthesis_harmonic",
    "wav_analysis_pixel",
    "wav_synthesis_pixel",
    "wav_analysis_pixel_batch",
    "wav_synthesis_pixel_batch",
]


@dataclass(frozen=True)
class TransformConfig:
    """(L, lam, j0, family, scheme, multires); validated like TilingParams."""

    L: int
    lam: float
    j0: int = 0
    family: KernelFamily = KernelFamily.SCALE_DISCRETISED
    scheme: SamplingScheme = SamplingScheme.GL
    multires: bool = True

    def __post_init__(self):
        TilingParams(self.L, self.lam, self.j0)

    @property
    def tiling(self) -> TilingParams:
        return TilingParams(self.L, self.lam, self.j0)


@lru_cache(maxsize=64)
def _kernels(L: int, lam: float, j0: int, family: KernelFamily) -> WaveletKernels:
    return build_kernels(TilingParams(L, lam, j0), family)


def kernels_for(config: TransformConfig) -> WaveletKernels:
    """Kernel tables of a config (cached; independent of resolution mode)."""
    return _kernels(config.L, config.lam, config.j0, config.family)


@dataclass(frozen=True, eq=False)
class HarmonicWaveletCoeffs:
    scaling: HarmonicCoeffs
    wavelets: tuple[HarmonicCoeffs, ...]


def scale_bands(config: TransformConfig, kernels: WaveletKernels) -> list[int]:
    """Band-limit per [scaling, j0..J] (transform.py:108-114)."""
    if config.multires:
        return [kernels.scaling_bandlimit, *kernels.scale_bandlimits]
    return [config.L] * (kernels.params.n_scales + 1)


def _scale_grids(config: TransformConfig, kernels: WaveletKernels) -> list[GridSpec]:
    return [make_grid(config.scheme, k) for k in scale_bands(config, kernels)]


@dataclass(frozen=True, eq=False)
class WaveletDecomposition:
    """Scaling map plus one wavelet map per scale j = j0..J."""

    config: TransformConfig
    scaling: SphereMap
    wavelets: tuple[SphereMap, ...]

    def __post_init__(self):
        kernels = kernels_for(self.config)
        n = kernels.params.n_scales
        if len(self.wavelets) != n:
            raise ParameterError(
                f"expected {n} wavelet maps for scales {kernels.params.j0}..{kernels.params.J},"
                f" got {len(self.wavelets)}"
            )
        want = _scale_grids(self.config, kernels)
        have = [self.scaling.grid] + [w.grid for w in self.wavelets]
        for g, w in zip(have, want):
            if g != w:
                raise ParameterError(
                    f"decomposition grid band-limit {g.L} does not match expected {w.L}"
                )


# ---------------------------------------------------------------- plans
def _plan(config: TransformConfig, batch: int, real: bool, scheme: SamplingScheme | None = None):
    kernels = kernels_for(config)
    sch = config.scheme if scheme is None else scheme
    return _device.wav_plan(
        scheme_code(sch), config.L, batch, real, kernels.table(), scale_bands(config, kernels)
    )


def _harmonic_plan(kernels: WaveletKernels, batch: int, real: bool, bands):
    return _device.wav_plan(scheme_code(SamplingScheme.GL), kernels.L, batch, real,
                            kernels.table(), bands)


# ---------------------------------------------------------------- harmonic space
def wav_analysis_harmonic(
    flm: HarmonicCoeffs, kernels: WaveletKernels, truncate: bool = False
) -> HarmonicWaveletCoeffs:
    """W_j = f * sqrt(4pi/(2l+1)) K_j, optionally truncated to band_j (transform.py:129-150)."""
    if flm.L != kernels.L:
        raise ParameterError(
            f"coefficient band-limit {flm.L} does not match kernels ({kernels.L})"
        )
    _device.require_cuda()
    L = kernels.L
    bands = [kernels.scaling_bandlimit, *kernels.scale_bandlimits]
    plan = _harmonic_plan(kernels, 1, flm.real_signal, bands)
    out_bands = bands if truncate else [L] * len(bands)
    f_dev = _device.to_device(flm.coeffs.view(np.float64))
    outs = [_device.empty(2 * b * b) for b in out_bands]
    _native.check(
        _native.load().s2w_wav_analysis_harmonic(
            plan.handle, int(bool(truncate)), _device.ptr(f_dev), _device.ptr_array(outs),
            _device.stream_handle(),
        )
    )
    sets = [
        HarmonicCoeffs(b, _device.to_host(o).view(np.complex128), flm.real_signal)
        for b, o in zip(out_bands, outs)
    ]
    return HarmonicWaveletCoeffs(sets[0], tuple(sets[1:]))


def wav_synthesis_harmonic(
    wcoeffs: HarmonicWaveletCoeffs, kernels: WaveletKernels
) -> HarmonicCoeffs:
    """f = sum_j sqrt(4pi/(2l+1)) K_j pad(W_j), scaling first (transform.py:153-172)."""
    if len(wcoeffs.wavelets) != len(kernels.psi):
        raise ParameterError(
            f"expected {len(kernels.psi)} wavelet coefficient sets, got {len(wcoeffs.wavelets)}"
        )
    L = kernels.L
    sets = [wcoeffs.scaling, *wcoeffs.wavelets]
    for s in sets:
        if s.L > L:
            raise ParameterError(f"coefficient set band-limit {s.L} exceeds kernels ({L})")
    _device.require_cuda()
    real = all(s.real_signal for s in sets)
    bands = [kernels.scaling_bandlimit, *kernels.scale_bandlimits]
    if all(s.L == b for s, b in zip(sets, bands)):
        full = 0
    else:
        full = 1
        sets = [pad_coeffs(s, L) for s in sets]
    plan = _harmonic_plan(kernels, 1, real, bands)
    ins = [_device.to_device(s.coeffs.view(np.float64)) for s in sets]
    out = _device.empty(2 * L * L)
    _native.check(
        _native.load().s2w_wav_synthesis_harmonic(
            plan.handle, full, _device.ptr_array(ins), _device.ptr(out), _device.stream_handle()
        )
    )
    return HarmonicCoeffs(L, _device.to_host(out).view(np.complex128), real_signal=real)


# ---------------------------------------------------------------- pixel space
def wav_analysis_pixel_batch(
    smaps: list[SphereMap], config: TransformConfig
) -> list[WaveletDecomposition]:
    """Decompose maps sharing one grid (one device pipeline for the batch)."""
    if not smaps:
        return []
    grid = smaps[0].grid
    for s in smaps:
        if s.grid.L != config.L:
            raise ParameterError(
                f"map band-limit {s.grid.L} does not match config ({config.L})"
            )
        if s.grid != grid:
            raise ParameterError("all maps in a batch must share one grid")
    real = smaps[0].is_real
    if any(s.is_real != real for s in smaps):
        raise ParameterError("cannot mix real and complex maps in one batch")
    _device.require_cuda()
    if grid.scheme is not config.scheme:
        # analysis on the input grid, scale maps on the config grids
        return [_analysis_mixed_scheme(s, config) for s in smaps]
    n = len(smaps)
    kernels = kernels_for(config)
    plan = _plan(config, n, real)
    grids = _scale_grids(config, kernels)
    x = maps_to_device(smaps, real)
    outs = [_device.empty(n * g.n_theta * g.n_phi * (1 if real else 2)) for g in grids]
    _native.check(
        _native.load().s2w_wav_analysis_pixel(
            plan.handle, _device.ptr(x), _device.ptr_array(outs), _device.stream_handle()
        )
    )
    per_scale = [maps_from_device(o, g, n, real) for o, g in zip(outs, grids)]
    return [
        WaveletDecomposition(config, per_scale[0][b], tuple(ps[b] for ps in per_scale[1:]))
        for b in range(n)
    ]


def _analysis_mixed_scheme(smap: SphereMap, config: TransformConfig) -> WaveletDecomposition:
    from .sht import sh_synthesis_stack

    kernels = kernels_for(config)
    flm = sh_analysis(smap)
    wc = wav_analysis_harmonic(flm, kernels, truncate=config.multires)
    grids = _scale_grids(config, kernels)
    maps = [sh_synthesis_stack([s], g)[0] for s, g in zip([wc.scaling, *wc.wavelets], grids)]
    return WaveletDecomposition(config, maps[0], tuple(maps[1:]))


def wav_analysis_pixel(smap: SphereMap, config: TransformConfig) -> WaveletDecomposition:
    """Scaling + wavelet maps of a band-limited map (transform.py:175-191)."""
    if smap.grid.L != config.L:
        raise ParameterError(
            f"map band-limit {smap.grid.L} does not match config ({config.L})"
        )
    return wav_analysis_pixel_batch([smap], config)[0]


def wav_synthesis_pixel_batch(decomps: list[WaveletDecomposition]) -> list[SphereMap]:
    """Reconstruct several decompositions sharing one config."""
    if not decomps:
        return []
    config = decomps[0].config
    if any(d.config != config for d in decomps):
        raise ParameterError("all decompositions in a batch must share one config")
    _device.require_cuda()
    n = len(decomps)
    kernels = kernels_for(config)
    grids = _scale_grids(config, kernels)
    per_scale = [[d.scaling, *d.wavelets] for d in decomps]
    real = all(m.is_real for row in per_scale for m in row)
    plan = _plan(config, n, real)
    ins = []
    for j in range(len(grids)):
        maps = [row[j] for row in per_scale]
        if not real:
            maps = [SphereMap(m.grid, m.values, is_real=False) for m in maps]
        ins.append(maps_to_device(maps, real))
    out = _device.empty(n * config.L * (2 * config.L - 1) * (1 if real else 2))
    _native.check(
        _native.load().s2w_wav_synthesis_pixel(
            plan.handle, _device.ptr_array(ins), _device.ptr(out), _device.stream_handle()
        )
    )
    return maps_from_device(out, make_grid(config.scheme, config.L), n, real)


def wav_synthesis_pixel(decomp: WaveletDecomposition) -> SphereMap:
    """Exact inverse of wav_analysis_pixel (transform.py:194-202)."""
    return wav_synthesis_pixel_batch([decomp])[0]
