"""Spherical harmonic transforms (drop-in for sphwav/sht.py).

Public names, layouts and error behaviour follow the reference
(sht.py:35-355); the arithmetic runs in the sm_100a kernels of libs2w.so:

* ``sh_synthesis[_stack]``  -> ``s2w_sh_synthesis``: on-the-fly FP64 Legendre
  recursion + contraction (legendre_kernels.cu), ring inverse DFTs and the MW
  pole pinning (fft_kernels.cu);
* ``sh_analysis[_stack]``   -> ``s2w_sh_analysis``: ring DFTs, the MW theta
  stage (the reference raises on MW, sht.py:300-303; here MW analysis is
  exact) and the deterministic ring reduction;
* ``assoc_legendre_ring``   -> ``s2w_assoc_legendre_ring`` (extended-exponent
  recursion, valid to L = 4096 (the FFT engine limit), unlike the reference's 1e-280 flush).

Coefficients use the flat ``l*l + l + m`` layout; real-signal sets carry the
exact conjugate symmetry ``f(l,-m) = (-1)^m conj f(l,m)``.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _device, _native
from .errors import ParameterError
from .grid import GridSpec, SamplingScheme, SphereMap, scheme_code

__all__ = [
    "HarmonicCoeffs",
    "lm_index",
    "sh_synthesis",
    "sh_analysis",
    "sh_synthesis_stack",
    "sh_analysis_stack",
    "assoc_legendre_ring",
    "pad_coeffs",
    "truncate_coeffs",
]


def lm_index(ell: int, m: int) -> int:
    """Flat index of (ell, m): ell^2 + ell + m (sht.py:50-52)."""
    return ell * ell + ell + m


@lru_cache(maxsize=32)
def _mirror_index(L: int):
    """Index arrays (pos, neg, sign, m0) pairing (l, m>0) with (l, -m)."""
    ell = np.repeat(np.arange(L), np.arange(L))            # l for every m in 1..l
    m = np.concatenate([np.arange(1, l + 1) for l in range(L)]) if L > 1 else np.zeros(0, int)
    base = ell * ell + ell
    sign = np.where(m % 2 == 1, -1.0, 1.0)
    m0 = np.arange(L) ** 2 + np.arange(L)
    return base + m, base - m, sign, m0


def _is_conj_symmetric(L: int, c: np.ndarray) -> bool:
    pos, neg, sign, m0 = _mirror_index(L)
    if np.any(c[m0].imag != 0.0):
        return False
    return bool(np.all(c[neg] == sign * np.conj(c[pos])))


@dataclass(frozen=True, eq=False)
class HarmonicCoeffs:
    """Band-limited coefficients, flat layout ``idx = l^2 + l + m`` (sht.py:55-91)."""

    L: int
    coeffs: np.ndarray
    real_signal: bool = False

    def __post_init__(self):
        if self.L < 1:
            raise ParameterError(f"band-limit must be >= 1, got {self.L}")
        c = np.ascontiguousarray(self.coeffs, dtype=np.complex128)
        if c.shape != (self.L * self.L,):
            raise ParameterError(f"expected {self.L * self.L} coefficients, got shape {c.shape}")
        if self.real_signal and not _is_conj_symmetric(self.L, c):
            raise ParameterError("coefficients flagged real-signal lack conjugate symmetry")
        c.setflags(write=False)
        object.__setattr__(self, "coeffs", c)

    @classmethod
    def zeros(cls, L: int, real_signal: bool = False) -> "HarmonicCoeffs":
        return cls(L, np.zeros(L * L, dtype=np.complex128), real_signal)

    def __getitem__(self, lm: tuple[int, int]) -> complex:
        ell, m = lm
        if not (0 <= ell < self.L and abs(m) <= ell):
            raise ParameterError(f"(ell, m) = {lm} out of range for L = {self.L}")
        return complex(self.coeffs[lm_index(ell, m)])


def pad_coeffs(flm: HarmonicCoeffs, L: int) -> HarmonicCoeffs:
    """Zero rows above flm.L (prefix copy, sht.py:120-128)."""
    if L < flm.L:
        raise ParameterError(f"cannot pad band-limit {flm.L} down to {L}")
    if L == flm.L:
        return flm
    out = np.zeros(L * L, dtype=np.complex128)
    out[: flm.L * flm.L] = flm.coeffs
    return HarmonicCoeffs(L, out, flm.real_signal)


def truncate_coeffs(flm: HarmonicCoeffs, L: int) -> HarmonicCoeffs:
    """Keep degrees below L: a prefix of the flat layout (sht.py:131-137)."""
    if L > flm.L:
        raise ParameterError(f"cannot truncate band-limit {flm.L} up to {L}")
    if L == flm.L:
        return flm
    return HarmonicCoeffs(L, flm.coeffs[: L * L].copy(), flm.real_signal)


def assoc_legendre_ring(L: int, theta: float) -> np.ndarray:
    """(L, L) table of orthonormal P_lm(cos theta), zero above the diagonal."""
    if not 0.0 <= theta <= np.pi:
        raise ParameterError(f"colatitude must lie in [0, pi], got {theta}")
    if L < 1:
        raise ParameterError(f"band-limit must be >= 1, got {L}")
    _device.require_cuda()
    out = _device.empty(L * L)
    _native.check(
        _native.load().s2w_assoc_legendre_ring(
            L, float(theta), _device.ptr(out), _device.stream_handle()
        )
    )
    return _device.to_host(out).reshape(L, L)


# ---------------------------------------------------------------- device entry points
def synthesis_device(flm_dev, n_sets: int, L_coef: int, real: bool, grid: GridSpec):
    """Device tensors in/out: flm (n*Lc^2 complex as 2 doubles) -> map doubles."""
    _device.require_cuda()
    plan = _device.sht_plan(scheme_code(grid.scheme), grid.L)
    per = grid.n_theta * grid.n_phi * (1 if real else 2)
    out = _device.empty(n_sets * per)
    _native.check(
        _native.load().s2w_sh_synthesis(
            plan.handle, n_sets, L_coef, int(real), _device.ptr(flm_dev), _device.ptr(out),
            _device.stream_handle(),
        )
    )
    return out


def analysis_device(map_dev, n_sets: int, real: bool, grid: GridSpec):
    _device.require_cuda()
    plan = _device.sht_plan(scheme_code(grid.scheme), grid.L)
    out = _device.empty(n_sets * grid.L * grid.L * 2)
    _native.check(
        _native.load().s2w_sh_analysis(
            plan.handle, n_sets, int(real), _device.ptr(map_dev), _device.ptr(out),
            _device.stream_handle(),
        )
    )
    return out


def maps_to_device(smaps, real: bool):
    """Maps -> flat device doubles (real maps: their real parts).  The
    complex128 values travel as they are and the real part is taken on the
    device (s2w_complex_real_part): no host pass over the arrays."""
    vals = (smaps[0].values if len(smaps) == 1  # no stacking copy for a single map
            else np.stack([m.values for m in smaps]))
    cdev = _device.to_device(vals.view(np.float64).reshape(-1))
    if not real:
        return cdev
    n = cdev.numel() // 2
    out = _device.empty(n)
    _native.check(_native.load().s2w_complex_real_part(
        _device.ptr(cdev), _device.ptr(out), n, _device.stream_handle()))
    return out


def maps_from_device(dev, grid: GridSpec, n: int, real: bool) -> list[SphereMap]:
    """Flat device doubles -> maps.  Real maps become complex128 on the device
    (s2w_real_to_complex) and are copied straight into the arrays the maps
    own; the maps are built without re-checking what the pipeline guarantees
    (zero imaginary parts, the MW pole ring pinned by phi_inv)."""
    shape = (n, grid.n_theta, grid.n_phi)
    if real:
        cdev = _device.empty(2 * dev.numel())
        _native.check(_native.load().s2w_real_to_complex(
            _device.ptr(dev), _device.ptr(cdev), dev.numel(), _device.stream_handle()))
        dev = cdev
    vals = _device.host_result(dev, np.complex128).reshape(shape)
    return [_trusted_map(grid, vals[i], real) for i in range(n)]


def _trusted_map(grid: GridSpec, values: np.ndarray, real: bool) -> SphereMap:
    m = object.__new__(SphereMap)
    values.setflags(write=False)
    object.__setattr__(m, "grid", grid)
    object.__setattr__(m, "values", values)
    object.__setattr__(m, "is_real", bool(real))
    return m


# ---------------------------------------------------------------- numpy API
def sh_synthesis_stack(flms: list[HarmonicCoeffs], grid: GridSpec) -> list[SphereMap]:
    """Synthesise several sets sharing one grid in one launch (sht.py:222-281)."""
    if not flms:
        return []
    if any(f.L > grid.L for f in flms):
        raise ParameterError("coefficient band-limit exceeds the grid band-limit")
    real = flms[0].real_signal
    if any(f.real_signal != real for f in flms):
        raise ParameterError("cannot mix real-signal and complex sets in one sweep")
    n = len(flms)
    Lc = max(f.L for f in flms)
    host = np.zeros((n, Lc * Lc), dtype=np.complex128)
    for i, f in enumerate(flms):
        host[i, : f.L * f.L] = f.coeffs
    dev = _device.to_device(host.view(np.float64).reshape(-1))
    out = synthesis_device(dev, n, Lc, real, grid)
    return maps_from_device(out, grid, n, real)


def sh_synthesis(flm: HarmonicCoeffs, grid: GridSpec) -> SphereMap:
    """Evaluate the band-limited signal on every grid sample (sht.py:284-290)."""
    if grid.L < flm.L:
        raise ParameterError(f"grid band-limit {grid.L} is below coefficient band-limit {flm.L}")
    return sh_synthesis_stack([flm], grid)[0]


def sh_analysis_stack(smaps: list[SphereMap]) -> list[HarmonicCoeffs]:
    """Analyse maps sharing one grid (GL quadrature or MW sampling theorem)."""
    if not smaps:
        return []
    grid = smaps[0].grid
    if any(m.grid != grid for m in smaps):
        raise ParameterError("all maps in a sweep must share one grid")
    real = smaps[0].is_real
    if any(m.is_real != real for m in smaps):
        raise ParameterError("cannot mix real and complex maps in one sweep")
    n = len(smaps)
    dev = maps_to_device(smaps, real)
    out = analysis_device(dev, n, real, grid)
    flm = _device.to_host(out).view(np.complex128).reshape(n, grid.L * grid.L)
    return [HarmonicCoeffs(grid.L, flm[i], real_signal=real) for i in range(n)]


def sh_analysis(smap: SphereMap) -> HarmonicCoeffs:
    """Exact projection onto the harmonic basis (sht.py:349-355; MW supported)."""
    return sh_analysis_stack([smap])[0]
