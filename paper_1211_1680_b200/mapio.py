"""Bit-exact S2WM serialization of maps and coefficients (reference: mapio.py).

Same layout, names and errors as /root/reference/pkg/src/sphwav/mapio.py:

    offset  size  field
    0       4     magic "S2WM"
    4       4     version (u32) = 1
    8       1     scheme (u8): 0 = GL, 1 = MW
    9       4     band-limit L (u32)
    13      1     kind (u8): 0 = real map, 1 = complex map, 2 = harmonic coeffs
    14      8     payload_count (u64): samples (maps) or L^2 (coeffs)

followed by little-endian float64 values (real maps) or (re, im) pairs.  The
file I/O runs in the native library (``s2w_s2wm_*``); the ``*_device``
variants move payloads between files and device tensors through pinned,
double-buffered staging (no pageable copy), for the scale maps the wavelet
pipeline produces and consumes.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _device, _native
from .errors import (
    NotS2wmFileError,
    ParameterError,
    PayloadMismatchError,
    TruncatedFileError,
    UnsupportedVersionError,
)
from .grid import GridSpec, SamplingScheme, SphereMap, make_grid
from .sht import HarmonicCoeffs

__all__ = [
    "MAGIC",
    "VERSION",
    "HEADER_SIZE",
    "NotS2wmFileError",
    "UnsupportedVersionError",
    "TruncatedFileError",
    "PayloadMismatchError",
    "write_map",
    "read_map",
    "write_flm",
    "read_flm",
    "write_map_device",
    "read_map_device",
    "write_flm_device",
    "read_flm_device",
]

MAGIC = b"S2WM"
VERSION = 1
HEADER_SIZE = 22

_KIND_REAL_MAP = 0
_KIND_COMPLEX_MAP = 1
_KIND_COEFFS = 2
_SCHEME_CODE = {SamplingScheme.GL: 0, SamplingScheme.MW: 1}
_CODE_SCHEME = {v: k for k, v in _SCHEME_CODE.items()}


def _path(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _header(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path}: no such file")
    sc, L, kind, count = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_longlong()
    _native.check(_native.load().s2w_s2wm_read_header(
        _path(path), ctypes.byref(sc), ctypes.byref(L), ctypes.byref(kind), ctypes.byref(count)))
    return sc.value, L.value, kind.value, count.value


def _write(path, scheme_code, L, kind, count, complex_payload, ptr, device):
    _native.check(_native.load().s2w_s2wm_write(
        _path(path), scheme_code, L, kind, count, int(complex_payload), ptr, int(device),
        _device.stream_handle() if device else None))


def _read_payload(path, count, complex_payload, ptr, device):
    _native.check(_native.load().s2w_s2wm_read_payload(
        _path(path), count, int(complex_payload), ptr, int(device),
        _device.stream_handle() if device else None))


def _map_grid(path, scheme_code, L, kind, count) -> GridSpec:
    """mapio.py:133-145 checks, in the reference's order."""
    if kind not in (_KIND_REAL_MAP, _KIND_COMPLEX_MAP):
        raise PayloadMismatchError(f"{path}: kind {kind} is not a map")
    if scheme_code not in _CODE_SCHEME:
        raise PayloadMismatchError(f"{path}: unknown sampling scheme code {scheme_code}")
    if L < 1:
        raise PayloadMismatchError(f"{path}: invalid band-limit {L}")
    grid = make_grid(_CODE_SCHEME[scheme_code], L)
    expected = grid.n_theta * grid.n_phi
    if count != expected:
        raise PayloadMismatchError(
            f"{path}: payload_count {count} does not match grid ({expected} samples)"
        )
    return grid


def _flm_band(path, kind, L, count) -> int:
    if kind != _KIND_COEFFS:
        raise PayloadMismatchError(f"{path}: kind {kind} is not a coefficient set")
    if L < 1 or count != L * L:
        raise PayloadMismatchError(f"{path}: payload_count {count} does not match band-limit {L}")
    return L


# ---------------------------------------------------------------- host containers
def write_map(path, smap: SphereMap) -> None:
    """Serialize a map; real maps store one float per sample (mapio.py:83-93)."""
    count = smap.grid.n_theta * smap.grid.n_phi
    if count < 1:
        raise ParameterError("refusing to write an empty map")
    if smap.is_real:
        payload = np.ascontiguousarray(smap.values.real, dtype="<f8")
    else:
        payload = np.ascontiguousarray(smap.values, dtype="<c16")
    kind = _KIND_REAL_MAP if smap.is_real else _KIND_COMPLEX_MAP
    _write(path, _SCHEME_CODE[smap.grid.scheme], smap.grid.L, kind, count, not smap.is_real,
           payload.ctypes.data, False)


def write_flm(path, flm: HarmonicCoeffs) -> None:
    """Serialize a coefficient set (always complex payload; mapio.py:96-99)."""
    payload = np.ascontiguousarray(flm.coeffs, dtype="<c16")
    _write(path, 0, flm.L, _KIND_COEFFS, flm.L * flm.L, True, payload.ctypes.data, False)


def read_map(path) -> SphereMap:
    """Re-read a map, rebuilding its grid from the header (mapio.py:133-153)."""
    sc, L, kind, count = _header(path)
    grid = _map_grid(path, sc, L, kind, count)
    real = kind == _KIND_REAL_MAP
    buf = np.empty(count, dtype=np.float64 if real else np.complex128)
    _read_payload(path, count, not real, buf.ctypes.data, False)
    try:
        return SphereMap(grid, buf.astype(np.complex128).reshape(grid.sample_shape), is_real=real)
    except ParameterError as exc:
        raise PayloadMismatchError(f"{path}: invalid payload ({exc})") from exc


def read_flm(path) -> HarmonicCoeffs:
    """Re-read a coefficient set, returned unflagged (mapio.py:156-170)."""
    _, L, kind, count = _header(path)
    _flm_band(path, kind, L, count)
    buf = np.empty(count, dtype=np.complex128)
    _read_payload(path, count, True, buf.ctypes.data, False)
    return HarmonicCoeffs(L, buf, real_signal=False)


# ---------------------------------------------------------------- device tensors
def write_map_device(path, grid: GridSpec, values, is_real: bool) -> None:
    """Write a device map tensor ((n_theta, n_phi) float64 for real maps,
    complex128 otherwise) straight from HBM."""
    th = _device.torch()
    want = th.float64 if is_real else th.complex128
    if values.dtype != want or tuple(values.shape) != grid.sample_shape or not values.is_cuda:
        raise ParameterError(f"expected a {want} CUDA tensor of shape {grid.sample_shape}")
    v = values.contiguous()
    kind = _KIND_REAL_MAP if is_real else _KIND_COMPLEX_MAP
    _write(path, _SCHEME_CODE[grid.scheme], grid.L, kind, grid.n_theta * grid.n_phi, not is_real,
           _device.ptr(v), True)


def read_map_device(path):
    """(grid, device tensor, is_real) of an S2WM map file."""
    th = _device.torch()
    sc, L, kind, count = _header(path)
    grid = _map_grid(path, sc, L, kind, count)
    real = kind == _KIND_REAL_MAP
    out = th.empty(grid.sample_shape, dtype=th.float64 if real else th.complex128,
                   device=f"cuda:{_device.device_index()}")
    _read_payload(path, count, not real, _device.ptr(out), True)
    if grid.scheme is SamplingScheme.MW and not bool(th.all(out[-1] == out[-1, 0])):
        raise PayloadMismatchError(f"{path}: invalid payload (MW pole ring must carry identical values)")
    return grid, out, real


def write_flm_device(path, flm_tensor, L: int) -> None:
    """Write a device coefficient tensor (L*L complex128)."""
    th = _device.torch()
    if flm_tensor.dtype != th.complex128 or flm_tensor.numel() != L * L or not flm_tensor.is_cuda:
        raise ParameterError(f"expected a complex128 CUDA tensor of {L * L} coefficients")
    _write(path, 0, L, _KIND_COEFFS, L * L, True, _device.ptr(flm_tensor.contiguous()), True)


def read_flm_device(path):
    """(L, device complex128 tensor of L*L coefficients)."""
    th = _device.torch()
    _, L, kind, count = _header(path)
    _flm_band(path, kind, L, count)
    out = th.empty(count, dtype=th.complex128, device=f"cuda:{_device.device_index()}")
    _read_payload(path, count, True, _device.ptr(out), True)
    return L, out
