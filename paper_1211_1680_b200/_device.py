"""Device plumbing: torch CUDA tensors, streams and cached C-ABI plans.

PyTorch provides device memory, pinned staging buffers and the current CUDA
stream; all arithmetic on the hot path happens in libs2w.so kernels.
"""
from __future__ import annotations

import ctypes
import os
import threading
import warnings

import numpy as np

from . import _native
from .errors import SphwavError

_lock = threading.Lock()
_sht_plans: dict = {}
_wav_plans: dict = {}


def torch():
    import torch as _t

    return _t


def require_cuda() -> None:
    t = torch()
    if not t.cuda.is_available():
        raise SphwavError(
            "s2w requires a CUDA device (B200, sm_100a); there is no CPU fallback"
        )
    _native.load()


def device_index() -> int:
    return torch().cuda.current_device()


def stream_handle():
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(tensor.data_ptr())


def to_device(arr: np.ndarray):
    """Host numpy -> CUDA tensor.  Pageable source: the driver stages it (a
    per-call pin_memory() allocation costs more than it saves)."""
    t = torch()
    arr = np.require(arr, requirements=["C"])
    with warnings.catch_warnings():
        # read-only inputs (SphereMap values) are only read by the copy
        warnings.simplefilter("ignore", UserWarning)
        host = t.from_numpy(arr)
    return host.to(device=f"cuda:{device_index()}")


def to_host(tensor) -> np.ndarray:
    """Device float64 tensor -> a new flat host float64 array (host_result)."""
    return host_result(tensor, np.float64)


def copy_to_host(tensor, arr: np.ndarray) -> None:
    """Device tensor -> an existing host array (same number of elements)."""
    t = torch()
    t.from_numpy(arr).copy_(tensor.reshape(-1).view(t.from_numpy(arr).dtype))


# Result arrays up to this many bytes come from torch's caching pinned-host
# allocator (S2W_PINNED_RESULT_MB, 0 disables): page-locked memory takes the
# device->host copy at PCIe rate with no driver staging and no first-touch
# page faults, and a map handed back to the next call (run_trial's
# analysis -> synthesis pair, reference bench.py:84-92) goes host->device at
# PCIe rate too.  The numpy array keeps the tensor (and so the block) alive;
# when the caller drops it the block returns to torch's pool for the next call.
_PINNED_CAP = int(float(os.environ.get("S2W_PINNED_RESULT_MB", "2048")) * (1 << 20))


def host_result(tensor, dtype) -> np.ndarray:
    """Device tensor -> a new host array of `dtype` (flat), through a
    page-locked buffer when it fits the cap, else a pageable numpy array."""
    t = torch()
    flat = tensor.reshape(-1)
    nbytes = flat.numel() * flat.element_size()
    if 0 < nbytes <= _PINNED_CAP:
        try:
            host = t.empty(flat.shape, dtype=flat.dtype, pin_memory=True)
        except RuntimeError:
            host = None  # pinned pool exhausted: fall through to pageable memory
        if host is not None:
            host.copy_(flat, non_blocking=True)
            t.cuda.current_stream().synchronize()
            return host.numpy().view(dtype)
    arr = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
    copy_to_host(flat, arr.view(np.float64) if flat.dtype == t.float64 else arr)
    return arr


def empty(n: int, dtype="float64"):
    t = torch()
    return t.empty(n, dtype=getattr(t, dtype), device=f"cuda:{device_index()}")


class ShtPlan:
    """Owner of an ``s2w_sht_plan`` (one grid on one device)."""

    def __init__(self, scheme_code: int, L: int, device: int):
        lib = _native.load()
        h = ctypes.c_void_p()
        _native.check(lib.s2w_sht_plan_create(scheme_code, L, device, ctypes.byref(h)))
        self.handle, self.L, self.device = h, L, device

    def __del__(self):
        try:
            _native.load().s2w_sht_plan_destroy(self.handle)
        except Exception:
            pass


def sht_plan(scheme_code: int, L: int) -> ShtPlan:
    key = (scheme_code, L, device_index())
    with _lock:
        p = _sht_plans.get(key)
        if p is None:
            p = ShtPlan(scheme_code, L, key[2])
            _sht_plans[key] = p
        return p


class WavPlan:
    """Owner of an ``s2w_wav_plan``: tiling factors, per-scale grids, workspaces."""

    def __init__(self, scheme_code, L, batch, real, kernels: np.ndarray, bands, device):
        lib = _native.load()
        kern = np.ascontiguousarray(kernels, dtype=np.float64)
        nk = kern.shape[0]
        bands_c = (ctypes.c_int * nk)(*[int(b) for b in bands])
        h = ctypes.c_void_p()
        _native.check(
            lib.s2w_wav_plan_create(
                scheme_code, L, batch, int(bool(real)), nk,
                kern.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), bands_c, device,
                ctypes.byref(h),
            )
        )
        self.handle, self.L, self.batch, self.real = h, L, batch, bool(real)
        self.n_kern, self.bands, self.device = nk, tuple(int(b) for b in bands), device

    def __del__(self):
        try:
            _native.load().s2w_wav_plan_destroy(self.handle)
        except Exception:
            pass


def wav_plan(scheme_code, L, batch, real, kernels, bands) -> WavPlan:
    kern = np.ascontiguousarray(kernels, dtype=np.float64)
    key = (scheme_code, L, batch, bool(real), kern.tobytes(), tuple(bands), device_index())
    with _lock:
        p = _wav_plans.get(key)
        if p is None:
            p = WavPlan(scheme_code, L, batch, real, kern, bands, key[-1])
            _wav_plans[key] = p
        return p


def ptr_array(tensors):
    arr = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    return arr
