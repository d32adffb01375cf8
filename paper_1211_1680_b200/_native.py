"""ctypes binding of the sm_100a C-ABI library ``lib/libs2w.so`` (include/s2w.h).

There is no CPU fallback: importing works without a GPU (host-only entry
points such as ``s2w_grid_nodes`` are usable), but every compute entry point
requires the CUDA library and a CUDA device, and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ParameterError, SphwavError

_LIB_PATH = Path(os.environ.get("S2W_LIB") or
                 Path(__file__).resolve().parent / "lib" / "libs2w.so")

S2W_OK, S2W_EPARAM = 0, 1
SCHEME_GL, SCHEME_MW = 0, 1

_c_int, _c_double, _vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)

_PROTOS = {
    "s2w_version": (ctypes.c_char_p, []),
    "s2w_last_error": (ctypes.c_char_p, []),
    "s2w_grid_nodes": (_c_int, [_c_int, _c_int, _dp, _dp]),
    "s2w_assoc_legendre_ring": (_c_int, [_c_int, _c_double, _vp, _vp]),
    "s2w_sht_plan_create": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_vp)]),
    "s2w_sht_plan_destroy": (_c_int, [_vp]),
    "s2w_sh_synthesis": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "s2w_sh_analysis": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _vp]),
    "s2w_wav_plan_create": (
        _c_int,
        [_c_int, _c_int, _c_int, _c_int, _c_int, _dp, ctypes.POINTER(_c_int), _c_int,
         ctypes.POINTER(_vp)],
    ),
    "s2w_wav_plan_destroy": (_c_int, [_vp]),
    "s2w_wav_plan_flm": (_c_int, [_vp, ctypes.POINTER(_vp)]),
    "s2w_wav_plan_set_concurrency": (_c_int, [_vp, _c_int]),
    "s2w_wav_analysis_harmonic": (_c_int, [_vp, _c_int, _vp, ctypes.POINTER(_vp), _vp]),
    "s2w_wav_synthesis_harmonic": (_c_int, [_vp, _c_int, ctypes.POINTER(_vp), _vp, _vp]),
    "s2w_wav_analysis_pixel": (_c_int, [_vp, _vp, ctypes.POINTER(_vp), _vp]),
    "s2w_wav_synthesis_pixel": (_c_int, [_vp, ctypes.POINTER(_vp), _vp, _vp]),
    "s2w_wav_analysis_pixel_threshold": (_c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_double),
                                                  ctypes.POINTER(_vp), _vp]),
    "s2w_wav_denoise_pixel": (_c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(_vp), _vp, _vp]),
    "s2w_s2wm_read_header": (_c_int, [ctypes.c_char_p, ctypes.POINTER(_c_int),
                                      ctypes.POINTER(_c_int), ctypes.POINTER(_c_int),
                                      ctypes.POINTER(ctypes.c_longlong)]),
    "s2w_s2wm_read_payload": (_c_int, [ctypes.c_char_p, ctypes.c_longlong, _c_int, _vp, _c_int,
                                       _vp]),
    "s2w_s2wm_write": (_c_int, [ctypes.c_char_p, _c_int, _c_int, _c_int, ctypes.c_longlong, _c_int,
                                _vp, _c_int, _vp]),
    "s2w_shard_plan_create": (
        _c_int,
        [_c_int, _c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_int), _c_int, _c_int, _c_int,
         _dp, _c_int, ctypes.POINTER(_vp)],
    ),
    "s2w_shard_plan_destroy": (_c_int, [_vp]),
    "s2w_shard_bins": (_c_int, [_vp, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)]),
    "s2w_shard_rings_forward": (_c_int, [_vp, _vp, _vp, _vp]),
    "s2w_shard_rings_inverse": (_c_int, [_vp, _vp, _vp, _vp]),
    "s2w_shard_theta": (_c_int, [_vp, _vp, _vp]),
    "s2w_shard_legendre_synthesis": (_c_int, [_vp, _vp, _c_int, _c_int, _vp, _vp]),
    "s2w_shard_legendre_analysis": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp]),
    "s2w_shard_legendre_synthesis_sets": (_c_int, [_vp, _vp, _c_int, _c_int, ctypes.POINTER(_c_int),
                                                   ctypes.POINTER(_vp), _vp]),
    "s2w_shard_legendre_analysis_sets": (_c_int, [_vp, _c_int, ctypes.POINTER(_vp),
                                                  ctypes.POINTER(_c_int), _vp, _c_int, _c_int, _vp]),
    "s2w_shard_set_peers": (_c_int, [_vp, _c_int, _c_int, ctypes.POINTER(_c_int),
                                     ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)]),
    "s2w_shard_gather_rings": (_c_int, [_vp, ctypes.POINTER(_vp), _vp, _vp]),
    "s2w_shard_rings_forward_peers": (_c_int, [_vp, _vp, ctypes.POINTER(_vp), _vp]),
    "s2w_shard_push_rings": (_c_int, [_vp, _vp, ctypes.POINTER(_vp), _vp]),
    "s2w_shard_scatter_bins": (_c_int, [_vp, ctypes.POINTER(_vp), _vp, _vp]),
    "s2w_real_to_complex": (_c_int, [_vp, _vp, ctypes.c_longlong, _vp]),
    "s2w_complex_real_part": (_c_int, [_vp, _vp, ctypes.c_longlong, _vp]),
    "s2w_kernel_launches": (ctypes.c_longlong, []),
    "s2w_profile_enable": (_c_int, [_c_int]),
    "s2w_profile_read": (
        _c_int, [_c_int, _dp, ctypes.POINTER(ctypes.c_longlong), _c_int]),
    "s2w_profile_stage_name": (ctypes.c_char_p, [_c_int]),
    "s2w_fp64_peak": (_c_int, [_dp, _vp]),
    "s2w_dmma_peak": (_c_int, [_dp, _vp]),
}

EXPORTED_SYMBOLS = tuple(_PROTOS)

# stage hooks (include/s2w_testing.h), bound lazily by tests
_TEST_PROTOS = {
    "s2w_test_rings_inverse": (_c_int, [_c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "s2w_test_rings_forward": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
}

_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load() -> ctypes.CDLL:
    """Load libs2w.so (once).  Raises RuntimeError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise RuntimeError(
            f"s2w CUDA library not found at {_LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (or `make`)"
        )
    lib = ctypes.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
    for name, (res, args) in {**_PROTOS, **_TEST_PROTOS}.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    """Translate a C-ABI status into the reference's exception types."""
    if status == S2W_OK:
        return
    from . import errors as E

    msg = load().s2w_last_error().decode(errors="replace")
    if status == S2W_EPARAM:
        raise ParameterError(msg)
    fmt = {5: E.NotS2wmFileError, 6: E.UnsupportedVersionError, 7: E.TruncatedFileError,
           8: E.PayloadMismatchError}
    if status in fmt:
        raise fmt[status](msg)
    if status == 9:
        raise OSError(msg)
    raise SphwavError(f"s2w status {status}: {msg}")


def version() -> str:
    return load().s2w_version().decode()


N_STAGES = 7


def kernel_launches() -> int:
    return int(load().s2w_kernel_launches())


_profile_on = False


def profile_enable(on: bool) -> None:
    global _profile_on
    check(load().s2w_profile_enable(int(bool(on))))
    _profile_on = bool(on)


def profile_enabled() -> bool:
    return _profile_on


def profile_read(reset: bool = True) -> dict:
    """{stage: (milliseconds, launches)} accumulated since the last reset."""
    lib = load()
    ms = (ctypes.c_double * N_STAGES)()
    cnt = (ctypes.c_longlong * N_STAGES)()
    check(lib.s2w_profile_read(N_STAGES, ms, cnt, int(reset)))
    return {lib.s2w_profile_stage_name(i).decode(): (ms[i], int(cnt[i])) for i in range(N_STAGES)}


def fp64_peak_tflops(stream=None) -> float:
    v = ctypes.c_double()
    check(load().s2w_fp64_peak(ctypes.byref(v), stream))
    return v.value


def dmma_peak_tflops(stream=None) -> float:
    v = ctypes.c_double()
    check(load().s2w_dmma_peak(ctypes.byref(v), stream))
    return v.value
