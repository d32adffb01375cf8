"""The C-ABI library loads and exports every symbol include/s2w.h declares.

No GPU compute happens here: only host entry points are called.
"""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1211_1680_b200 import _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "s2w.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(s2w_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_all_symbols():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} missing from libs2w.so"
    assert set(syms) == set(_native.EXPORTED_SYMBOLS)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.lib_path())],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_errors():
    assert _native.version().startswith("s2w-b200")
    lib = _native.load()
    theta = np.zeros(4)
    rc = lib.s2w_grid_nodes(0, 0, theta.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), None)
    assert rc == _native.S2W_EPARAM
    assert "band-limit" in lib.s2w_last_error().decode()
    with pytest.raises(Exception) as ei:
        _native.check(rc)
    from paper_1211_1680_b200 import ParameterError

    assert isinstance(ei.value, ParameterError)


def test_grid_nodes_host_only():
    lib = _native.load()
    th = np.zeros(5)
    w = np.zeros(5)
    p = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    assert lib.s2w_grid_nodes(1, 5, p(th), p(w)) == 0
    assert np.allclose(th, (2 * np.arange(5) + 1) * np.pi / 9)
    assert np.all(w == 0)  # untouched for MW
    assert lib.s2w_grid_nodes(0, 5, p(th), p(w)) == 0
    assert abs(w.sum() - 2.0) < 1e-14
