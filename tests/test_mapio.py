"""S2WM files (reference mapio.py): byte-identity with the reference's own
writer (golden bytes from tests/golden/make_golden.py) and its error cases.
Host paths only (no GPU needed); the device variants are in test_gpu_mapio.py."""
import numpy as np
import pytest

import paper_1211_1680_b200 as sw
from paper_1211_1680_b200 import mapio


@pytest.fixture
def files(golden, tmp_path):
    g = golden("mapio")
    out = {}
    for name in ("gl_real", "mw_cplx", "flm"):
        p = tmp_path / f"{name}.s2wm"
        p.write_bytes(g[name].tobytes())
        out[name] = p
    return out, g


def test_round_trip_is_byte_identical(files, tmp_path):
    f, g = files
    for name in ("gl_real", "mw_cplx"):
        smap = sw.read_map(f[name])
        assert smap.is_real == (name == "gl_real")
        p = tmp_path / f"re_{name}.s2wm"
        sw.write_map(p, smap)
        assert p.read_bytes() == f[name].read_bytes()
    flm = sw.read_flm(f["flm"])
    assert np.array_equal(flm.coeffs, g["f_mw_cplx"])
    assert not flm.real_signal
    p = tmp_path / "re_flm.s2wm"
    sw.write_flm(p, flm)
    assert p.read_bytes() == f["flm"].read_bytes()
    assert mapio.HEADER_SIZE == 22 and mapio.MAGIC == b"S2WM" and mapio.VERSION == 1


def _patch(path, off, data):
    b = bytearray(path.read_bytes())
    b[off:off + len(data)] = data
    path.write_bytes(bytes(b))


def test_errors(files, tmp_path):
    f, _ = files
    p = tmp_path / "x.s2wm"
    p.write_bytes(b"S2WM\x01")
    with pytest.raises(mapio.TruncatedFileError):
        sw.read_map(p)
    p.write_bytes(f["gl_real"].read_bytes())
    _patch(p, 0, b"XXXX")
    with pytest.raises(mapio.NotS2wmFileError):
        sw.read_map(p)
    p.write_bytes(f["gl_real"].read_bytes())
    _patch(p, 4, (2).to_bytes(4, "little"))
    with pytest.raises(mapio.UnsupportedVersionError):
        sw.read_map(p)
    with pytest.raises(mapio.PayloadMismatchError):
        sw.read_map(f["flm"])
    with pytest.raises(mapio.PayloadMismatchError):
        sw.read_flm(f["gl_real"])
    p.write_bytes(f["gl_real"].read_bytes())
    _patch(p, 8, b"\x07")
    with pytest.raises(mapio.PayloadMismatchError):
        sw.read_map(p)
    p.write_bytes(f["gl_real"].read_bytes())
    _patch(p, 9, (0).to_bytes(4, "little"))
    with pytest.raises(mapio.PayloadMismatchError):
        sw.read_map(p)
    p.write_bytes(f["gl_real"].read_bytes())
    _patch(p, 14, (7).to_bytes(8, "little"))
    with pytest.raises(mapio.PayloadMismatchError):
        sw.read_map(p)
    p.write_bytes(f["gl_real"].read_bytes()[:-8])
    with pytest.raises(mapio.TruncatedFileError):
        sw.read_map(p)
    # MW pole ring with differing samples
    b = bytearray(f["mw_cplx"].read_bytes())
    b[-16:-8] = np.float64(12345.0).tobytes()
    p.write_bytes(bytes(b))
    with pytest.raises(mapio.PayloadMismatchError):
        sw.read_map(p)
    with pytest.raises(FileNotFoundError):
        sw.read_map(tmp_path / "missing.s2wm")
    assert issubclass(mapio.TruncatedFileError, sw.FormatError)
