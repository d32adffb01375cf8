"""GPU parity of the SHT path against reference golden vectors.

Golden maps were produced by the reference's own sh_synthesis / sh_analysis
(tests/golden/make_golden.py).  Tolerance: 1e-10 normwise relative (the
north-star bar), plus the reference's own KAT tolerances where stricter.
"""
import math

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-10
LS = (1, 2, 4, 5, 7, 8, 16, 24, 33, 64)


@pytest.fixture(scope="module")
def sw():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as m

    return m


def coeffs(sw, g, L, real):
    tag = f"L{L}_{'r' if real else 'c'}"
    return sw.HarmonicCoeffs(L, g(f"sht_small")[f"f_{tag}"], real_signal=real), tag


@pytest.mark.parametrize("L", LS)
@pytest.mark.parametrize("real", [True, False])
@pytest.mark.parametrize("scheme", ["GL", "MW"])
def test_synthesis_matches_reference(sw, golden, L, real, scheme):
    f, tag = coeffs(sw, golden, L, real)
    grid = sw.make_grid(getattr(sw.SamplingScheme, scheme), L)
    m = sw.sh_synthesis(f, grid)
    ref = golden("sht_small")[f"{scheme.lower()}_map_{tag}"]
    assert rel_err(m.values, ref) <= TOL
    assert m.is_real == real
    if real:
        assert np.all(m.values.imag == 0.0)
    if scheme == "MW":
        assert np.all(m.values[-1] == m.values[-1, 0])


@pytest.mark.parametrize("L", LS)
@pytest.mark.parametrize("real", [True, False])
def test_gl_analysis_matches_reference(sw, golden, L, real):
    f, tag = coeffs(sw, golden, L, real)
    grid = sw.make_grid(sw.SamplingScheme.GL, L)
    smap = sw.SphereMap(grid, golden("sht_small")[f"gl_map_{tag}"], is_real=real)
    out = sw.sh_analysis(smap)
    assert rel_err(out.coeffs, golden("sht_small")[f"gl_ana_{tag}"]) <= TOL
    assert np.abs(out.coeffs - f.coeffs).max() <= 1e-10
    assert out.real_signal == real


@pytest.mark.parametrize("L", LS)
@pytest.mark.parametrize("real", [True, False])
def test_mw_analysis_recovers_reference_coefficients(sw, golden, L, real):
    """MW forward transform (absent in the reference): analysing the reference's
    own MW synthesis must return the seeded f_lm."""
    f, tag = coeffs(sw, golden, L, real)
    grid = sw.make_grid(sw.SamplingScheme.MW, L)
    smap = sw.SphereMap(grid, golden("sht_small")[f"mw_map_{tag}"], is_real=real)
    out = sw.sh_analysis(smap)
    assert np.abs(out.coeffs - f.coeffs).max() <= 1e-10
    assert out.real_signal == real


def test_upsampled_synthesis(sw, golden):
    g = golden("sht_small")
    f = sw.HarmonicCoeffs(6, g["f_up6"], real_signal=True)
    for scheme in ("GL", "MW"):
        m = sw.sh_synthesis(f, sw.make_grid(getattr(sw.SamplingScheme, scheme), 13))
        assert rel_err(m.values, g[f"{scheme.lower()}_map_up6_13"]) <= TOL
        back = sw.truncate_coeffs(sw.sh_analysis(m), 6)
        assert np.abs(back.coeffs - f.coeffs).max() <= 1e-12


def test_constant_and_closed_forms(sw):
    L = 4
    c = np.zeros(L * L, complex)
    c[0] = math.sqrt(4 * math.pi)
    for scheme in (sw.SamplingScheme.GL, sw.SamplingScheme.MW):
        m = sw.sh_synthesis(sw.HarmonicCoeffs(L, c, real_signal=True), sw.make_grid(scheme, L))
        np.testing.assert_allclose(m.values.real, 1.0, atol=1e-14)
        flm = sw.sh_analysis(sw.map_constant(sw.make_grid(scheme, 8), 1.0))
        assert abs(flm.coeffs[0] - math.sqrt(4 * math.pi)) <= 1e-13
        assert np.abs(flm.coeffs[1:]).max() <= 1e-12
    # Y21 closed form (test_sht.py:46-51 KAT)
    grid = sw.make_grid(sw.SamplingScheme.GL, 4)
    d = np.zeros(16, complex)
    d[sw.lm_index(2, 1)] = 1.0
    m = sw.sh_synthesis(sw.HarmonicCoeffs(4, d), grid)
    th, ph = np.meshgrid(grid.theta_nodes, grid.phis, indexing="ij")
    y21 = -math.sqrt(15 / (8 * math.pi)) * np.sin(th) * np.cos(th) * np.exp(1j * ph)
    assert np.abs(m.values - y21).max() <= 1e-14


@pytest.mark.parametrize("scheme", ["GL", "MW"])
@pytest.mark.parametrize("real", [True, False])
@pytest.mark.parametrize("L", [2, 3, 7, 32, 100, 128, 256])
def test_round_trip(sw, scheme, real, L):
    rng = np.random.default_rng(L + 17 * real)
    f = sw.gaussian_coeffs(L, rng, real_signal=real)
    grid = sw.make_grid(getattr(sw.SamplingScheme, scheme), L)
    rec = sw.sh_analysis(sw.sh_synthesis(f, grid))
    assert np.abs(rec.coeffs - f.coeffs).max() <= 1e-10
    assert rec.real_signal == real


def test_stack_matches_single(sw):
    rng = np.random.default_rng(3)
    grid = sw.make_grid(sw.SamplingScheme.MW, 40)
    fs = [sw.gaussian_coeffs(40, rng, real_signal=False) for _ in range(5)]
    maps = sw.sh_synthesis_stack(fs, grid)
    for f, m in zip(fs, maps):
        assert np.array_equal(m.values, sw.sh_synthesis(f, grid).values)
    outs = sw.sh_analysis_stack(maps)
    for f, o in zip(fs, outs):
        assert np.abs(o.coeffs - f.coeffs).max() <= 1e-11


def test_deterministic(sw):
    rng = np.random.default_rng(9)
    f = sw.gaussian_coeffs(96, rng, real_signal=False)
    grid = sw.make_grid(sw.SamplingScheme.MW, 96)
    a = sw.sh_analysis(sw.sh_synthesis(f, grid)).coeffs
    b = sw.sh_analysis(sw.sh_synthesis(f, grid)).coeffs
    assert np.array_equal(a, b)


def test_legendre_ring(sw, golden):
    g = golden("legendre")
    assert rel_err(sw.assoc_legendre_ring(16, 1.0), g["ring_L16_t1"]) <= 1e-13
    assert rel_err(sw.assoc_legendre_ring(40, 0.3), g["ring_L40_t03"]) <= 1e-13
    assert rel_err(sw.assoc_legendre_ring(1536, 0.7)[::97], g["ring_L1536_t07_rows"]) <= 1e-12
    big = sw.assoc_legendre_ring(4096, 0.7)
    assert np.all(np.isfinite(big))
    assert np.abs(big).max() <= math.sqrt((2 * 4096 - 1) / (4 * math.pi)) * 1.01


@pytest.mark.parametrize("scheme", ["GL", "MW"])
@pytest.mark.parametrize("real", [True, False])
@pytest.mark.parametrize("L", [700, 1100])
def test_multi_window_multi_pass_vs_oracle(sw, scheme, real, L):
    """Band-limits that need several shared-memory windows and ring passes."""
    from oracle import oracle as orc

    rng = np.random.default_rng(L + real)
    f = sw.gaussian_coeffs(L, rng, real_signal=real)
    grid = sw.make_grid(getattr(sw.SamplingScheme, scheme), L)
    m = sw.sh_synthesis(f, grid)
    orders = np.array([0, 1, 5, L // 3, L // 2, L - 2, L - 1], dtype=np.int32)
    G = orc.legendre_synth(f.coeffs[None], L, real, scheme.lower(), orders=orders)
    # compare the ring Fourier modes of our map at the sampled orders
    F = np.fft.fft(m.values, axis=1) if not real else np.fft.rfft(m.values.real, axis=1)
    Fo = orc.rings_forward(orc.rings_inverse(G, L, real, scheme.lower()), L, real)[0].T
    scale = np.abs(F).max()
    N = 2 * L - 1
    for mm in orders:
        if scheme == "MW":
            got, want = F[:-1, mm] / N, Fo[:-1, mm]   # pole ring is pinned
        else:
            got, want = F[:, mm] / N, Fo[:, mm]
        assert np.abs(got - want).max() <= 1e-10 * scale / N
    rec = sw.sh_analysis(m)
    assert np.abs(rec.coeffs - f.coeffs).max() <= 1e-10


@pytest.mark.parametrize("scheme", ["GL", "MW"])
@pytest.mark.parametrize("real,L", [(False, 2049), (True, 3001), (True, 4096), (False, 4096)])
def test_split_fft_sizes_round_trip(sw, scheme, real, L):
    """L > 2048 uses the split (two half-length) FFT convolutions: M = 16384."""
    import torch
    from paper_1211_1680_b200.device import SphericalHarmonicTransform

    rng = np.random.default_rng(L)
    f = sw.gaussian_coeffs(L, rng, real_signal=real).coeffs
    sht = SphericalHarmonicTransform(getattr(sw.SamplingScheme, scheme), L)
    x = sht.synthesis(torch.from_numpy(f[None].copy()).cuda(), real=real)
    back = sht.analysis(x).cpu().numpy()[0]
    assert np.abs(back - f).max() <= 2e-10 * max(1.0, np.abs(f).max())


@pytest.mark.parametrize("scheme", ["GL", "MW"])
@pytest.mark.parametrize("real", [True, False])
def test_round_trip_L2048_pfa(sw, scheme, real):
    """L = 2048 (N = 4095): ring DFTs and MW theta stages on the prime-factor engine."""
    import torch
    from paper_1211_1680_b200.device import SphericalHarmonicTransform

    L = 2048
    f = sw.gaussian_coeffs(L, np.random.default_rng(5 + real), real_signal=real).coeffs
    sht = SphericalHarmonicTransform(getattr(sw.SamplingScheme, scheme), L)
    x = sht.synthesis(torch.from_numpy(f[None].copy()).cuda(), real=real)
    back = sht.analysis(x).cpu().numpy()[0]
    assert np.abs(back - f).max() <= 1e-10 * max(1.0, np.abs(f).max())


@pytest.mark.parametrize("real", [False, True])
def test_round_trip_L2048_batch2(sw, real):
    """Two maps per call at L = 2048: the k2 stage kernels over several sets
    (rows of set 1 follow set 0) and the batched Legendre kernels."""
    import torch
    from paper_1211_1680_b200.device import SphericalHarmonicTransform

    L = 2048
    f = np.stack([sw.gaussian_coeffs(L, np.random.default_rng(40 + b), real_signal=real).coeffs
                  for b in range(2)])
    sht = SphericalHarmonicTransform(sw.SamplingScheme.MW, L)
    x = sht.synthesis(torch.from_numpy(f).cuda(), real=real)
    one = sht.synthesis(torch.from_numpy(f[1:].copy()).cuda(), real=real)
    assert torch.equal(x[1:], one)  # set 1 does not depend on set 0
    back = sht.analysis(x).cpu().numpy()
    assert np.abs(back - f).max() <= 1e-10 * max(1.0, np.abs(f).max())


def test_pipelined_analysis_matches_default():
    """The opt-in pipelined analysis kernel (S2W_ANA_PIPE=1: lanes own degree
    blocks, rings stream through the warp) against the default reduce-scatter
    kernel on the same map, complex and real, including the polar rings'
    scaled-exponent hand-off between passes (L = 600: 3 degree passes)."""
    import os

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as sw
    from paper_1211_1680_b200 import _device
    from paper_1211_1680_b200.device import SphericalHarmonicTransform

    L = 600
    for real in (False, True):
        f = sw.gaussian_coeffs(L, np.random.default_rng(600 + real), real_signal=real).coeffs
        sht = SphericalHarmonicTransform(sw.SamplingScheme.MW, L)
        x = sht.synthesis(torch.from_numpy(f[None].copy()).cuda(), real=real)
        ref = sht.analysis(x).cpu().numpy()
        os.environ["S2W_ANA_PIPE"] = "1"
        try:
            with _device._lock:
                _device._sht_plans.clear()   # a fresh plan builds its launch with the switch on
            got = SphericalHarmonicTransform(sw.SamplingScheme.MW, L).analysis(x).cpu().numpy()
        finally:
            del os.environ["S2W_ANA_PIPE"]
            with _device._lock:
                _device._sht_plans.clear()
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.abs(got - f).max() <= 1e-10 * np.abs(f).max()


@pytest.mark.parametrize("l0,m0", [(2040, 900), (1200, 64), (2047, 2000), (1500, 33)])
def test_terms_left_out_stay_below_the_threshold(sw, l0, m0):
    """The Legendre kernels hold a ring out of the sums until its column can
    pass 2^-80 before the ring is looked at again (ring_fix,
    csrc/legendre_kernels.cu; the reference flushes at 1e-280, sht.py:179-184).
    One unit coefficient makes every ring's Fourier mode a single term
    P_lm(theta_t): where the device holds the term back the oracle's value must
    lie below that level; everywhere else the two agree, the tiny polar values
    to 1e-8 of themselves.  GL grid: no theta resampling between the Legendre
    sums and the rings."""
    from oracle import oracle as orc

    L = 2048
    f = np.zeros(L * L, dtype=np.complex128)
    f[l0 * l0 + l0 + m0] = 1.0
    grid = sw.make_grid(sw.SamplingScheme.GL, L)
    smap = sw.sh_synthesis(sw.HarmonicCoeffs(L, f, real_signal=False), grid)
    got = np.fft.fft(np.asarray(smap.values), axis=1)[:, m0] / (2 * L - 1)
    want = orc.legendre_synth(f[None], L, False, "gl", orders=[m0])[0][:, m0]
    err = np.abs(got - want)
    # small values keep their own relative accuracy (1e-8 of themselves, down to
    # the threshold); near the zero crossings the error is relative to the column
    assert np.all(err <= 1e-8 * np.abs(want) + 1e-13 * np.abs(want).max() + 2.0 ** -78)
    assert rel_err(got, want) < TOL
    held = got == 0.0
    if held.any():
        assert np.abs(want[held]).max() < 2.0 ** -80
    # a column that has not passed 2^-400 cannot reach 2^-80 within a chunk
    # (growth < 2^8 per degree): those rings are held back, exact zeros, which
    # includes rings round 1's 2^-600 level would have summed
    assert np.all(held[np.abs(want) < 2.0 ** -400])
