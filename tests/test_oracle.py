"""Pin the CPU oracle (oracle/) against the reference package.

Golden vectors come from the reference's own public API
(tests/golden/make_golden.py); known-answer tests mirror the reference's
tests (test_sht.py:153-159 Rodrigues, test_sht.py:46-71 Y21/Y30).  Above
L ~ 1600, where the reference itself is wrong (SURVEY.md finding 2), the
oracle's extended-exponent recursion is pinned against mpmath at 50 digits
and against its own GL round trip on the orders the reference zeroes.
"""
import math

import numpy as np
import pytest

from conftest import rel_err
from oracle import oracle as orc

LS = (1, 2, 4, 5, 7, 8, 16, 24, 33, 64)


@pytest.mark.parametrize("L", LS)
@pytest.mark.parametrize("real", [True, False])
@pytest.mark.parametrize("scheme", ["gl", "mw"])
def test_oracle_sht_matches_reference(golden, L, real, scheme):
    g = golden("sht_small")
    tag = f"L{L}_{'r' if real else 'c'}"
    f = g[f"f_{tag}"]
    m = orc.sh_synthesis(f[None], L, real, scheme)[0]
    assert rel_err(m, g[f"{scheme}_map_{tag}"]) <= 1e-13
    back = orc.sh_analysis(g[f"{scheme}_map_{tag}"][None], L, real, scheme)[0]
    assert np.abs(back - f).max() <= 1e-12
    if scheme == "gl":
        assert rel_err(back, g[f"gl_ana_{tag}"]) <= 1e-13
    if real:
        assert np.all(back[np.arange(L) ** 2 + np.arange(L)].imag == 0.0)


def _rodrigues(ell, m, theta):
    """Exact-rational normalised Legendre value (independent of any recursion)."""
    from fractions import Fraction

    coeffs = [Fraction(0)] * (2 * ell + 1)
    for k in range(ell + 1):
        coeffs[2 * k] = Fraction(math.comb(ell, k)) * (-1) ** (ell - k)
    for _ in range(ell + m):
        coeffs = [Fraction(i) * coeffs[i] for i in range(1, len(coeffs))] or [Fraction(0)]
    x = Fraction(math.cos(theta))
    acc = Fraction(0)
    for c in reversed(coeffs):
        acc = acc * x + c
    acc /= Fraction(2**ell) * math.factorial(ell)
    norm = math.sqrt((2 * ell + 1) / (4 * math.pi) * math.factorial(ell - m) / math.factorial(ell + m))
    return (-1.0) ** m * math.sin(theta) ** m * float(acc) * norm


def test_oracle_legendre_known_answers(golden):
    tab = orc.legendre_table(16, 1.0)
    for ell in range(16):
        for m in range(ell + 1):
            assert abs(tab[ell, m] - _rodrigues(ell, m, 1.0)) <= 1e-12
    g = golden("legendre")
    assert rel_err(tab, g["ring_L16_t1"]) <= 1e-14
    assert rel_err(orc.legendre_table(40, 0.3), g["ring_L40_t03"]) <= 1e-13
    assert rel_err(orc.legendre_table(1536, 0.7)[::97], g["ring_L1536_t07_rows"]) <= 1e-12
    assert orc.legendre_table(2, math.pi / 2)[1, 0] == pytest.approx(0.0, abs=1e-16)
    pole = orc.legendre_table(3, 0.0)
    assert np.all(pole[1:, 1:][np.tril_indices(2)] == 0.0)


def test_oracle_legendre_high_degree_vs_mpmath():
    """Where the reference flushes to zero (L = 2048, theta = 0.38, m in [651, 830])."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 50
    L, theta = 2048, 0.38
    tab = orc.legendre_table(L, theta)
    x = mpmath.cos(mpmath.mpf(theta))
    for ell, m in [(2047, 700), (2047, 760), (2047, 830), (1900, 651), (1200, 300), (2047, 3)]:
        p = mpmath.legenp(ell, m, x, type=2)
        norm = mpmath.sqrt((2 * ell + 1) / (4 * mpmath.pi) * mpmath.factorial(ell - m)
                           / mpmath.factorial(ell + m))
        ref = float(p * norm)
        scale = math.sqrt((2 * ell + 1) / (4 * math.pi))
        assert abs(tab[ell, m] - ref) <= 1e-12 * scale, (ell, m, tab[ell, m], ref)


def test_oracle_round_trip_beyond_reference_range():
    """L = 2048 GL Legendre round trip on the orders the reference zeroes
    (sht.py:179-184 flush; the reference's own round trip gives eps = 1.13)."""
    L = 2048
    orders = np.array([0, 651, 700, 830, 1500, 2047], dtype=np.int32)
    rng = np.random.default_rng(2048)
    f = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    G = orc.legendre_synth(f[None], L, False, "gl", orders=orders)
    H = np.ascontiguousarray(np.swapaxes(G, 1, 2))
    back = orc.legendre_ana(H, L, False, "gl", orc.ring_weights("gl", L), orders=orders)[0]
    idx = np.concatenate([np.arange(m, L) ** 2 + np.arange(m, L) + s * m
                          for m in orders for s in ((1, -1) if m else (1,))])
    assert np.abs(back[idx] - f[idx]).max() <= 1e-10


@pytest.mark.parametrize("name,L,nmaps,real,spec", [
    ("C1", 64, 1, False, "flat"),
    ("C2", 256, 2, True, "cl"),
])
def test_oracle_matches_reference_at_configs(golden, name, L, nmaps, real, spec):
    import bench

    g = golden("configs")
    for b in range(nmaps):
        f = bench.seeded_coeffs(L, real, spec, 1000 + b)
        mw = orc.sh_synthesis(f[None], L, real, "mw")[0]
        idx, vals = g[f"{name}_b{b}_idx"], g[f"{name}_b{b}_vals"]
        assert rel_err(mw.reshape(-1)[idx], vals) <= 1e-12
        assert np.sum(np.abs(mw) ** 2) == pytest.approx(g[f"{name}_b{b}_norm2"][0], rel=1e-12)
        back = orc.sh_analysis(mw[None], L, real, "mw")[0]
        assert np.abs(back - f).max() <= 1e-10 * max(1.0, np.abs(f).max())


@pytest.mark.parametrize("name", ["c1", "c2s", "gl32", "gl32full"])
@pytest.mark.parametrize("scheme", ["gl", "mw"])
def test_oracle_wavelets_match_reference(golden, name, scheme):
    from paper_1211_1680_b200.tiling import KernelFamily, TilingParams, build_kernels

    L, lam, j0, multires, real = {
        "c1": (64, 2.0, 0, False, False), "c2s": (64, 2.0, 2, True, True),
        "gl32": (32, 2.0, 0, True, True), "gl32full": (32, 3.0, 1, False, False)}[name]
    g = golden("wavelet")
    f = g[f"f_{name}"]
    kern = build_kernels(TilingParams(L, lam, j0), KernelFamily.SCALE_DISCRETISED)
    bands = [kern.scaling_bandlimit, *kern.scale_bandlimits] if multires else [L] * (len(kern.psi) + 1)
    smap = orc.sh_synthesis(f[None], L, real, scheme)
    maps = orc.wav_analysis_pixel(smap, L, real, scheme, kern.table(), bands)
    for j, mj in enumerate(maps):
        # normwise relative per map; low-band scaling maps are ~1e-4 of the input
        assert rel_err(mj[0], g[f"scale{j}_{name}_{scheme}"]) <= 1e-10
    rec = orc.wav_synthesis_pixel(maps, L, real, scheme, kern.table(), bands)
    back = orc.sh_analysis(rec, L, real, scheme)[0]
    assert np.abs(back - f).max() <= 1e-10


@pytest.mark.parametrize("L,lam,j0,multires", [(64, 2.0, 0, False), (256, 2.0, 2, True),
                                               (1024, 2.0, 3, True), (2048, 3.0, 2, True),
                                               (4096, 2.0, 0, True), (128, 3.0, 2, True)])
def test_oracle_bands_match_kernel_tables(golden, L, lam, j0, multires):
    """The oracle's own band layout (reference tiling.py:58-73, 304-309) equals
    the reference's (kernels.npz) and the product's host tables."""
    from paper_1211_1680_b200.tiling import KernelFamily, TilingParams, build_kernels

    k = build_kernels(TilingParams(L, lam, j0), KernelFamily.SCALE_DISCRETISED)
    want = [k.scaling_bandlimit, *k.scale_bandlimits] if multires else [L] * (len(k.psi) + 1)
    assert orc.sd_bands(L, lam, j0, multires) == want
    tag = f"SCALE_DISCRETISED_{L}_{lam:g}_{j0}"
    g = golden("kernels")
    if multires and f"bands_{tag}" in g:
        assert orc.sd_bands(L, lam, j0, True) == list(g[f"bands_{tag}"])


def test_oracle_c2_scale_maps_match_reference(golden):
    """C2 at full size (L = 256, real, lambda = 2, J0 = 2, multires): the oracle's
    scale maps of the seeded map 0 vs the reference's (configs_wav.npz)."""
    import bench
    from paper_1211_1680_b200.tiling import KernelFamily, TilingParams, build_kernels

    g = golden("configs_wav")
    L = 256
    f = bench.seeded_coeffs(L, True, "cl", 1000)
    kern = build_kernels(TilingParams(L, 2.0, 2), KernelFamily.SCALE_DISCRETISED)
    bands = orc.sd_bands(L, 2.0, 2, True)
    assert bands == list(g["C2_bands"])
    smap = orc.sh_synthesis(f[None], L, True, "mw")
    maps = orc.wav_analysis_pixel(smap, L, True, "mw", kern.table(), bands)
    for j, m in enumerate(maps):
        v = m[0].reshape(-1)
        assert rel_err(v[g[f"C2_s{j}_idx"]], g[f"C2_s{j}_vals"]) <= 1e-10, j


def test_oracle_polar_rings_l4096_vs_mpmath():
    """The checker's long-double recursion on the first MW rings of L = 4096,
    where the double (reference) arithmetic drifts by ~1.6e-10 of the P_l
    scale (the recursion's own rounding near x = 1), vs mpmath at 40 digits."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    L = 4096
    N = 2 * L - 1
    worst_precise, worst_double = 0.0, 0.0
    for t in (0, 1, 3):
        theta = (2 * t + 1) * math.pi / N
        tab = orc.legendre_table(L, theta)
        tabd = orc.legendre_table(L, theta, precise=False)
        x = mpmath.cos(mpmath.mpf(theta))
        for ell, m in ((4095, 0), (4000, 0), (4095, 1), (2000, 0), (4095, 5)):
            p = mpmath.legenp(ell, m, x, type=2) * mpmath.sqrt(
                (2 * ell + 1) / (4 * mpmath.pi) * mpmath.factorial(ell - m) / mpmath.factorial(ell + m))
            scale = math.sqrt((2 * ell + 1) / (4 * math.pi))
            worst_precise = max(worst_precise, abs(tab[ell, m] - float(p)) / scale)
            worst_double = max(worst_double, abs(tabd[ell, m] - float(p)) / scale)
    assert worst_precise <= 1e-12
    assert worst_double > 1e-11  # the drift the checker exists to avoid
