"""Host-side logic of the drop-in (no GPU): grids, containers, tiling, errors.

Mirrors the reference's own tests for these types (test_grid.py, test_tiling.py,
test_sht.py:311-333, test_transform.py:237-248) against golden tables.
"""
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1211_1680_b200 as sw
from conftest import rel_err

GL, MW = sw.SamplingScheme.GL, sw.SamplingScheme.MW


def test_mw_grid_layout():
    g = sw.make_grid(MW, 4)
    assert (g.n_theta, g.n_phi) == (4, 7)
    assert g.theta_nodes[0] == pytest.approx(math.pi / 7)
    assert g.theta_nodes[-1] == pytest.approx(math.pi)
    assert g.quad_weights is None
    assert sw.distinct_sample_count(sw.make_grid(MW, 128)) == 32386
    assert sw.distinct_sample_count(sw.make_grid(MW, 1)) == 1
    assert sw.distinct_sample_count(sw.make_grid(GL, 4)) == 28


@pytest.mark.parametrize("L", [1, 2, 3, 8, 64, 257])
def test_gl_grid(L):
    g = sw.make_grid(GL, L)
    x, w = np.polynomial.legendre.leggauss(L)
    assert np.abs(np.cos(g.theta_nodes) - x[::-1]).max() <= 1e-14
    assert abs(g.quad_weights.sum() - 2.0) <= 1e-13
    assert np.all(np.diff(g.theta_nodes) > 0)
    n = np.arange(2 * L)
    # exactness: sum w P_n(x) = int P_n
    for k in range(0, 2 * L, max(1, L // 4)):
        pk = np.polynomial.legendre.legval(np.cos(g.theta_nodes), np.eye(2 * L)[k])
        assert abs(np.sum(g.quad_weights * pk) - (2.0 if k == 0 else 0.0)) <= 1e-12


def test_grid_validation():
    with pytest.raises(sw.ParameterError):
        sw.make_grid(GL, 0)
    with pytest.raises(sw.ParameterError):
        sw.make_grid(GL, 2.5)
    with pytest.raises(sw.ParameterError):
        sw.make_grid("gl", 4)
    assert sw.make_grid(GL, 8) is sw.make_grid(GL, 8)
    assert sw.make_grid(GL, 8) == sw.make_grid(GL, 8)
    assert sw.make_grid(GL, 8) != sw.make_grid(MW, 8)


def test_sphere_map_invariants():
    g = sw.make_grid(MW, 4)
    v = np.ones(g.sample_shape, complex)
    sw.SphereMap(g, v, is_real=True)
    bad = v.copy()
    bad[0, 0] += 1e-300j
    with pytest.raises(sw.ParameterError):
        sw.SphereMap(g, bad, is_real=True)
    pole = v.copy()
    pole[-1, 3] = 2.0
    with pytest.raises(sw.ParameterError):
        sw.SphereMap(g, pole)
    with pytest.raises(sw.ParameterError):
        sw.SphereMap(g, np.ones((3, 7)))
    assert not sw.map_constant(g, 1j).is_real


def test_coefficient_container(rng):
    with pytest.raises(sw.ParameterError):
        sw.HarmonicCoeffs(3, np.zeros(5, complex))
    bad = np.zeros(4, complex)
    bad[sw.lm_index(1, 1)] = 1.0
    with pytest.raises(sw.ParameterError):
        sw.HarmonicCoeffs(2, bad, real_signal=True)
    c = sw.HarmonicCoeffs.zeros(3)
    assert c[2, -2] == 0.0
    with pytest.raises(sw.ParameterError):
        c[3, 0]
    f = sw.gaussian_coeffs(5, rng, real_signal=True)
    p = sw.pad_coeffs(f, 9)
    assert p.L == 9 and p.real_signal
    assert np.array_equal(sw.truncate_coeffs(p, 5).coeffs, f.coeffs)
    with pytest.raises(sw.ParameterError):
        sw.pad_coeffs(f, 3)
    with pytest.raises(sw.ParameterError):
        sw.truncate_coeffs(f, 8)


def test_gaussian_coeffs_bitwise_match_reference(golden):
    """Same seeds give the reference's inputs bit for bit (bench.py:54-72)."""
    g = golden("sht_small")
    for L in (2, 5, 33, 64):
        for real in (True, False):
            seed = 100 + 2 * L + int(real)
            f = sw.gaussian_coeffs(L, np.random.default_rng(seed), real_signal=real)
            assert np.array_equal(f.coeffs, g[f"f_L{L}_{'r' if real else 'c'}"])


def test_kernels_match_reference(golden):
    g = golden("kernels")
    for key in g:
        if not key.startswith("phi_"):
            continue
        tag = key[4:]
        fam, L, lam, j0 = tag.rsplit("_", 3)
        k = sw.build_kernels(sw.TilingParams(int(L), float(lam), int(j0)),
                             getattr(sw.KernelFamily, fam))
        tol = 1e-12 if fam == "BSPLINE" else 1e-15
        assert np.abs(k.phi - g[key]).max() <= tol
        assert np.abs(k.psi - g[f"psi_{tag}"]).max() <= tol
        assert [k.scaling_bandlimit, *k.scale_bandlimits] == list(g[f"bands_{tag}"])
        assert sw.admissibility_residual(k) <= (1e-8 if fam == "NEEDLET" else 1e-10)


def test_tiling_params_and_jmax():
    assert sw.j_max(128, 3.0) == 5
    assert sw.j_max(2, 2.0) == 0
    assert sw.j_max(1024, 2.0) == 10
    assert sw.j_max(1025, 2.0) == 10
    with pytest.raises(sw.ParameterError):
        sw.j_max(1, 2.0)
    with pytest.raises(sw.ParameterError):
        sw.j_max(16, 1.0)
    with pytest.raises(sw.ParameterError):
        sw.TransformConfig(128, 3.0, 7)
    with pytest.raises(sw.ParameterError):
        sw.TransformConfig(2, 2.0, 0)
    cfg = sw.TransformConfig(128, 3.0, 2)
    assert cfg.tiling.n_scales == 4
    a = sw.kernels_for(sw.TransformConfig(32, 2.0, 0))
    assert a is sw.kernels_for(sw.TransformConfig(32, 2.0, 0, multires=False))


def test_decomposition_validation():
    cfg = sw.TransformConfig(16, 2.0, 0, scheme=MW)
    kern = sw.kernels_for(cfg)
    grids = [sw.make_grid(MW, k) for k in [kern.scaling_bandlimit, *kern.scale_bandlimits]]
    maps = [sw.map_constant(g, 0.0) for g in grids]
    sw.WaveletDecomposition(cfg, maps[0], tuple(maps[1:]))
    with pytest.raises(sw.ParameterError):
        sw.WaveletDecomposition(cfg, maps[0], tuple(maps[1:-1]))
    with pytest.raises(sw.ParameterError):
        sw.WaveletDecomposition(sw.TransformConfig(16, 2.0, 0, scheme=MW, multires=False),
                                maps[0], tuple(maps[1:]))


def test_error_hierarchy():
    assert issubclass(sw.ParameterError, sw.SphwavError)
    assert issubclass(sw.ParameterError, ValueError)
    assert issubclass(sw.FormatError, sw.SphwavError)


# ---------------------------------------------------------------- denoise host logic
def test_noise_model_matches_reference(golden):
    g = golden("denoise")
    for name in ("r32", "c24"):
        L, lam, j0, real, sigma = g[f"params_{name}"]
        cfg = sw.TransformConfig(int(L), lam, int(j0), scheme=sw.SamplingScheme.GL, multires=True)
        model = sw.make_noise_model(sigma, sw.kernels_for(cfg), 3.0)
        assert np.allclose(model.sigma_scales, g[f"sigma_scales_{name}"], rtol=1e-14, atol=0)
        assert np.allclose(model.thresholds, 3.0 * g[f"sigma_scales_{name}"], rtol=1e-14, atol=0)
    with pytest.raises(sw.ParameterError):
        sw.make_noise_model(-0.1, sw.kernels_for(sw.TransformConfig(16, 2.0, 0)))
    with pytest.raises(sw.ParameterError):
        sw.NoiseModel(-1.0, np.zeros(3))


def test_snr_db(rng):
    f = sw.gaussian_coeffs(8, rng)
    assert sw.snr_db(f, f) == math.inf
    g = sw.HarmonicCoeffs(8, f.coeffs * 1.1)
    assert abs(sw.snr_db(f, g) - 20.0) < 1e-9
    with pytest.raises(sw.ParameterError):
        sw.snr_db(f, sw.gaussian_coeffs(4, rng))
    with pytest.raises(sw.ParameterError):
        sw.snr_db(sw.HarmonicCoeffs(8, np.zeros(64, complex)), f)


def test_hard_threshold_host_semantics():
    cfg = sw.TransformConfig(16, 2.0, 0, scheme=MW)
    kern = sw.kernels_for(cfg)
    grids = [sw.make_grid(MW, k) for k in [kern.scaling_bandlimit, *kern.scale_bandlimits]]
    rng = np.random.default_rng(3)
    maps = []
    for g in grids:
        v = rng.standard_normal(g.sample_shape)
        v[-1] = v[-1, 0]  # MW pole ring holds one value
        maps.append(sw.SphereMap(g, v + 0j, is_real=True))
    dec = sw.WaveletDecomposition(cfg, maps[0], tuple(maps[1:]))
    model = sw.make_noise_model(0.5, kern, 1.0)
    out = sw.hard_threshold(dec, model)
    assert np.array_equal(out.scaling.values, dec.scaling.values)
    for a, b, t in zip(dec.wavelets, out.wavelets, model.thresholds):
        assert np.array_equal(b.values, np.where(np.abs(a.values) < t, 0, a.values))
    bad = sw.NoiseModel(0.5, model.sigma_scales[:-1])
    with pytest.raises(sw.ParameterError):
        sw.hard_threshold(dec, bad)
