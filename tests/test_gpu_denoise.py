"""Denoising (reference denoise.py) on the device: golden vectors from the
reference's own denoise_pipeline (GL), and the oracle for MW grids."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def sw():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as m

    return m


@pytest.mark.parametrize("name", ["r32", "c24"])
def test_denoise_matches_reference(sw, golden, name):
    g = golden("denoise")
    L, lam, j0, real, sigma = g[f"params_{name}"]
    L, j0, real = int(L), int(j0), bool(real)
    grid = sw.make_grid(sw.SamplingScheme.GL, L)
    noisy = sw.SphereMap(grid, g[f"noisy_{name}"], is_real=real)
    cfg = sw.TransformConfig(L, lam, j0, scheme=sw.SamplingScheme.GL, multires=True)
    out = sw.denoise_pipeline(noisy, sigma, cfg, 3.0)
    assert out.is_real == real
    assert rel_err(out.values, g[f"denoised_{name}"]) <= TOL


@pytest.mark.parametrize("real", [True, False])
def test_denoise_mw_vs_oracle(sw, real):
    from oracle import oracle as orc

    L, sigma = 32, 0.05
    rng = np.random.default_rng(9)
    f = sw.gaussian_coeffs(L, rng, real_signal=real)
    noise = sw.gaussian_coeffs(L, rng, real_signal=real)
    coeffs = f.coeffs * np.repeat(1.0 / (np.arange(L) + 1.0), 2 * np.arange(L) + 1)
    noisy_f = sw.HarmonicCoeffs(L, coeffs + sigma * noise.coeffs, real_signal=real)
    grid = sw.make_grid(sw.SamplingScheme.MW, L)
    noisy = sw.sh_synthesis(noisy_f, grid)
    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.MW, multires=True)
    kern = sw.kernels_for(cfg)
    model = sw.make_noise_model(sigma, kern, 3.0)
    bands = [kern.scaling_bandlimit, *kern.scale_bandlimits]
    # oracle: analysis, hard threshold of the wavelet maps, synthesis
    scale = orc.wav_analysis_pixel(noisy.values[None], L, real, "mw", kern.table(), bands)
    kept = [scale[0]] + [np.where(np.abs(m) < t, 0.0, m) for m, t in zip(scale[1:], model.thresholds)]
    want = orc.wav_synthesis_pixel(kept, L, real, "mw", kern.table(), bands)[0]
    got = sw.denoise_pipeline(noisy, sigma, cfg, 3.0)
    assert rel_err(got.values, want) <= TOL
    # the threshold matters here: the result differs from a plain round trip
    plain = sw.wav_synthesis_pixel(sw.wav_analysis_pixel(noisy, cfg))
    assert rel_err(got.values, plain.values) > 1e-3


def test_threshold_fused_matches_host_threshold(sw):
    L = 48
    rng = np.random.default_rng(4)
    f = sw.gaussian_coeffs(L, rng, real_signal=False)
    grid = sw.make_grid(sw.SamplingScheme.MW, L)
    noisy = sw.sh_synthesis(f, grid)
    cfg = sw.TransformConfig(L, 2.0, 1, scheme=sw.SamplingScheme.MW, multires=True)
    model = sw.make_noise_model(0.2, sw.kernels_for(cfg), 2.0)
    dec = sw.wav_analysis_pixel(noisy, cfg)
    host = sw.hard_threshold(dec, model)
    # idempotent (denoise.py:84-85)
    again = sw.hard_threshold(host, model)
    for a, b in zip(host.wavelets, again.wavelets):
        assert np.array_equal(a.values, b.values)
    got = sw.denoise_pipeline(noisy, 0.2, cfg, 2.0)
    want = sw.wav_synthesis_pixel(host)
    assert rel_err(got.values, want.values) <= TOL


def test_denoise_errors(sw):
    L = 16
    grid = sw.make_grid(sw.SamplingScheme.GL, L)
    smap = sw.sh_synthesis(sw.gaussian_coeffs(L, np.random.default_rng(1)), grid)
    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.GL)
    with pytest.raises(sw.ParameterError):
        sw.denoise_pipeline(smap, -1.0, cfg)
    with pytest.raises(sw.ParameterError):
        sw.denoise_pipeline(smap, 0.1, sw.TransformConfig(8, 2.0, 0))
