"""GPU parity of the wavelet path against reference golden vectors."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10

CASES = {
    "c1": (64, 2.0, 0, False, False),
    "c2s": (64, 2.0, 2, True, True),
    "gl32": (32, 2.0, 0, True, True),
    "gl32full": (32, 3.0, 1, False, False),
}


@pytest.fixture(scope="module")
def sw():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as m

    return m


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("scheme", ["GL", "MW"])
def test_wavelet_maps_and_round_trip(sw, golden, name, scheme):
    L, lam, j0, multires, real = CASES[name]
    g = golden("wavelet")
    f = sw.HarmonicCoeffs(L, g[f"f_{name}"], real_signal=real)
    sch = getattr(sw.SamplingScheme, scheme)
    cfg = sw.TransformConfig(L, lam, j0, scheme=sch, multires=multires)
    smap = sw.sh_synthesis(f, sw.make_grid(sch, L))
    dec = sw.wav_analysis_pixel(smap, cfg)
    maps = [dec.scaling, *dec.wavelets]
    tag = f"{name}_{scheme.lower()}"
    for j, m in enumerate(maps):
        assert rel_err(m.values, g[f"scale{j}_{tag}"]) <= TOL, j
        assert m.is_real == real
        if scheme == "GL":
            assert rel_err(m.values, g[f"pix{j}_{tag}"]) <= TOL
    rec = sw.wav_synthesis_pixel(dec)
    assert rec.is_real == real
    back = sw.sh_analysis(rec)
    assert np.abs(back.coeffs - f.coeffs).max() <= 1e-10
    if scheme == "GL":
        assert rel_err(rec.values, g[f"rec_{tag}"]) <= TOL


def test_harmonic_tiling(sw, rng):
    L = 64
    kern = sw.kernels_for(sw.TransformConfig(L, 2.0, 0))
    f = sw.gaussian_coeffs(L, rng, real_signal=True)
    for trunc in (False, True):
        wc = sw.wav_analysis_harmonic(f, kern, truncate=trunc)
        ell = np.arange(L)
        for s, K in zip([wc.scaling, *wc.wavelets], [kern.phi, *kern.psi]):
            w = np.repeat(np.sqrt(4 * np.pi / (2 * ell + 1)) * K, 2 * ell + 1)
            assert np.array_equal(s.coeffs, (f.coeffs * w)[: s.L * s.L])
            assert s.real_signal
        rec = sw.wav_synthesis_harmonic(wc, kern)
        assert np.abs(rec.coeffs - f.coeffs).max() <= 1e-10


def test_batch_matches_single(sw):
    L = 48
    rng = np.random.default_rng(5)
    cfg = sw.TransformConfig(L, 2.0, 1, scheme=sw.SamplingScheme.MW, multires=True)
    grid = sw.make_grid(sw.SamplingScheme.MW, L)
    maps = [sw.sh_synthesis(sw.gaussian_coeffs(L, rng, real_signal=False), grid) for _ in range(3)]
    decs = sw.wav_analysis_pixel_batch(maps, cfg)
    for m, d in zip(maps, decs):
        single = sw.wav_analysis_pixel(m, cfg)
        for a, b in zip([d.scaling, *d.wavelets], [single.scaling, *single.wavelets]):
            assert rel_err(a.values, b.values) <= 1e-13
    recs = sw.wav_synthesis_pixel_batch(decs)
    for m, r in zip(maps, recs):
        assert rel_err(r.values, m.values) <= 1e-10


def test_round_trip_stream_matches_round_trip(sw):
    import torch

    from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform

    L = 64
    cfg = sw.TransformConfig(L, 2.0, 1, scheme=sw.SamplingScheme.MW, multires=True)
    wt = WaveletTransform(cfg, batch=2, real=False)
    rng = np.random.default_rng(8)
    sht = SphericalHarmonicTransform(sw.SamplingScheme.MW, L)
    ins = []
    for i in range(5):
        f = np.stack([sw.gaussian_coeffs(L, rng, real_signal=False).coeffs for _ in range(2)])
        ins.append(sht.synthesis(torch.from_numpy(f).cuda()).cpu().pin_memory())
    outs = [torch.empty_like(t).pin_memory() for t in ins]
    wt.round_trip_stream(ins, outs)
    torch.cuda.synchronize()
    for a, b in zip(ins, outs):
        want = wt.round_trip(a.cuda()).cpu()
        assert torch.equal(b, want)


def test_round_trip_graph_matches_eager(sw):
    import torch

    from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform

    L = 48
    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.MW, multires=True)
    wt = WaveletTransform(cfg, batch=1, real=True)
    f = sw.gaussian_coeffs(L, np.random.default_rng(12), real_signal=True)
    sht = SphericalHarmonicTransform(sw.SamplingScheme.MW, L)
    x = sht.synthesis(torch.from_numpy(f.coeffs[None].copy()).cuda(), real=True)
    scale = wt.alloc_scale_maps()
    out = torch.empty_like(x)
    want = wt.round_trip(x, wt.alloc_scale_maps(), torch.empty_like(x)).clone()
    for _ in range(3):
        wt.round_trip_graph(x, scale, out)
        torch.cuda.synchronize()
        assert torch.equal(out, want)
    x.mul_(2.0)  # replays read the buffers' current contents
    wt.round_trip_graph(x, scale, out)
    torch.cuda.synchronize()
    assert torch.allclose(out, 2.0 * want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("L,real", [(128, False), (96, True)])
def test_concurrent_scales_bit_identical(sw, rng, L, real):
    """Per-scale ring stages on forked side streams (default) give the same
    bits as the serial order, for both directions and for CUDA-graph replay."""
    import torch

    from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform

    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.MW, multires=True)
    f = sw.gaussian_coeffs(L, rng, real_signal=real).coeffs[None]
    x = SphericalHarmonicTransform(sw.SamplingScheme.MW, L).synthesis(
        torch.from_numpy(f).cuda(), real=real)
    wt = WaveletTransform(cfg, batch=1, real=real)
    outs = {}
    for on in (True, False):
        wt.set_concurrency(on)
        maps = wt.analysis(x)
        rec = wt.synthesis(maps)
        torch.cuda.synchronize()
        outs[on] = ([m.clone() for m in maps], rec.clone())
    for a, b in zip(outs[True][0], outs[False][0]):
        assert torch.equal(a, b)
    assert torch.equal(outs[True][1], outs[False][1])
    wt.set_concurrency(True)
    scale = wt.alloc_scale_maps()
    out = torch.empty_like(x)
    for _ in range(2):
        g = wt.round_trip_graph(x, scale, out)
    torch.cuda.synchronize()
    assert torch.equal(g, outs[False][1])


def test_results_in_page_locked_arrays(sw, monkeypatch):
    """Result arrays come from the pinned-host pool (same values as the
    pageable path, S2W_PINNED_RESULT_MB = 0), outlive the call that made them
    and are not overwritten by later calls."""
    import torch

    from paper_1211_1680_b200 import _device

    L = 48
    rng = np.random.default_rng(7)
    f = sw.gaussian_coeffs(L, rng, real_signal=False)
    cfg = sw.TransformConfig(L, 2.0, 1, scheme=sw.SamplingScheme.MW, multires=True)
    smap = sw.sh_synthesis(f, sw.make_grid(sw.SamplingScheme.MW, L))
    assert torch.from_numpy(np.asarray(smap.values)).is_pinned()
    dec = sw.wav_analysis_pixel(smap, cfg)
    kept = [np.array(m.values) for m in (dec.scaling, *dec.wavelets)]
    assert all(torch.from_numpy(np.asarray(m.values)).is_pinned() for m in dec.wavelets)
    # later calls reuse freed blocks only: the maps still held keep their values
    for _ in range(3):
        back = sw.wav_synthesis_pixel(sw.wav_analysis_pixel(smap, cfg))
    for m, k in zip((dec.scaling, *dec.wavelets), kept):
        assert np.array_equal(m.values, k)
    assert rel_err(back.values, smap.values) < TOL
    monkeypatch.setattr(_device, "_PINNED_CAP", 0)
    dec0 = sw.wav_analysis_pixel(smap, cfg)
    assert not torch.from_numpy(np.asarray(dec0.scaling.values)).is_pinned()
    for m, m0 in zip((dec.scaling, *dec.wavelets), (dec0.scaling, *dec0.wavelets)):
        assert np.array_equal(m.values, m0.values)
