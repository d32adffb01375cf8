"""The device API refuses malformed tensors with ParameterError before any
native call (the C ABI trusts its pointers; a wrong extent would fault the
context).  Afterwards the context must still be healthy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as sw
    from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform

    return torch, sw, SphericalHarmonicTransform, WaveletTransform


def test_sht_rejects_bad_tensors(env):
    th, sw, SHT, _ = env
    L = 16
    sht = SHT(sw.SamplingScheme.MW, L)
    dev = "cuda"
    good = th.zeros((2, L * L), dtype=th.complex128, device=dev)
    for bad in (th.zeros((2, 15), dtype=th.complex128, device=dev),       # not a square
                th.zeros((2, 17 * 17), dtype=th.complex128, device=dev),  # Lc > L
                th.zeros((2, L * L), dtype=th.float64, device=dev),       # dtype
                th.zeros((L * L,), dtype=th.complex128, device=dev)):     # rank
        with pytest.raises(sw.ParameterError):
            sht.synthesis(bad)
    m = sht.synthesis(good)
    assert m.shape == (2, L, 2 * L - 1)
    with pytest.raises(sw.ParameterError):
        sht.analysis(th.zeros((2, L, 2 * L), dtype=th.complex128, device=dev))
    with pytest.raises(sw.ParameterError):
        sht.analysis(th.zeros((2, L + 1, 2 * L - 1), dtype=th.float64, device=dev))
    # a non-contiguous input view is copied, not misread
    big = th.zeros((2, L, 2 * (2 * L - 1)), dtype=th.float64, device=dev)
    big[:, :, ::2] = 1.0
    a = sht.analysis(big[:, :, ::2])
    assert th.equal(a, sht.analysis(th.ones((2, L, 2 * L - 1), dtype=th.float64, device=dev)))
    assert float(sht.analysis(m).abs().max()) == 0.0


def test_wavelet_rejects_bad_scale_lists(env):
    th, sw, _, WT = env
    L = 32
    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.MW, multires=True)
    wt = WT(cfg, batch=1, real=False)
    x = th.zeros(wt.map_shape, dtype=th.complex128, device="cuda")
    outs = wt.analysis(x)
    with pytest.raises(sw.ParameterError):
        wt.synthesis(outs[:-1])                                   # short list
    with pytest.raises(sw.ParameterError):
        wt.synthesis([o.real.contiguous() for o in outs])         # float64 for complex
    with pytest.raises(sw.ParameterError):
        wt.analysis(x, outs=[*outs[:-1], th.zeros((1, 3, 5), dtype=th.complex128, device="cuda")])
    with pytest.raises(sw.ParameterError):
        wt.analysis(x.real.contiguous())
    with pytest.raises(sw.ParameterError):
        wt.round_trip(x, out=th.zeros((1, L, 2 * L - 1), dtype=th.float64, device="cuda"))
    with pytest.raises(sw.ParameterError):   # outputs must be contiguous (written in place)
        wide = th.zeros((1, L, 2 * (2 * L - 1)), dtype=th.complex128, device="cuda")
        wt.round_trip(x, out=wide[:, :, ::2])
    rec = wt.synthesis(outs)
    th.cuda.synchronize()
    assert float(rec.abs().max()) == 0.0


def test_round_trip_stream_outputs_ready_on_return(env):
    th, sw, _, WT = env
    L = 64
    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.MW, multires=True)
    wt = WT(cfg, batch=1, real=True)
    rng = np.random.default_rng(5)
    f = np.stack([sw.gaussian_coeffs(L, rng, real_signal=True).coeffs])
    x = sw.sh_synthesis(sw.HarmonicCoeffs(L, f[0], real_signal=True),
                        sw.make_grid(sw.SamplingScheme.MW, L)).values.real
    ins = [th.from_numpy(x[None].copy()).pin_memory() for _ in range(3)]
    outs = [th.full(wt.map_shape, np.nan, dtype=th.float64).pin_memory() for _ in range(3)]
    wt.round_trip_stream(ins, outs)
    # no synchronize here: the call itself must have completed the copies
    for o in outs:
        assert np.abs(o.numpy() - x).max() <= 1e-10 * np.abs(x).max()
