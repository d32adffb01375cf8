"""S2WM device variants: payloads between files and device tensors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sw():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as m

    return m


@pytest.mark.parametrize("L,real,scheme", [(5, False, "MW"), (6, True, "GL"), (1024, False, "MW"),
                                           (700, True, "MW")])
def test_device_map_round_trip(sw, tmp_path, L, real, scheme):
    import torch

    from paper_1211_1680_b200 import mapio

    sch = getattr(sw.SamplingScheme, scheme)
    f = sw.gaussian_coeffs(L, np.random.default_rng(L), real_signal=real)
    smap = sw.sh_synthesis(f, sw.make_grid(sch, L))
    host = tmp_path / "host.s2wm"
    sw.write_map(host, smap)
    grid, t, is_real = mapio.read_map_device(host)
    assert is_real == real and grid == smap.grid
    want = smap.values.real if real else smap.values
    assert np.array_equal(t.cpu().numpy(), want)
    dev = tmp_path / "dev.s2wm"
    mapio.write_map_device(dev, grid, t, is_real)
    assert dev.read_bytes() == host.read_bytes()   # > one 32 MB staging chunk at L = 1024
    with pytest.raises(sw.ParameterError):
        mapio.write_map_device(dev, grid, t.cpu(), is_real)


def test_device_flm_round_trip(sw, tmp_path):
    from paper_1211_1680_b200 import mapio

    f = sw.gaussian_coeffs(33, np.random.default_rng(3))
    p = tmp_path / "f.s2wm"
    sw.write_flm(p, f)
    L, t = mapio.read_flm_device(p)
    assert L == 33 and np.array_equal(t.cpu().numpy(), f.coeffs)
    q = tmp_path / "g.s2wm"
    mapio.write_flm_device(q, t, L)
    assert q.read_bytes() == p.read_bytes()
