"""Stage-level parity of the CUDA kernels (include/s2w_testing.h hooks).

phi stages against numpy's pocketfft (the reference's FFT, sht.py:266-273,
322, 335); the MW theta stage against the oracle's dense direct sums.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1211_1680_b200 import _device, _native

    return torch, _native, _device


def _run_inverse(env, scheme, L, G, real):
    torch, nat, dev = env
    n = G.shape[0]
    g = torch.from_numpy(np.ascontiguousarray(G)).cuda()
    out = torch.empty((n, L, 2 * L - 1), dtype=torch.float64 if real else torch.complex128,
                      device="cuda")
    nat.check(nat.load().s2w_test_rings_inverse(scheme, L, n, int(real), dev.ptr(g), dev.ptr(out),
                                                dev.stream_handle()))
    return out.cpu().numpy()


def _run_forward(env, scheme, L, maps, real, theta):
    torch, nat, dev = env
    n = maps.shape[0]
    x = torch.from_numpy(np.ascontiguousarray(maps.real if real else maps)).cuda()
    nb = L if real else 2 * L - 1
    out = torch.empty((n, nb, L), dtype=torch.complex128, device="cuda")
    nat.check(nat.load().s2w_test_rings_forward(scheme, L, n, int(real), int(theta), dev.ptr(x),
                                                dev.ptr(out), dev.stream_handle()))
    return out.cpu().numpy()


@pytest.mark.parametrize("L", [1, 2, 7, 64, 300, 1024, 2048])
@pytest.mark.parametrize("real", [True, False])
def test_phi_stages_vs_numpy(env, L, real):
    rng = np.random.default_rng(L)
    N = 2 * L - 1
    nb = L if real else N
    G = rng.standard_normal((2, L, nb)) + 1j * rng.standard_normal((2, L, nb))
    if real:
        G[:, :, 0] = G[:, :, 0].real
        want = np.fft.irfft(G, n=N, axis=-1, norm="forward")
    else:
        want = np.fft.ifft(G, axis=-1, norm="forward")
    got = _run_inverse(env, 0, L, G, real)  # GL: no pole pinning
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-14 * scale * max(1.0, np.log2(N))
    maps = want
    F = (np.fft.rfft(maps, axis=-1) if real else np.fft.fft(maps, axis=-1)) / N
    got_f = _run_forward(env, 0, L, maps if not real else maps.astype(complex), real, 0)
    assert np.abs(got_f - np.swapaxes(F, 1, 2)).max() <= 1e-14 * np.abs(F).max() * max(1, np.log2(N))


@pytest.mark.parametrize("L", [2, 5, 33, 128, 511])
@pytest.mark.parametrize("real", [True, False])
def test_theta_stage_vs_oracle(env, L, real):
    from oracle import oracle as orc

    rng = np.random.default_rng(L + 7)
    f = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    if real:
        import paper_1211_1680_b200 as sw

        f = sw.gaussian_coeffs(L, rng, real_signal=True).coeffs
    maps = orc.sh_synthesis(f[None], L, real, "mw")
    H = _run_forward(env, 1, L, maps, real, 1)
    # the CUDA theta stage evaluates H on the analysis rings (2j+1) pi / 2L
    Href = orc.mw_theta_stage_rings(orc.rings_forward(maps, L, real), L, real)
    scale = np.abs(Href).max()
    assert np.abs(H - Href).max() <= 1e-12 * scale


@pytest.mark.parametrize("L", [2049, 4096])
@pytest.mark.parametrize("real", [True, False])
def test_phi_stages_large_odd_n_vs_numpy(env, L, real):
    """L = 2049: generic split-mode Bluestein rows; L = 4096: the k4 Rader kernels."""
    rng = np.random.default_rng(L)
    N = 2 * L - 1
    nb = L if real else N
    G = rng.standard_normal((1, L, nb)) + 1j * rng.standard_normal((1, L, nb))
    if real:
        G[:, :, 0] = G[:, :, 0].real
        want = np.fft.irfft(G, n=N, axis=-1, norm="forward")
    else:
        want = np.fft.ifft(G, axis=-1, norm="forward")
    got = _run_inverse(env, 0, L, G, real)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max() * np.log2(N)
    F = (np.fft.rfft(want, axis=-1) if real else np.fft.fft(want, axis=-1)) / N
    got_f = _run_forward(env, 0, L, want if not real else want.astype(complex), real, 0)
    assert np.abs(got_f - np.swapaxes(F, 1, 2)).max() <= 1e-14 * np.abs(F).max() * np.log2(N)


@pytest.mark.parametrize("L", [2048, 4096])
@pytest.mark.parametrize("real", [True, False])
def test_theta_stage_pfa_vs_oracle(env, real, L):
    """L = 2048: the theta stage's DFT_4095 runs on the prime-factor engine;
    L = 4096: DFT_8191 by Rader over the prime-factor DFT_8190 (k4 kernels)."""
    from oracle import oracle as orc

    rng = np.random.default_rng(11 + real)
    maps = rng.standard_normal((1, L, 2 * L - 1))
    if not real:
        maps = maps + 1j * rng.standard_normal((1, L, 2 * L - 1))
    maps[:, -1, :] = maps[:, -1, :1]  # a sampled function is constant on the pole ring
    H = _run_forward(env, 1, L, maps if not real else maps.astype(complex), real, 1)
    Href = orc.mw_theta_stage_rings(orc.rings_forward(maps, L, real), L, real)
    # at L = 4096 the oracle's dense double-precision operator (8191-term dot
    # products) carries ~2e-12 itself: the Rader kernels and the former
    # split-mode Bluestein kernels agree to 2.5e-15 and both sit 2.1e-12 from it
    tol = 1e-12 if L <= 2048 else 4e-12
    assert np.abs(H - Href).max() <= tol * np.abs(Href).max()
