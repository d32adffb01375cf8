"""CPU checks (numpy) of the index algebra the sm_100a FFT kernels rely on:
the prime-factor DFT slot map (pfa.cuh), Rader's DFT_8191 over the
prime-factor DFT_8190 (k4 kernels), and the parity-class split of the MW
theta-stage convolution (theta_k2 / theta_k4).  These restate the kernels'
algorithms in numpy and compare them with np.fft / a direct convolution."""
import numpy as np
import pytest


def pfa(x, factors, inv=False):
    """The kernels' pass structure: for every factor P, each line of slots
    (P r + j N/P) mod N goes through an in-place DFT_P."""
    N = len(x)
    b = x.astype(complex).copy()
    for P in factors:
        A = N // P
        W = np.exp((2j if inv else -2j) * np.pi * np.outer(np.arange(P), np.arange(P)) / P)
        r = np.arange(A)[:, None]
        idx = (P * r + np.arange(P)[None, :] * A) % N      # (A, P)
        b[idx] = b[idx] @ W.T
    return b


@pytest.mark.parametrize("N,factors,step", [(4095, (13, 7, 5, 9), 2174),
                                            (8190, (13, 7, 5, 9, 2), 253)])
def test_pfa_slot_map(N, factors, step):
    """Natural order in; bin k at slot (k * sum N/P_i) mod N out (pfa_pos); the
    inverse passes take that slot order back to natural order."""
    assert step == sum(N // P for P in factors) % N
    rng = np.random.default_rng(N)
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    pos = (np.arange(N) * step) % N
    X = np.fft.fft(x)
    assert np.abs(pfa(x, factors)[pos] - X).max() <= 1e-12 * np.abs(X).max()
    c = np.zeros(N, complex)
    c[pos] = X
    assert np.abs(pfa(c, factors, inv=True) / N - x).max() <= 1e-13 * np.abs(x).max()


def test_rader_dft_8191():
    """X_0 = sum x; X_{g^-p} = x_0 + (a * d)_p with a_q = x_{g^q}, d_j = w^{g^-j},
    the length-8190 cyclic convolution through forward PFA -> spectrum in slot
    order -> inverse PFA (pfa.cuh rader8191); inverse DFT = conj(DFT(conj))."""
    N, M, g, step = 8191, 8190, 17, 253
    factors = (13, 7, 5, 9, 2)
    assert all(pow(g, M // f, N) != 1 for f in (2, 3, 5, 7, 13))  # primitive root
    gpow = np.array([pow(g, q, N) for q in range(M)])
    ginv = pow(g, N - 2, N)
    gneg = np.array([pow(ginv, j, N) for j in range(M)])
    plog = np.zeros(N, int)
    plog[gneg] = np.arange(M)
    d = np.exp(-2j * np.pi * gneg / N)
    pos = (np.arange(M) * step) % M
    D = np.zeros(M, complex)
    D[pos] = np.fft.fft(d) / M
    rng = np.random.default_rng(8191)
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)

    def rader(v):
        c = pfa(pfa(v[gpow], factors) * D, factors, inv=True)
        out = np.empty(N, complex)
        out[0] = v.sum()
        out[1:] = v[0] + c[plog[1:]]
        return out

    X = np.fft.fft(x)
    assert np.abs(rader(x) - X).max() <= 1e-12 * np.abs(X).max()
    Y = np.conj(rader(np.conj(x)))
    assert np.abs(Y - N * np.fft.ifft(x)).max() <= 1e-12 * np.abs(Y).max()


@pytest.mark.parametrize("k", [64, 2048])
def test_theta_parity_class_convolution(k):
    """H'(q) = sum_m' a_m' w(q - m'), |q|, |m'| <= k-1, w(p) = 4/(1-p^2) at even p
    and 0 at odd p: equal to two cyclic convolutions of length 2k (one per
    parity class of q, kernel w(2d)), as theta_k2 (k = 2048) / theta_k4 compute it."""
    rng = np.random.default_rng(k)
    q = np.arange(-(k - 1), k)
    a = rng.standard_normal(2 * k - 1) + 1j * rng.standard_normal(2 * k - 1)
    p = q[:, None] - q[None, :]
    pe = np.where(p % 2 == 0, p, 0).astype(float)  # odd p: 0 (masked below)
    w = np.where(p % 2 == 0, 4.0 / (1.0 - pe ** 2), 0.0)
    want = w @ a
    M = 2 * k
    d = np.arange(-(M // 2 - 1), M // 2)
    ker = np.zeros(M)
    ker[d % M] = 4.0 / (1.0 - 4.0 * d.astype(float) ** 2)
    K = np.fft.fft(ker)
    got = np.empty_like(want)
    for par in (0, 1):
        sel = (q % 2) == par
        b = (q[sel] - par) // 2                     # class index: q = 2b + par
        buf = np.zeros(M, complex)
        buf[b % M] = a[sel]
        y = np.fft.ifft(np.fft.fft(buf) * K)
        got[sel] = y[b % M]
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
