"""The Reinsch form of the low orders' Legendre recursion (legendre_kernels.cu
ring_step_rein, table built by capi.cu rein_rows), restated in numpy: at the
most polar ring of L = 4096 the plain three-term recursion of the reference
(sht.py:157-187) loses ~1e-10 of the column in double arithmetic (its
characteristic roots coalesce at x = 1); the Reinsch form with the x = 1
ratios computed in long double stays at ~1e-13.  CPU only: the algebra, not
the device code (the -m gpu tests pin the device against the oracle)."""
import numpy as np
import pytest

L = 4096


def ab(l, m, dt):
    l, m = dt(l), dt(m)
    den = l * l - m * m
    return (np.sqrt((4 * l * l - 1) / den),
            np.sqrt((2 * l + 1) / (2 * l - 3) * ((l - 1) * (l - 1) - m * m) / den))


def rein_row(m):
    """(lambda'_l, kappa'_l) as capi.cu rein_rows: rho from the x = 1 recursion."""
    ld = np.longdouble
    row = np.zeros((L, 2))
    row[m] = (0.0, 1.0)
    rho_prev = ld(0)
    for l in range(m + 1, L):
        a, b = ab(l, m, ld)
        rho = a if l == m + 1 else a - b / rho_prev
        kap = ld(0) if l == m + 1 else b / (a * rho_prev)
        row[l] = (float(rho / a), float(kap))
        rho_prev = rho
    return row


def seed(m, theta, dt):
    c = dt(1) / np.sqrt(4 * dt(np.pi))
    for k in range(1, m + 1):
        c *= np.sqrt(dt(2 * k + 1) / dt(2 * k))
    return c * (-np.sin(dt(theta))) ** m


def plain(m, theta, dt):
    """P_lm by the reference recursion in arithmetic dt."""
    x = np.cos(dt(theta))
    P = np.zeros(L, dt)
    P[m] = seed(m, theta, dt)
    for l in range(m + 1, L):
        a, b = ab(l, m, dt)
        P[l] = a * x * P[l - 1] - (b * P[l - 2] if l > m + 1 else 0)
    return P


def reinsch_normalised(m, theta, row):
    """The kernel's state in double: chunks of 32 degrees from l = m, within a
    chunk Q_l = P_l / gamma_l with gamma_l = prod_{j = l0..l} a_j, both state
    values rebased by the chunk's last gamma (ring_rebase), stepped by
    ring_step_rein; mapped back to P_l."""
    u = 2.0 * np.sin(theta / 2) ** 2
    Q1, d = 0.0, float(seed(m, theta, np.float64))
    gamma = 1.0
    P = np.zeros(L)
    for l in range(m, L):
        lam, kap = row[l]
        uq = u * Q1
        d = kap * d - uq
        Q1 = lam * Q1 + d
        if l > m:
            gamma *= float(ab(l, m, np.float64)[0])
        P[l] = Q1 * gamma
        if (l - m) % 32 == 31:          # chunk end: rebase
            Q1, d, gamma = Q1 * gamma, d * gamma, 1.0
    return P


@pytest.mark.parametrize("m", [0, 3])
def test_reinsch_form_at_the_pole(m):
    theta = np.pi / (2 * L)                       # first MW analysis ring at L = 4096
    exact = plain(m, theta, np.longdouble).astype(np.float64)
    scale = np.abs(exact).max()
    e_plain = np.abs(plain(m, theta, np.float64) - exact).max() / scale
    e_rein = np.abs(reinsch_normalised(m, theta, rein_row(m)) - exact).max() / scale
    assert e_plain > 1e-11          # the reference's own double recursion
    assert e_rein < 2e-12           # O(l eps) (long-double exact value itself ~1e-13)
    assert e_rein < e_plain / 20


def test_reinsch_table_identities():
    row = rein_row(5)
    lam, kap = row[:, 0], row[:, 1]
    assert lam[5] == 0.0 and kap[5] == 1.0 and lam[6] == 1.0 and kap[6] == 0.0
    # lambda'_l = 1 - kappa'_l and kappa'_l = beta_l / lambda'_{l-1}
    l = np.arange(7, L)
    assert np.abs(lam[l] - (1 - kap[l])).max() < 1e-15
    beta = np.array([ab(i, 5, np.float64)[1] / (ab(i, 5, np.float64)[0] * ab(i - 1, 5, np.float64)[0])
                     if i > 6 else 0.0 for i in l])
    assert np.abs(kap[l] - beta / lam[l - 1]).max() < 1e-13
