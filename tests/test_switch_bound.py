"""The predictive significance switch of the Legendre kernels (ring_fix in
csrc/legendre_kernels.cu), restated in numpy: below the classical turning
point |P_lm(theta)| grows with l at a falling rate, so the last step's growth
bounds every later one and

    level(l) + n * log2(|P_l| / |P_{l-1}|)  >=  level(l + j),  0 <= j <= n.

The kernels look at a ring once per 32-degree chunk and leave its terms out of
the contraction until that bound passes 2^-80; this test checks the bound on
the recursion itself (reference sht.py:140-187 coefficients, log2-scaled), for
every ring of an L = 2048 analysis set at sampled orders, and the seed bound
a_{m+1,m} x <= sqrt(2m + 3) used before the first look.
"""
import numpy as np
import pytest

L = 2048
NEXT = 32


def _levels(m, x, s):
    """log2 |P_lm| for l = m .. L-1 on the rings (x, s) by the scaled recursion."""
    logc = 0.5 * np.log2(1.0 / (4.0 * np.pi))
    for i in range(1, m + 1):
        logc += 0.5 * np.log2((2.0 * i + 1.0) / (2.0 * i))
    E = logc + m * np.log2(s)
    pm2 = np.zeros_like(x)
    pm1 = np.ones_like(x)
    out = [E + 0.0]
    for l in range(m + 1, L):
        a = np.sqrt((4.0 * l * l - 1.0) / (l * l - m * m))
        b = np.sqrt(((l - 1.0) ** 2 - m * m) / (4.0 * (l - 1.0) ** 2 - 1.0)) if l - 1 > m else 0.0
        pn = a * (x * pm1 - b * pm2)
        pm2, pm1 = pm1, pn
        big = np.abs(pm1) > 2.0 ** 200
        pm1 = np.where(big, pm1 * 2.0 ** -200, pm1)
        pm2 = np.where(big, pm2 * 2.0 ** -200, pm2)
        E = np.where(big, E + 200.0, E)
        with np.errstate(divide="ignore"):
            out.append(E + np.log2(np.abs(pm1)))
    return np.array(out)


@pytest.mark.parametrize("m", [32, 100, 333, 1000, 1800])
def test_growth_bound_in_the_forbidden_region(m):
    j = np.arange(L // 2)
    theta = (2 * j + 1) * np.pi / (2 * L)
    lv = _levels(m, np.cos(theta), np.sin(theta))  # [l - m][ring]
    n = lv.shape[0]
    checked = 0
    for i in range(NEXT - 1, n - 1, NEXT):  # chunk ends (chunks start at l = m)
        low = lv[i] < -40.0  # rings the kernels still hold back (or soon would)
        if not low.any():
            continue
        g = np.maximum(lv[i] - lv[i - 1], 0.0)
        reach = lv[i] + NEXT * g
        top = lv[i:min(i + NEXT + 1, n)].max(axis=0)
        assert np.all(top[low] <= reach[low] + 1e-6)
        checked += int(low.sum())
    assert checked > 0
    # the seed: the first look comes NEXT - 1 steps after l = m
    g0 = 0.5 * np.log2(2.0 * m + 3.0)
    top0 = lv[:min(NEXT, n)].max(axis=0)
    assert np.all(top0 <= lv[0] + (NEXT - 1) * g0 + 1e-6)
