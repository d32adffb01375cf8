"""Legendre-stage accuracy at large L: GPU synthesis vs the CPU oracle on sampled orders."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1211_1680_b200 as sw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1211_1680_b200.device import SphericalHarmonicTransform  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
rng = np.random.default_rng(5)
f = (rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)) / np.sqrt(2)
orders = np.array([0, 1, 100, L // 3, L // 2, L - 300, L - 2], dtype=np.int32)
for scheme, sch in ((sw.SamplingScheme.GL, "gl"), (sw.SamplingScheme.MW, "mw")):
    sht = SphericalHarmonicTransform(scheme, L)
    x = sht.synthesis(torch.from_numpy(f[None].copy()).cuda()).cpu().numpy()[0]
    N = 2 * L - 1
    Gg = np.fft.fft(x, axis=-1) / N  # ring-major, accurate pocketfft
    Go = orc.legendre_synth(f[None], L, False, sch, orders=orders)[0]
    for m in orders:
        for mm in ((m, -m) if m else (m,)):
            b = mm % N
            rows = slice(0, L - 1) if sch == "mw" else slice(0, L)
            d = np.abs(Gg[rows, b] - Go[rows, b]).max()
            print(f"L={L} {sch} m={mm:5d} max|G| {np.abs(Go[rows, b]).max():9.3e}  max|dG| {d:9.2e}")
    # analysis of the oracle-exact map at the sampled orders
    xo = orc.rings_inverse(Go[None], L, False, sch)
    fb = sht.analysis(torch.from_numpy(xo).cuda()).cpu().numpy()[0]
    idx = np.concatenate([np.arange(m, L) ** 2 + np.arange(m, L) + s * m
                          for m in orders for s in ((1, -1) if m else (1,))])
    print(f"L={L} {sch} analysis of oracle map: max|df| {np.abs(fb[idx] - f[idx]).max():.2e}")
