"""Accuracy diagnostics on the GPU: SHT and wavelet round trips per stage.

    python scripts/accuracy_probe.py [L ...]        (default 256 1024 2048)
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1211_1680_b200 as sw  # noqa: E402
from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform  # noqa: E402

for L in [int(a) for a in (sys.argv[1:] or ["256", "1024", "2048"])]:
    for real in (False, True):
        rng = np.random.default_rng(L)
        f = sw.gaussian_coeffs(L, rng, real_signal=real).coeffs
        ft = torch.from_numpy(f[None]).cuda()
        for scheme in (sw.SamplingScheme.GL, sw.SamplingScheme.MW):
            sht = SphericalHarmonicTransform(scheme, L)
            x = sht.synthesis(ft, real=real)
            back = sht.analysis(x)
            d = (back - ft).abs()[0].cpu().numpy()
            ell = np.floor(np.sqrt(np.arange(L * L))).astype(int)
            per_l = np.zeros(L)
            np.maximum.at(per_l, ell, d)
            worst = np.argsort(per_l)[-3:][::-1]
            print(f"L={L} real={real} {scheme.value} SHT rt max|df|={d.max():.2e} "
                  f"(|f|max={np.abs(f).max():.1f}); worst l {list(worst)}")
            cfg = sw.TransformConfig(L, 2.0, 0, scheme=scheme, multires=True)
            wt = WaveletTransform(cfg, real=real)
            y = wt.round_trip(x)
            fb = sht.analysis(y)
            print(f"   wavelet rt: map rel {((y-x).abs().max()/x.abs().max()).item():.2e}  "
                  f"flm abs {(fb-ft).abs().max().item():.2e}")
