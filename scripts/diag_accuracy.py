"""Accuracy diagnostics on the GPU box (not a test): where do the L = 4096
errors sit, and who is right -- the device, the oracle's double recursion or
its long-double recursion?

  python scripts/diag_accuracy.py [sections...]   (sections: m0 c5top eps)
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import paper_1211_1680_b200 as sw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1211_1680_b200.device import SphericalHarmonicTransform, WaveletTransform  # noqa: E402


def modes(x, real):
    N = x.shape[-1]
    return (np.fft.rfft(x.real, axis=-1) if real else np.fft.fft(x, axis=-1)) / N


def m0(L=4096, real=False):
    f = sw.gaussian_coeffs(L, np.random.default_rng(L + 3 * real), real_signal=real).coeffs
    sht = SphericalHarmonicTransform(sw.SamplingScheme.MW, L)
    x = sht.synthesis(torch.from_numpy(f[None].copy()).cuda(), real=real)[0].cpu().numpy()
    got = modes(x, real)
    orders = np.array([0, 1, 2, 17, 100, 700], np.int32)
    Gp = orc.legendre_synth(f[None], L, real, "mw", orders=orders, precise=True)[0]
    Gd = orc.legendre_synth(f[None], L, real, "mw", orders=orders, precise=False)[0]
    for m in orders:
        gp, gd, gg = Gp[:, m], Gd[:, m], got[:, m]
        s = np.abs(gp).max()
        eg, ed = np.abs(gg - gp) / s, np.abs(gd - gp) / s
        top = np.argsort(eg[:-1])[-5:][::-1]
        print(f"L={L} real={real} m={m}: dev-vs-precise max {eg[:-1].max():.2e} at rings {top.tolist()}"
              f"  double-vs-precise max {ed[:-1].max():.2e} (ring {int(np.argmax(ed[:-1]))})"
              f"  pole dev {eg[-1]:.2e} double {ed[-1]:.2e}")
        print("   dev err by ring decile:", " ".join(f"{v:.1e}" for v in
                                                   [eg[i * L // 10:(i + 1) * L // 10].max() for i in range(10)]))


def c5top():
    L, real = 4096, True
    f = bench.seeded_coeffs(L, real, "beam", 1000)
    cfg = sw.TransformConfig(L, 2.0, 0, scheme=sw.SamplingScheme.MW, multires=True)
    kern = sw.kernels_for(cfg).table()
    wt = WaveletTransform(cfg, batch=1, real=real)
    sht = SphericalHarmonicTransform(sw.SamplingScheme.MW, L)
    x = sht.synthesis(torch.from_numpy(f[None].copy()).cuda(), real=real)
    maps = wt.analysis(x)
    j = len(wt.bands) - 1
    k = wt.bands[j]
    ell = np.arange(k)
    W = f[: k * k] * np.repeat(np.sqrt(4 * np.pi / (2 * ell + 1.0)) * kern[j, :k], 2 * ell + 1)
    got = modes(maps[j][0].cpu().numpy(), real)
    orders = np.array([0, 1, 2, 17, 100, 700, 2048, 4000], np.int32)
    Gp = orc.legendre_synth(W[None], k, real, "mw", orders=orders, precise=True)[0]
    Gd = orc.legendre_synth(W[None], k, real, "mw", orders=orders, precise=False)[0]
    xin = np.abs(x.cpu().numpy()).max()
    print(f"C5 top scale j={j} k={k}: input max {xin:.3e}")
    for m in orders:
        s = np.abs(Gp[:, m]).max()
        eg = np.abs(got[:-1, m] - Gp[:-1, m]).max()
        ed = np.abs(Gd[:-1, m] - Gp[:-1, m]).max()
        print(f"  m={m}: |G| max {s:.3e}  dev-vs-precise {eg:.2e} (rel {eg / s:.1e})  "
              f"double-vs-precise {ed:.2e} (rel {ed / s:.1e})")


def eps():
    for sch in ("GL", "MW"):
        S = getattr(sw.SamplingScheme, sch)
        e = []
        for s in range(20):
            L = 32
            flm = sw.gaussian_coeffs(L, np.random.default_rng(s), real_signal=True)
            fmap = sw.sh_synthesis(flm, sw.make_grid(S, L))
            dec = sw.wav_analysis_pixel(fmap, sw.TransformConfig(L, 2.0, 0, scheme=S))
            rec = sw.wav_synthesis_pixel(dec)
            d = np.abs(flm.coeffs - sw.sh_analysis(rec).coeffs)
            i = int(np.argmax(d))
            l = int(np.sqrt(i))
            e.append(d[i])
            print(f"{sch} seed {s}: eps {d[i]:.3e} at l={l} m={i - l * l - l}  "
                  f"map-rt {np.abs(rec.values - fmap.values).max():.2e}  sht-only "
                  f"{np.abs(sw.sh_analysis(fmap).coeffs - flm.coeffs).max():.2e}")
        e = np.array(e)
        print(f"{sch}: rel var {np.var(e) / np.mean(e) ** 2:.4f} mean {np.mean(e):.3e}")


if __name__ == "__main__":
    secs = sys.argv[1:] or ["m0", "c5top", "eps"]
    for s in secs:
        if s == "m0":
            m0(4096, False)
            m0(4096, True)
            m0(2048, False)
        else:
            globals()[s]()
