"""Generate golden vectors from the reference package (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (sphwav, /root/reference/pkg/src) is imported read-only and its
own public API produces every output stored here; nothing in the repository
imports it at run time.  Seeds and sizes are recorded in each file.  Large maps
are stored as seeded random subsamples (index + value) plus full-array norms.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import sphwav as sw  # noqa: E402

OUT = Path(__file__).resolve().parent
GL, MW = sw.SamplingScheme.GL, sw.SamplingScheme.MW


def scaled_coeffs(L, seed, real, spectrum):
    """sphwav.gaussian_coeffs with row l scaled by sqrt(C_l)."""
    f = sw.gaussian_coeffs(L, np.random.default_rng(seed), real_signal=real)
    ell = np.repeat(np.arange(L), 2 * np.arange(L) + 1)
    c = np.sqrt(spectrum(np.arange(L).astype(float)))[ell]
    return sw.HarmonicCoeffs(L, f.coeffs * c, real_signal=real)


def flat(_l):
    return np.ones_like(_l)


def sub(arr, n, seed):
    a = np.asarray(arr).reshape(-1)
    if a.size <= n:
        return np.arange(a.size), a
    idx = np.sort(np.random.default_rng(seed).choice(a.size, n, replace=False))
    return idx, a[idx]


def sht_cases():
    d = {}
    for L in (1, 2, 4, 5, 7, 8, 16, 24, 33, 64):
        for real in (True, False):
            seed = 100 + 2 * L + int(real)
            f = sw.gaussian_coeffs(L, np.random.default_rng(seed), real_signal=real)
            tag = f"L{L}_{'r' if real else 'c'}"
            d[f"f_{tag}"] = f.coeffs
            gl = sw.sh_synthesis(f, sw.make_grid(GL, L))
            mw = sw.sh_synthesis(f, sw.make_grid(MW, L))
            d[f"gl_map_{tag}"] = gl.values
            d[f"mw_map_{tag}"] = mw.values
            d[f"gl_ana_{tag}"] = sw.sh_analysis(gl).coeffs
    # synthesis of a lower band on a finer grid (sht.py:230)
    f6 = sw.gaussian_coeffs(6, np.random.default_rng(5), real_signal=True)
    d["f_up6"] = f6.coeffs
    d["gl_map_up6_13"] = sw.sh_synthesis(f6, sw.make_grid(GL, 13)).values
    d["mw_map_up6_13"] = sw.sh_synthesis(f6, sw.make_grid(MW, 13)).values
    np.savez_compressed(OUT / "sht_small.npz", **d)


def legendre_cases():
    d = {}
    d["ring_L16_t1"] = sw.assoc_legendre_ring(16, 1.0)
    d["ring_L40_t03"] = sw.assoc_legendre_ring(40, 0.3)
    d["ring_L1536_t07_rows"] = sw.assoc_legendre_ring(1536, 0.7)[::97]
    np.savez_compressed(OUT / "legendre.npz", **d)


def kernel_cases():
    d = {}
    for fam in ("SCALE_DISCRETISED", "NEEDLET", "BSPLINE"):
        for L, lam, j0 in ((64, 2.0, 0), (128, 3.0, 2), (256, 2.0, 2), (2048, 3.0, 2)):
            if fam == "NEEDLET" and L > 256:
                continue
            k = sw.build_kernels(sw.TilingParams(L, lam, j0), getattr(sw.KernelFamily, fam))
            tag = f"{fam}_{L}_{lam:g}_{j0}"
            d[f"phi_{tag}"] = k.phi
            d[f"psi_{tag}"] = k.psi
            d[f"bands_{tag}"] = np.array([k.scaling_bandlimit, *k.scale_bandlimits])
    np.savez_compressed(OUT / "kernels.npz", **d)


def wavelet_cases():
    """Reference wavelet maps.  GL: wav_analysis_pixel directly.  MW: the
    reference cannot analyse MW maps (sht.py:300-303), so the MW golden scale
    maps are its harmonic tiling (transform.py:129) followed by its MW
    synthesis per scale grid (transform.py:212-229) of the known f_lm."""
    d = {}
    cases = [
        ("c1", 64, 2.0, 0, False, False, flat),
        ("c2s", 64, 2.0, 2, True, True, lambda l: np.where(l >= 2, 1.0 / np.maximum(l * (l + 1), 1), 0.0)),
        ("gl32", 32, 2.0, 0, True, True, flat),
        ("gl32full", 32, 3.0, 1, False, False, flat),
    ]
    for name, L, lam, j0, multires, real, spec in cases:
        f = scaled_coeffs(L, 7, real, spec)
        d[f"f_{name}"] = f.coeffs
        for scheme in (GL, MW):
            cfg = sw.TransformConfig(L, lam, j0, scheme=scheme, multires=multires)
            kern = sw.kernels_for(cfg)
            wc = sw.wav_analysis_harmonic(f, kern, truncate=multires)
            grids = sw.transform._scale_grids(cfg, kern)
            sets = [wc.scaling, *wc.wavelets]
            maps = [sw.sh_synthesis(s, g) for s, g in zip(sets, grids)]
            tag = f"{name}_{scheme.value}"
            for j, m in enumerate(maps):
                d[f"scale{j}_{tag}"] = m.values
            if scheme is GL:
                smap = sw.sh_synthesis(f, sw.make_grid(GL, L))
                dec = sw.wav_analysis_pixel(smap, cfg)
                for j, m in enumerate([dec.scaling, *dec.wavelets]):
                    d[f"pix{j}_{tag}"] = m.values
                rec = sw.wav_synthesis_pixel(dec)
                d[f"rec_{tag}"] = rec.values
                d[f"recflm_{tag}"] = sw.sh_analysis(rec).coeffs
    np.savez_compressed(OUT / "wavelet.npz", **d)


def denoise_cases():
    """Reference denoise_pipeline (denoise.py:99-103) on a GL map (its only
    analysable scheme): seeded signal + white noise of harmonic variance sigma^2."""
    d = {}
    for name, L, lam, j0, real in (("r32", 32, 2.0, 0, True), ("c24", 24, 2.0, 1, False)):
        sig = scaled_coeffs(L, 31, real, lambda l: np.where(l >= 2, 1.0 / np.maximum(l * (l + 1), 1), 0.0))
        noise = sw.gaussian_coeffs(L, np.random.default_rng(32), real_signal=real)
        sigma = 0.05
        f = sw.HarmonicCoeffs(L, sig.coeffs + sigma * noise.coeffs, real_signal=real)
        grid = sw.make_grid(GL, L)
        noisy = sw.sh_synthesis(f, grid)
        cfg = sw.TransformConfig(L, lam, j0, scheme=GL, multires=True)
        model = sw.denoise.make_noise_model(sigma, sw.kernels_for(cfg), 3.0)
        out = sw.denoise.denoise_pipeline(noisy, sigma, cfg, 3.0)
        d[f"noisy_{name}"] = noisy.values
        d[f"sigma_scales_{name}"] = model.sigma_scales
        d[f"denoised_{name}"] = out.values
        d[f"params_{name}"] = np.array([L, lam, j0, int(real), sigma])
    np.savez_compressed(OUT / "denoise.npz", **d)


def mapio_cases():
    """Bytes the reference's own writers produce (mapio.py:83-99)."""
    import tempfile

    d = {}
    with tempfile.TemporaryDirectory() as tmp:
        items = []
        f = sw.gaussian_coeffs(6, np.random.default_rng(41), real_signal=True)
        items.append(("gl_real", lambda p: sw.write_map(p, sw.sh_synthesis(f, sw.make_grid(GL, 6)))))
        g = sw.gaussian_coeffs(5, np.random.default_rng(42), real_signal=False)
        items.append(("mw_cplx", lambda p: sw.write_map(p, sw.sh_synthesis(g, sw.make_grid(MW, 5)))))
        items.append(("flm", lambda p: sw.write_flm(p, g)))
        for name, fn in items:
            path = Path(tmp) / f"{name}.s2wm"
            fn(path)
            d[name] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
        d["f_gl_real"] = f.coeffs
        d["f_mw_cplx"] = g.coeffs
    np.savez_compressed(OUT / "mapio.npz", **d)


def config_cases():
    """BASELINE configs C1-C3 at full size through the reference (L <= 1024,
    where its recursion is valid): MW synthesis of the seeded inputs, stored as
    subsamples + norms; the known f_lm is regenerated from the seed."""
    d = {}
    specs = {
        "C1": (64, 1, False, flat),
        "C2": (256, 2, True, lambda l: np.where(l >= 2, 1.0 / np.maximum(l * (l + 1), 1), 0.0)),
        "C3": (1024, 1, False, flat),
    }
    for name, (L, nmaps, real, spec) in specs.items():
        for b in range(nmaps):
            f = scaled_coeffs(L, 1000 + b, real, spec)
            mw = sw.sh_synthesis(f, sw.make_grid(MW, L)).values
            idx, vals = sub(mw, 4096, 11 + b)
            d[f"{name}_b{b}_idx"] = idx
            d[f"{name}_b{b}_vals"] = vals
            d[f"{name}_b{b}_norm2"] = np.array([np.sum(np.abs(mw) ** 2)])
            d[f"{name}_b{b}_max"] = np.array([np.abs(mw).max()])
            d[f"{name}_b{b}_pole"] = mw[-1, :1]
    np.savez_compressed(OUT / "configs.npz", **d)


def config_wavelet_cases():
    """Wavelet scale maps at the full C2 (L=256, real, lambda=2, J0=2) and C3
    (L=1024, complex, lambda=2, J0=3) sizes, multires, MW, map 0 of each batch.
    As in wavelet_cases the reference cannot analyse MW maps, so its scale maps
    are its own harmonic tiling of the seeded f_lm (transform.py:129-150)
    followed by its own MW synthesis on each scale grid (transform.py:108-114,
    212-229).  Stored as seeded subsamples + norms, like config_cases."""
    d = {}
    specs = {
        "C2": (256, 2.0, 2, True, lambda l: np.where(l >= 2, 1.0 / np.maximum(l * (l + 1), 1), 0.0)),
        "C3": (1024, 2.0, 3, False, flat),
    }
    for name, (L, lam, j0, real, spec) in specs.items():
        f = scaled_coeffs(L, 1000, real, spec)
        cfg = sw.TransformConfig(L, lam, j0, scheme=MW, multires=True)
        kern = sw.kernels_for(cfg)
        wc = sw.wav_analysis_harmonic(f, kern, truncate=True)
        grids = sw.transform._scale_grids(cfg, kern)
        d[f"{name}_bands"] = np.array([g.L for g in grids])
        for j, (s, g) in enumerate(zip([wc.scaling, *wc.wavelets], grids)):
            m = sw.sh_synthesis(s, g).values
            idx, vals = sub(m, 4096, 50 + j)
            d[f"{name}_s{j}_idx"] = idx
            d[f"{name}_s{j}_vals"] = vals
            d[f"{name}_s{j}_norm2"] = np.array([np.sum(np.abs(m) ** 2)])
            d[f"{name}_s{j}_max"] = np.array([np.abs(m).max()])
    np.savez_compressed(OUT / "configs_wav.npz", **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["sht", "legendre", "kernels", "wavelet", "configs", "configs_wav",
                             "denoise", "mapio"]
    for w in which:
        {"sht": sht_cases, "legendre": legendre_cases, "kernels": kernel_cases,
         "wavelet": wavelet_cases, "configs": config_cases,
         "configs_wav": config_wavelet_cases, "denoise": denoise_cases,
         "mapio": mapio_cases}[w]()
        print("wrote", w)
