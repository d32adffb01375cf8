"""Accuracy and timing trials (drop-in for sphwav/bench.py).

Seeded inputs use the reference's draw order exactly (bench.py:54-72), so a
seed produces bit-identical f_lm here and in the reference.
"""
from __future__ import annotations

import statistics
import time
from dataclasses import asdict, dataclass

import numpy as np

from .errors import ParameterError
from .grid import make_grid
from .sht import HarmonicCoeffs, lm_index, sh_analysis, sh_synthesis
from .tiling import KernelFamily
from .transform import TransformConfig, wav_analysis_pixel, wav_synthesis_pixel

__all__ = ["BenchRecord", "gaussian_coeffs", "run_trial", "run_bench", "fit_scaling"]


@dataclass(frozen=True)
class BenchRecord:
    L: int
    family: str
    eps_full: float
    eps_multi: float
    t_full_ms: float
    t_multi_ms: float
    t_full_median_ms: float
    t_multi_median_ms: float
    reps: int
    seed: int

    def __post_init__(self):
        if self.reps < 1:
            raise ParameterError(f"reps must be >= 1, got {self.reps}")
        if self.eps_full < 0.0 or self.eps_multi < 0.0:
            raise ParameterError("error metrics cannot be negative")

    def as_dict(self) -> dict:
        return asdict(self)


def gaussian_coeffs(L: int, rng: np.random.Generator, real_signal: bool = True) -> HarmonicCoeffs:
    """Unit-variance Gaussian f_lm; exact conjugate symmetry when real_signal."""
    if not real_signal:
        re = rng.standard_normal(L * L)
        im = rng.standard_normal(L * L)
        return HarmonicCoeffs(L, (re + 1j * im) / np.sqrt(2.0), real_signal=False)
    c = np.zeros(L * L, dtype=np.complex128)
    for ell in range(L):
        i0 = lm_index(ell, 0)
        c[i0] = rng.standard_normal()
        if ell == 0:
            continue
        pos = (rng.standard_normal(ell) + 1j * rng.standard_normal(ell)) / np.sqrt(2.0)
        c[i0 + 1 : i0 + ell + 1] = pos
        m = np.arange(1, ell + 1)
        c[i0 - m] = np.where(m % 2 == 0, 1.0, -1.0) * np.conj(pos)
    return HarmonicCoeffs(L, c, real_signal=True)


def run_trial(L: int, config: TransformConfig, seed: int) -> tuple[float, float]:
    """One timed wavelet round trip: (max |f - f_rec|, mean of the two halves in ms)."""
    if config.L != L:
        config = TransformConfig(L, config.lam, config.j0, config.family, config.scheme,
                                 config.multires)
    flm = gaussian_coeffs(L, np.random.default_rng(seed), real_signal=True)
    fmap = sh_synthesis(flm, make_grid(config.scheme, L))
    t0 = time.perf_counter()
    decomp = wav_analysis_pixel(fmap, config)
    t1 = time.perf_counter()
    rec = wav_synthesis_pixel(decomp)
    t2 = time.perf_counter()
    eps = float(np.max(np.abs(flm.coeffs - sh_analysis(rec).coeffs)))
    return eps, 1000.0 * ((t1 - t0) + (t2 - t1)) / 2.0


def run_bench(L_values, lam: float = 2.0, j0: int = 0,
              family: KernelFamily = KernelFamily.SCALE_DISCRETISED, reps: int = 3,
              seed: int = 0) -> list[BenchRecord]:
    """Mean error / time per band-limit for full- and multi-resolution."""
    if reps < 1:
        raise ParameterError(f"reps must be >= 1, got {reps}")
    out = []
    for L in L_values:
        res = {}
        for multires in (False, True):
            cfg = TransformConfig(L, lam, j0, family, multires=multires)
            run_trial(L, cfg, seed)
            eps, ts = zip(*(run_trial(L, cfg, seed + r) for r in range(reps)))
            res[multires] = (float(np.mean(eps)), float(np.mean(ts)), float(statistics.median(ts)))
        out.append(BenchRecord(L, family.value, res[False][0], res[True][0], res[False][1],
                               res[True][1], res[False][2], res[True][2], reps, seed))
    return out


def fit_scaling(records, min_L: int = 64, timing: str = "full") -> float:
    """Least-squares slope of log(time) against log(L)."""
    if timing not in ("full", "multi"):
        raise ParameterError(f"timing must be 'full' or 'multi', got {timing!r}")
    pts = [(r.L, r.t_full_ms if timing == "full" else r.t_multi_ms) for r in records if r.L >= min_L]
    if len(pts) < 3:
        raise ParameterError(f"need at least 3 records with L >= {min_L}, got {len(pts)}")
    slope, _ = np.polyfit(np.log([p[0] for p in pts]), np.log([p[1] for p in pts]), 1)
    return float(slope)
