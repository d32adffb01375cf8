"""Per-stage timing of one SHT pair on the device (development aid).

    python scripts/time_sht.py --L 2048 --scheme mw --batch 1 [--real] [--reps 5]

Prints the library's per-stage CUDA-event times (ms per call) for analysis and
synthesis separately, and the canonical-FLOP rate of the Legendre stages.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import torch  # noqa: E402

from paper_1211_1680_b200 import _native  # noqa: E402
from paper_1211_1680_b200.device import SphericalHarmonicTransform  # noqa: E402
from paper_1211_1680_b200.grid import SamplingScheme  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=2048)
    ap.add_argument("--scheme", default="mw")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--real", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    L, B = a.L, a.batch
    sht = SphericalHarmonicTransform(SamplingScheme.MW if a.scheme == "mw" else SamplingScheme.GL, L)
    g = torch.Generator(device="cuda").manual_seed(1)
    flm = torch.randn((B, L * L), dtype=torch.complex128, device="cuda", generator=g)
    if a.real:
        # real-signal coefficients via a real map round trip
        flm = sht.analysis(sht.synthesis(flm).real.contiguous())
    maps = sht.synthesis(flm, real=a.real)
    for _ in range(2):
        sht.analysis(maps)
        sht.synthesis(flm, real=a.real)
    torch.cuda.synchronize()
    S = L * (L + 1) // 2 if a.real else L * L
    F = 4.0 * B * L * S + 4.0 * L * L * (L + 1) / 2
    for name, fn in [("analysis", lambda: sht.analysis(maps)),
                     ("synthesis", lambda: sht.synthesis(flm, real=a.real))]:
        _native.profile_enable(True)
        _native.profile_read(reset=True)
        for _ in range(a.reps):
            fn()
        torch.cuda.synchronize()
        prof = _native.profile_read(reset=True)
        _native.profile_enable(False)
        st = {k: round(v[0] / a.reps, 3) for k, v in prof.items() if v[1]}
        leg = [v for k, v in st.items() if k.startswith("leg")][0]
        print(f"{name:9s} L={L} B={B} real={a.real}: {st}  legendre {F / leg / 1e9:.2f} TFLOP/s")


if __name__ == "__main__":
    main()
