"""CLI (reference cli.py): exit codes and the CPU-only commands; the
transform commands run on the GPU (marked)."""
import numpy as np
import pytest

import paper_1211_1680_b200 as sw
from paper_1211_1680_b200 import cli


def test_usage_and_io_exit_codes(tmp_path, capsys):
    assert cli.main(["analyze"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--lmax-exp", "1", "--report", str(tmp_path / "r.json")]) == cli.EXIT_USAGE
    assert cli.main(["plot", "--in", "x", "--out", "y"]) == cli.EXIT_USAGE
    assert cli.main(["analyze", "--in", str(tmp_path / "missing.s2wm"), "--lambda", "2",
                     "--out-prefix", str(tmp_path / "p")]) == cli.EXIT_IO
    bad = tmp_path / "bad.s2wm"
    bad.write_bytes(b"nope")
    assert cli.main(["analyze", "--in", str(bad), "--lambda", "2",
                     "--out-prefix", str(tmp_path / "p")]) == cli.EXIT_FORMAT


def test_kernels_tsv(tmp_path):
    out = tmp_path / "k.tsv"
    assert cli.main(["kernels", "--bandlimit", "32", "--lambda", "2", "--out", str(out)]) == cli.EXIT_OK
    lines = out.read_text().splitlines()
    assert lines[0].startswith("# ell\tscaling\twavelet_j0")
    assert len(lines) == 32 + 2 and lines[-1].startswith("# identity residual = ")
    kern = sw.build_kernels(sw.TilingParams(32, 2.0, 0), sw.KernelFamily.SCALE_DISCRETISED)
    row = lines[1 + 5].split("\t")
    assert float(row[1]) == float(f"{kern.phi[5]:.16e}")


@pytest.mark.gpu
def test_analyze_synthesize_denoise(tmp_path, capsys):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    L = 32
    f = sw.gaussian_coeffs(L, np.random.default_rng(2), real_signal=True)
    smap = sw.sh_synthesis(f, sw.make_grid(sw.SamplingScheme.GL, L))
    src = tmp_path / "in.s2wm"
    sw.write_map(src, smap)
    prefix = str(tmp_path / "w")
    assert cli.main(["analyze", "--in", str(src), "--lambda", "2", "--out-prefix", prefix]) == 0
    out = tmp_path / "rec.s2wm"
    assert cli.main(["synthesize", "--in-prefix", prefix, "--lambda", "2", "--bandlimit", str(L),
                     "--out", str(out), "--reference", str(src)]) == 0
    eps = float(capsys.readouterr().out.strip().splitlines()[-1].split("=")[1])
    assert eps <= 1e-12
    rec = sw.read_map(out)
    assert np.abs(rec.values - smap.values).max() <= 1e-12
    # wrong band-limit: parameter error
    assert cli.main(["synthesize", "--in-prefix", prefix, "--lambda", "3", "--bandlimit", str(L),
                     "--out", str(out)]) == cli.EXIT_PARAMETER
    den = tmp_path / "den.s2wm"
    assert cli.main(["denoise", "--in", str(src), "--sigma", "0.01", "--lambda", "2",
                     "--out", str(den), "--reference", str(src)]) == 0
    want = sw.denoise_pipeline(smap, 0.01, sw.TransformConfig(L, 2.0, 0))
    assert np.array_equal(sw.read_map(den).values, want.values)
