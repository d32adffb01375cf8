"""`python -m paper_1211_1680_b200 bench` (reference cli.py:236-268): usage
errors on CPU, the report schema on the GPU (marked)."""
import json

import pytest

from paper_1211_1680_b200 import cli


def test_usage_exit_codes(tmp_path):
    rep = str(tmp_path / "r.json")
    assert cli.main([]) == cli.EXIT_USAGE
    assert cli.main(["analyze", "--in", "x"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--report", rep]) == cli.EXIT_USAGE          # missing --lmax-exp
    assert cli.main(["bench", "--lmax-exp", "1", "--report", rep]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--lmax-exp", "3", "--reps", "0", "--report", rep]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--lmax-exp", "3", "--family", "haar", "--report", rep]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--lmax-exp", "x", "--report", rep]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--lmax-exp", "3", "--bogus", "1", "--report", rep]) == cli.EXIT_USAGE


@pytest.mark.gpu
def test_bench_report_schema(tmp_path, capsys):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rep = tmp_path / "r.json"
    assert cli.main(["bench", "--lmax-exp", "7", "--reps", "1", "--report", str(rep)]) == cli.EXIT_OK
    d = json.loads(rep.read_text())
    assert d["family"] == "sd" and d["lambda"] == 2.0 and d["jmin"] == 0
    assert [r["L"] for r in d["records"]] == [4, 8, 16, 32, 64, 128]
    keys = {"L", "family", "eps_full", "eps_multi", "t_full_ms", "t_multi_ms",
            "t_full_median_ms", "t_multi_median_ms", "reps", "seed"}
    for r in d["records"]:
        assert set(r) == keys
        assert r["eps_full"] <= 1e-11 and r["eps_multi"] <= 1e-11
    assert "slope_full" not in d          # only two records with L >= 64
    out = capsys.readouterr().out.strip().splitlines()
    assert out[0].startswith("L=4 eps_full=")
    # a bad lambda is a ParameterError -> exit 4
    assert cli.main(["bench", "--lmax-exp", "3", "--lambda", "1.0", "--report", str(rep)]) == cli.EXIT_PARAMETER
