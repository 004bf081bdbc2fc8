"""CLI surface (ref `cli.py`, tests `test_cli.py`) on CPU: argument handling,
usage errors (exit 2), the CSV schema, and the loud no-GPU failure (exit 1)."""

import pytest


def run(argv):
    from paper_2212_14191_b200 import cli
    return cli.main(argv)


def test_schema_matches_reference():
    from paper_2212_14191_b200 import cli
    assert cli.CSV_FIELDS == ["op", "backend", "n", "level", "batch", "threads", "reps",
                              "wall_ms_median", "ops_per_sec"]
    assert cli.BENCH_OPS == ("ntt", "intt", "hmult", "hadd", "hrotate", "rescale", "cmult",
                             "forbenius_map")


def test_unknown_op_is_usage_error():
    with pytest.raises(SystemExit) as exc:
        run(["bench", "--ops", "quantum"])
    assert exc.value.code == 2


def test_bad_preset_is_usage_error():
    with pytest.raises(SystemExit) as exc:
        run(["selftest", "--preset", "bogus"])
    assert exc.value.code == 2


def test_sweep_bad_n_rejected(capsys):
    assert run(["sweep-n", "--n-values", "1000"]) == 2


def test_empty_sweep_header_only(tmp_path):
    out = tmp_path / "s.csv"
    assert run(["sweep-n", "--n-values", "", "--out", str(out)]) == 0
    from paper_2212_14191_b200 import cli
    assert out.read_text().strip().splitlines() == [",".join(cli.CSV_FIELDS)]


def test_no_gpu_fails_loudly(capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("checks the no-GPU behaviour")
    assert run(["selftest", "--preset", "default"]) == 1
    assert "no CUDA device" in capsys.readouterr().err
