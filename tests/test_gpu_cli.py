"""CLI on the B200 (ref tests `test_cli.py`): selftest passes on the device
path, bench rows follow the CSV schema with ops_per_sec = batch * 1000 /
wall_ms, sweep-n emits one row per degree; cmult_batch parity."""

import csv
import json

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def run(argv):
    from paper_2212_14191_b200 import cli
    return cli.main(argv)


def test_selftest_default(capsys):
    assert run(["selftest", "--preset", "default"]) == 0
    out = capsys.readouterr().out
    assert "transform: PASS" in out
    assert "roundtrip: PASS" in out
    assert "homomorphism: PASS" in out


@pytest.mark.parametrize("length,rot", [(1, 0), (128, 7)])
def test_workload_dotproduct(capsys, length, rot):
    assert run(["workload-dotproduct", "--length", str(length)]) == 0
    report = json.loads(capsys.readouterr().out)
    assert report["op_counts"]["hrotate"] == rot
    assert report["relative_error"] < 2 ** -15


def test_workload_too_long(capsys):
    assert run(["workload-dotproduct", "--length", "99999"]) == 2


def test_selftest_fault_injection(capsys, monkeypatch):
    from paper_2212_14191_b200 import cli
    monkeypatch.setattr(cli, "INJECT_TWIDDLE_FAULT", True)
    assert run(["selftest"]) == 1
    assert "transform: FAIL" in capsys.readouterr().out


@pytest.mark.parametrize("resident", [False, True])
def test_bench_schema_and_rate_identity(tmp_path, resident):
    from paper_2212_14191_b200 import cli
    out = tmp_path / "b.csv"
    argv = ["bench", "--ops", "ntt,hadd,hmult,rescale,hrotate,cmult,forbenius_map,intt",
            "--batch-sizes", "1,4", "--reps", "2", "--out", str(out)]
    assert run(argv + (["--resident"] if resident else [])) == 0
    rows = list(csv.DictReader(out.open()))
    assert [r["op"] for r in rows] == [o for o in ("ntt", "hadd", "hmult", "rescale", "hrotate",
                                                   "cmult", "forbenius_map", "intt")
                                       for _ in range(2)]
    assert list(rows[0]) == cli.CSV_FIELDS
    for r in rows:
        rate = float(r["batch"]) * 1000.0 / float(r["wall_ms_median"])
        assert abs(rate - float(r["ops_per_sec"])) / rate < 0.01


def test_bench_json_and_sweep(tmp_path):
    out = tmp_path / "b.json"
    assert run(["bench", "--ops", "ntt", "--batch-sizes", "2", "--reps", "1",
                "--out", str(out), "--preset", "p_default"]) == 0
    assert json.loads(out.read_text())[0]["n"] == 1 << 16
    out = tmp_path / "s.csv"
    assert run(["sweep-n", "--n-values", "1024,2048,65536", "--batch-sizes", "2",
                "--reps", "1", "--out", str(out)]) == 0
    assert [int(r["n"]) for r in csv.DictReader(out.open())] == [1024, 2048, 65536]


def test_cmult_batch_vs_oracle():
    from oracle import oracle as O
    from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.from_preset("set_b")
    ck = CkksContext(p)
    rng = np.random.default_rng(7)
    basis = p.q_basis(p.l_max)
    ct = np.stack([O.uniform_rows(rng, basis, (3, p.n)) for _ in range(2)])
    pt = O.uniform_rows(rng, basis, (3, p.n))
    d = lambda a: torch.from_numpy(a.view(np.int32)).cuda()  # noqa: E731
    got = ck.cmult_batch(CiphertextBatch(d(ct), p.l_max), d(pt), pt_scale=3).data.cpu().numpy().view(np.uint32)
    for c in range(2):
        assert np.array_equal(got[c], O.hada_mult(ct[c], pt, basis))
    shared = pt[:, 0]
    cb = ck.cmult_batch(CiphertextBatch(d(ct), p.l_max, scale=5), d(np.ascontiguousarray(shared)),
                        pt_scale=3)
    assert cb.scale == 15
    got = cb.data.cpu().numpy().view(np.uint32)
    for c in range(2):
        assert np.array_equal(got[c], O.hada_mult(ct[c], shared[:, None, :], basis))


def test_hadd_hsub_batch_vs_oracle():
    """hadd_batch / hsub_batch reduce every limb of both components mod its
    own prime (ref `ckks.py:246-256`), and reject mismatched operands."""
    from oracle import oracle as O
    from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext
    from paper_2212_14191_b200.errors import ParameterError
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.from_preset("default")
    ck = CkksContext(p)
    rng = np.random.default_rng(8)
    basis = p.q_basis(p.l_max)
    c0 = np.stack([O.uniform_rows(rng, basis, (3, p.n)) for _ in range(2)])
    c1 = np.stack([O.uniform_rows(rng, basis, (3, p.n)) for _ in range(2)])
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()  # noqa: E731
    b0, b1 = CiphertextBatch(d(c0), p.l_max), CiphertextBatch(d(c1), p.l_max)
    add = ck.hadd_batch(b0, b1).data.cpu().numpy().view(np.uint32)
    sub = ck.hsub_batch(b0, b1).data.cpu().numpy().view(np.uint32)
    for c in range(2):
        assert np.array_equal(add[c], O.ele_add(c0[c], c1[c], basis))
        assert np.array_equal(sub[c], O.ele_sub(c0[c], c1[c], basis))
    with pytest.raises(ParameterError):
        ck.hadd_batch(b0, CiphertextBatch(d(c1[:, :-1]), p.l_max - 1))
    with pytest.raises(ParameterError):
        ck.hsub_batch(b0, CiphertextBatch(d(c1), p.l_max, scale=3))


@pytest.mark.parametrize("n", [256, 1 << 12, 1 << 16])
def test_device_twiddle_fault_is_detected(n):
    """tfhe_debug_corrupt_twiddle flips a byte of the DEVICE twiddle tables
    (small-n tiles and TS planes): transforms mod that prime then disagree
    with the oracle, other primes and fresh contexts are unaffected."""
    from oracle import oracle as O
    from paper_2212_14191_b200 import _lib
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    qs = generate_primes(n, [30, 29])
    bad = DeviceContext(n, qs)           # private: not in the shared cache
    _lib.check(bad.lib.tfhe_debug_corrupt_twiddle(bad.handle, 0), "corrupt")
    x = O.uniform_rows(np.random.default_rng(n), qs, (2, n))
    d = torch.from_numpy(x.view(np.int32)).cuda()
    got = bad.ntt(d, qs).cpu().numpy().view(np.uint32)
    want = O.ntt(x, qs)
    assert not np.array_equal(got[0], want[0])
    assert np.array_equal(got[1], want[1])
    good = DeviceContext.get(n, tuple(qs))
    assert np.array_equal(good.ntt(d, qs).cpu().numpy().view(np.uint32), want)
