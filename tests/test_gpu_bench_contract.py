"""bench.py's driver contract on one B200, at a small configuration: exactly
one JSON line with the required keys, the dominant-kernel roofline timed by
the library's per-launch events, e2e with host-copy byte counts, clocks,
a parity spot check of the timed path, and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--steps", "3", "--warmup", "3", "--batch", "8", "--hmult-batch", "2",
         "--set-a-batch", "64", "--hbm-kernels", "0", "--dnum5-batch", "0", "--sweep", "0",
         "--batch-sweep", "0", "--cpu-members", "1", "--cpu-numpy", "0", "--hmult-check", "0"]


def _run(extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + extra,
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run(SMALL)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["parity_spot_check"] is True
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert r["launches"] == 2 * 3 and r["launch_ms"] > 0          # column pass, fwd + inv
    assert set(r["kernels"]) == {"ntt_col_kernel", "ntt_row_kernel"}
    assert d["gpu_launches"] == 4 * 3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["roundtrip_exact"] is True
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["hmult"]["ops_per_s"] > 0 and d["hrotate"]["ops_per_s"] > 0


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-members", "1"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0
