"""bench.py's multi-GPU entry: `--gpus N` outside torchrun starts N ranks
itself (torch.distributed.run on 127.0.0.1) and rank 0 reports all of them.
Run on CPU with --dry-run (gloo rank plumbing, no GPU work)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_2_spawns_two_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2
    assert sorted(r["rank"] for r in rec["ranks"]) == [0, 1]
    assert sorted(r["local_rank"] for r in rec["ranks"]) == [0, 1]
    assert len({r["pid"] for r in rec["ranks"]}) == 2
