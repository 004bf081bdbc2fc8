"""GPU parity: tensor-core NTT/INTT vs the golden vectors and the CPU oracle.

Bit-exact (integer path): every comparison is np.array_equal.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O
import synth

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "ntt_small.npz"))


@pytest.mark.parametrize("n", [16, 64, 256, 1024, 4096])
def test_transform_rows_golden_small(n, small, golden_params):
    from paper_2212_14191_b200 import ntt
    qs = golden_params["adhoc"][f"primes_{n}"]["q"]
    table = ntt.TwiddleTable(n, qs)
    for q in qs:
        x = small[f"x_{n}_{q}"]
        got = ntt.transform_rows(x, q, table, "segmented")
        assert np.array_equal(got, small[f"fwd_{n}_{q}"]), (n, q, "fwd")
        got = ntt.transform_rows(x, q, table, "segmented", inverse=True)
        assert np.array_equal(got, small[f"inv_{n}_{q}"]), (n, q, "inv")


@pytest.mark.parametrize("n", [1 << 13, 1 << 14, 1 << 15, 1 << 16])
def test_transform_rows_golden_large(n, golden_params):
    from paper_2212_14191_b200 import ntt
    with open(os.path.join(GOLDEN, "ntt_large.json")) as fh:
        rec = json.load(fh)
    qs = golden_params["adhoc"][f"primes_{n}"]["q"][:3]
    table = ntt.TwiddleTable(n, qs)
    for q in qs:
        x = synth.ntt_rows(n, q, rows=2)
        f = ntt.transform_rows(x, q, table, "segmented")
        i = ntt.transform_rows(x, q, table, "segmented", inverse=True)
        r = rec[f"{n}_{q}"]
        assert f[0, :8].tolist() == r["fwd_head"]
        assert _sha(f) == r["fwd"], (n, q)
        assert _sha(i) == r["inv"], (n, q)


@pytest.mark.parametrize("n,batch", [(1 << 12, 64), (1 << 16, 4), (1 << 16, 37), (1 << 15, 3)])
def test_batched_multilimb_vs_oracle(n, batch):
    import torch
    from paper_2212_14191_b200.device import DeviceContext
    primes = __import__("paper_2212_14191_b200.params", fromlist=["x"]).generate_primes(
        n, [29, 28, 30, 27, 26])
    ctx = DeviceContext.get(n, primes)
    rng = np.random.default_rng(n + batch)
    x = O.uniform_rows(rng, primes, (batch, n))
    xd = torch.from_numpy(x.view(np.int32)).cuda()
    f = ctx.ntt(xd, primes).cpu().numpy().view(np.uint32)
    assert np.array_equal(f, O.ntt(x, primes))
    b = ctx.ntt(torch.from_numpy(f.view(np.int32)).cuda(), primes, inverse=True)
    assert np.array_equal(b.cpu().numpy().view(np.uint32), x)


@pytest.mark.parametrize("n,batch,rows,kind", [(1 << 16, 64, 12, "pinned"),
                                               (1 << 16, 64, 7, "numpy"),
                                               (1 << 12, 64, 3, "numpy"),
                                               (1 << 16, 200, 2, "pinned")])
def test_batched_apply_host_streaming(n, batch, rows, kind):
    """batched_apply on host buffers streams through tfhe_ntt_host in chunks
    (several chunks, slot reuse, ragged last chunk): equal to the device path
    and to the oracle on a sample of rows, and INTT(NTT(x)) == x."""
    import torch
    from paper_2212_14191_b200.batch import BatchBuffer, batched_apply
    from paper_2212_14191_b200.ntt import TwiddleTable
    from paper_2212_14191_b200.params import generate_primes
    primes = generate_primes(n, [29] * rows)
    table = TwiddleTable(n, primes)
    rng = np.random.default_rng(rows * batch)
    x = O.uniform_rows(rng, primes, (batch, n))
    if kind == "pinned":
        data = torch.from_numpy(x.view(np.int32)).pin_memory()
    else:
        data = x
    f = batched_apply(BatchBuffer(data=data, basis=primes, domain="coeff"), "ntt", table=table)
    fh = f.data.numpy().view(np.uint32) if kind == "pinned" else f.data
    dev = table.context().ntt(torch.from_numpy(x.view(np.int32)).cuda(), primes)
    assert np.array_equal(fh, dev.cpu().numpy().view(np.uint32))
    assert np.array_equal(fh[:, :2], O.ntt(x[:, :2], primes))
    b = batched_apply(f, "intt", table=table)
    bh = b.data.numpy().view(np.uint32) if kind == "pinned" else b.data
    assert np.array_equal(bh, x)
