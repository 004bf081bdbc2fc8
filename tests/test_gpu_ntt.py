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
    # every prime of the sweep, incl. the 31-bit qs[4] where the lazy [0, 2q)
    # intermediates are tightest (ref test_acceptance.py:97-121)
    qs = golden_params["adhoc"][f"primes_{n}"]["q"]
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
        n, [29, 31, 30, 27, 26])
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


@pytest.mark.parametrize("n,batch", [(1 << 12, 5), (1 << 16, 3)])
def test_batched_apply_eltwise_and_frobenius_vs_oracle(n, batch):
    """The non-transform kernels of batched_apply (ref batch.py:98-127):
    hada_mult / ele_add / ele_sub against a second buffer and forbenius_map
    (NTT-domain automorphism) on device and host buffers, against the oracle."""
    import torch
    from paper_2212_14191_b200.batch import BatchBuffer, batched_apply
    from paper_2212_14191_b200.ntt import TwiddleTable
    from paper_2212_14191_b200.params import generate_primes
    primes = generate_primes(n, [31, 29, 28])
    table = TwiddleTable(n, primes)
    rng = np.random.default_rng(n + 17 * batch)
    x = O.uniform_rows(rng, primes, (batch, n))
    y = O.uniform_rows(rng, primes, (batch, n))
    want = {"hada_mult": O.hada_mult(x, y, primes), "ele_add": O.ele_add(x, y, primes),
            "ele_sub": O.ele_sub(x, y, primes)}
    for kind in ("numpy", "device"):
        conv = (lambda a: a) if kind == "numpy" else \
            (lambda a: torch.from_numpy(a.view(np.int32)).cuda())   # noqa: E731
        back = (lambda a: a) if kind == "numpy" else \
            (lambda a: a.cpu().numpy().view(np.uint32))             # noqa: E731
        bx = BatchBuffer(data=conv(x), basis=primes, domain="ntt")
        by = BatchBuffer(data=conv(y), basis=primes, domain="ntt")
        for op, w in want.items():
            got = batched_apply(bx, op, aux=by, table=table)
            assert np.array_equal(back(got.data), w), (kind, op)
        for r in (1, 3, -1):
            t = O.galois_element(r, n)
            got = batched_apply(bx, "forbenius_map", aux=r, table=table)
            assert np.array_equal(back(got.data), O.apply_automorphism(x, t, primes)), (kind, r)


def test_kernel_timer_counts_ntt_pass_launches():
    """tfhe_profile_enable/read (the bench's per-kernel timing): one N=2^16
    forward + inverse call = one column-pass and one row-pass launch each,
    with positive device times; disabled afterwards (no records)."""
    import torch
    from paper_2212_14191_b200 import _lib
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    n = 1 << 16
    qs = generate_primes(n, [29, 30])
    ctx = DeviceContext.get(n, tuple(qs))
    x = torch.randint(0, 1 << 28, (2, 3, n), dtype=torch.int32, device="cuda")
    with _lib.kernel_timer() as kt:
        f = ctx.ntt(x, qs)
        ctx.ntt(f, qs, inverse=True)
        torch.cuda.synchronize()
    got = {k: v for k, v in kt.times.items()}
    assert got["ntt_col_kernel<fwd>"][0] == 1 and got["ntt_col_kernel<inv>"][0] == 1, got
    assert got["ntt_row_kernel<store>"][0] == 2, got
    assert all(ms > 0 for _, ms in got.values()), got
    with _lib.kernel_timer() as kt2:
        pass
    assert kt2.times == {}


@pytest.mark.parametrize("seed", range(6))
def test_ntt_random_shapes_vs_oracle(seed):
    """Random degrees (2^12..2^16), limb counts, batch sizes (incl. odd and 1)
    and prime widths (26..31 bits): forward equals the oracle, inverse undoes
    it -- every plan (fused n=4096, TS, three-factor) on ragged shapes."""
    import torch
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    rng = np.random.default_rng(1000 + seed)
    n = 1 << int(rng.integers(12, 17))
    limbs = int(rng.integers(1, 4))
    batch = int(rng.choice([1, 2, 3, 5, 7, 9]))
    widths = [int(w) for w in rng.integers(26, 32, limbs)]
    qs = generate_primes(n, widths)
    ctx = DeviceContext.get(n, tuple(qs))
    x = O.uniform_rows(rng, qs, (batch, n))
    f = ctx.ntt(torch.from_numpy(x.view(np.int32)).cuda(), qs)
    got = f.cpu().numpy().view(np.uint32)
    sel = [0, batch - 1]                      # oracle cost: first and last member
    assert np.array_equal(got[:, sel], O.ntt(x[:, sel], qs)), (n, limbs, batch, widths)
    back = ctx.ntt(f, qs, inverse=True).cpu().numpy().view(np.uint32)
    assert np.array_equal(back, x), (n, limbs, batch, widths)
