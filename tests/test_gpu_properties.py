"""Size-independent properties at the bench's full shape (N=2^16, the 45
P-Default chain primes, batch 64), where the CPU oracle is too slow for a
full comparison: linearity of the transform, INTT(NTT(x)) == x, the
convolution theorem against the oracle on sampled rows, bit-exact agreement
with the oracle on a sample of (limb, member) rows, and HMULT linearity in
its first operand's b component (d0, d1 enter after the key switch).
All integer comparisons are exact."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, L, B = 1 << 16, 45, 64


@pytest.fixture(scope="module")
def setup():
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.from_preset("p_default")
    primes = list(p.chain.q)
    ctx = DeviceContext.get(N, tuple(p.chain.q) + tuple(p.chain.p), n_chain=L, n_special=1)
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    q = torch.tensor(primes, dtype=torch.int64, device="cuda").view(L, 1, 1)

    def rand():
        return (torch.randint(0, 1 << 62, (L, B, N), generator=g, device="cuda") % q).to(torch.int32)
    return p, primes, ctx, q, rand


def _add(x, y, q):
    return ((x.to(torch.int64) + y.to(torch.int64)) % q).to(torch.int32)


def test_linearity_and_roundtrip(setup):
    p, primes, ctx, q, rand = setup
    x, y = rand(), rand()
    fx, fy = ctx.ntt(x, primes), ctx.ntt(y, primes)
    fxy = ctx.ntt(_add(x, y, q), primes)
    assert torch.equal(fxy, _add(fx, fy, q))
    assert torch.equal(ctx.ntt(fx, primes, inverse=True), x)


def test_sampled_rows_and_convolution_vs_oracle(setup):
    from oracle import oracle as O
    p, primes, ctx, q, rand = setup
    x, y = rand(), rand()
    fx, fy = ctx.ntt(x, primes), ctx.ntt(y, primes)
    rng = np.random.default_rng(3)
    for limb, member in zip(rng.integers(0, L, 4), rng.integers(0, B, 4)):
        xs = x[limb, member].cpu().numpy().view(np.uint32)[None]
        got = fx[limb, member].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, O.ntt(xs, [primes[limb]])[0]), (limb, member)
    # convolution theorem: INTT(NTT(x) * NTT(y)) is the negacyclic product;
    # checked against the oracle's transform of the same rows
    prod = ctx.eltwise(2, fx, fy, primes)   # hada_mult
    conv = ctx.ntt(prod, primes, inverse=True)
    limb, member = 7, 11
    xs = x[limb, member].cpu().numpy().view(np.uint32)[None]
    ys = y[limb, member].cpu().numpy().view(np.uint32)[None]
    qq = primes[limb]
    want = O.intt((O.ntt(xs, [qq]).astype(np.uint64) * O.ntt(ys, [qq]) % qq).astype(np.uint32),
                  [qq])[0]
    assert np.array_equal(conv[limb, member].cpu().numpy().view(np.uint32), want)


def test_hmult_additive_in_d0(setup):
    """The key switch sees only d2 = a0 a1; d0 = b0 b1 and d1 = a0 b1 + b0 a1
    are added after it, so replacing b0 by b0 + delta shifts the outputs by
    exactly (delta b1, delta a1)."""
    from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext
    p, primes, ctx, q, rand = setup
    ck = CkksContext(p)
    Bh = 4
    c0 = torch.stack([rand()[:, :Bh], rand()[:, :Bh]]).contiguous()
    c1 = torch.stack([rand()[:, :Bh], rand()[:, :Bh]]).contiguous()
    key = torch.stack([torch.stack([rand()[:, 0], rand()[:, 0]]) for _ in range(p.dnum)])
    key = torch.cat([key, key[:, :, :1]], dim=2).contiguous()   # + the special row
    delta = rand()[:, :Bh].contiguous()
    c0d = c0.clone()
    c0d[0] = _add(c0[0], delta, q)
    base = ck.hmult_batch(CiphertextBatch(c0, p.l_max), CiphertextBatch(c1, p.l_max), key).data
    shifted = ck.hmult_batch(CiphertextBatch(c0d, p.l_max), CiphertextBatch(c1, p.l_max), key).data
    db = ctx.eltwise(2, delta, c1[0].contiguous(), primes)   # d0 = b0 b1 moves by delta b1
    da = ctx.eltwise(2, delta, c1[1].contiguous(), primes)   # d1 = a0 b1 + b0 a1 by delta a1
    assert torch.equal(shifted[0], _add(base[0], db, q))
    assert torch.equal(shifted[1], _add(base[1], da, q))


def test_small_n_full_shape_roundtrip_and_samples():
    """The Set_A-shaped resident small-n kernels at a large batch (N=2^12,
    2 limbs, B=8192, 8192 tiles per limb over all SMs): roundtrip exact and
    sampled rows equal the oracle."""
    from oracle import oracle as O
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    n, B = 1 << 12, 8192
    primes = generate_primes(n, [29, 29])
    ctx = DeviceContext.get(n, tuple(primes))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q = torch.tensor(primes, dtype=torch.int64, device="cuda").view(2, 1, 1)
    x = (torch.randint(0, 1 << 62, (2, B, n), generator=g, device="cuda") % q).to(torch.int32)
    f = ctx.ntt(x, primes)
    assert torch.equal(ctx.ntt(f, primes, inverse=True), x)
    for limb, member in ((0, 0), (1, 4097), (0, B - 1), (1, 1234)):
        xs = x[limb, member].cpu().numpy().view(np.uint32)[None]
        assert np.array_equal(f[limb, member].cpu().numpy().view(np.uint32),
                              O.ntt(xs, [primes[limb]])[0]), (limb, member)
