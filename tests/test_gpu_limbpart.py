"""GPU parity of the limb-partitioned mode on ONE device.

The G ranks of `paper_2212_14191_b200.limbpart` are simulated sequentially on
cuda:0 (`simulate` / `sim_*`: the all-gather and broadcast become
concatenation); every rank's kernels are the real ones
(tfhe_tensor_product, tfhe_keyswitch_part, tfhe_rescale_part, tfhe_ntt,
tfhe_automorphism).  Concatenated rank outputs must equal the unpartitioned
batched operators -- themselves pinned to the reference's golden outputs in
test_gpu_ckks.py -- bit for bit, and the small case is also checked against
the CPU oracle directly.  Covers the TS tensor-core path (n >= 2^14, alpha 1
and 2, K = 1 and 8) and the small-n path, uneven shards and empty ranks.
"""

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

CASES = [("small", 5, 2), ("small", 5, 4), ("small", 2, 4), ("n16", 3, 2), ("n16", 3, 3),
         ("set_c", 7, 3), ("set_c", 4, 8)]


def _params(kind):
    from paper_2212_14191_b200.params import CkksParams
    if kind == "small":
        return CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30)
    if kind == "n16":
        return CkksParams.generate(n=1 << 16, l_max=3, k=1, dnum=4, bit_size=28)
    return CkksParams.from_preset(kind)


_CTX = {}


def _ctx(kind):
    from paper_2212_14191_b200.ckks import CkksContext
    if kind not in _CTX:
        _CTX[kind] = CkksContext(_params(kind))
    return _CTX[kind]


def _batch(p, level, batch, seed):
    rng = np.random.default_rng(seed)
    basis = p.chain.q[:level + 1]
    ct = lambda: np.stack([synth.rows(rng, basis, (batch, p.n)) for _ in range(2)])  # noqa
    key = synth.switching_key(rng, p.chain.q, p.chain.p, p.n, p.dnum)
    return ct(), ct(), key


@pytest.mark.parametrize("kind,level,world", CASES)
def test_limb_partitioned_ops_equal_unpartitioned(kind, level, world):
    from paper_2212_14191_b200 import limbpart as LP
    from paper_2212_14191_b200.ckks import CiphertextBatch
    ck = _ctx(kind)
    p = ck.params
    B = 2
    c0, c1, key = _batch(p, level, B, 1000 * level + world)
    dev = lambda a: torch.from_numpy(a.view(np.int32)).cuda()  # noqa: E731
    t0, t1, tk = dev(c0), dev(c1), dev(key)
    cb0, cb1 = CiphertextBatch(t0, level), CiphertextBatch(t1, level)
    evs = LP.simulate(ck, world)

    want = ck.hmult_batch(cb0, cb1, tk).data
    got = LP.sim_hmult(evs, t0, t1, level, tk)
    assert torch.equal(got, want), "hmult"

    want = ck.key_switch_batch(t0[1].contiguous(), level, tk)
    got = LP.sim_key_switch(evs, t0[1].contiguous(), level, tk)
    assert torch.equal(got, want), "key_switch"

    want = ck.hrotate_batch(cb0, 1, tk).data
    got = LP.sim_hrotate(evs, t0, level, 1, tk)
    assert torch.equal(got, want), "hrotate"

    if level >= 1:
        want = ck.rescale_batch(cb0).data
        got = LP.sim_rescale(evs, t0, level)
        assert torch.equal(got, want), "rescale"

    if kind == "small":   # and straight against the CPU oracle
        from oracle import oracle as O
        basis = tuple(p.chain.q[:level + 1])
        hb, ha = O.hmult(c0[0], c0[1], c1[0], c1[1], basis, key, p.chain.q, p.chain.p,
                         p.alpha, p.dnum)
        got = LP.sim_hmult(evs, t0, t1, level, tk).cpu().numpy().view(np.uint32)
        assert np.array_equal(got[0], hb) and np.array_equal(got[1], ha), "hmult vs oracle"
