"""TFHE1 blobs straight into device batches: load_ciphertext_batch /
load_switching_key_device equal the host decode, and an HMULT on the loaded
batch + key equals the CPU oracle bit for bit."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
import synth

pytestmark = pytest.mark.gpu


def test_device_loaders_and_hmult():
    from oracle import oracle as O
    from paper_2212_14191_b200 import serialize as S
    from paper_2212_14191_b200.ckks import Ciphertext, CkksContext, SwitchingKey
    from paper_2212_14191_b200.params import CkksParams
    from paper_2212_14191_b200.rns import RnsPolynomial
    p = CkksParams.from_preset("set_b")
    ck = CkksContext(p)
    digest = p.digest()
    rng = np.random.default_rng(31)
    lvl = p.l_max
    basis = tuple(p.q_basis(lvl))
    ext = tuple(p.chain.q) + tuple(p.chain.p)
    poly = lambda rows, b=basis: RnsPolynomial(rows=rows, basis=b, domain="ntt")  # noqa
    cts = [[synth.rows(rng, basis, (p.n,)) for _ in range(2)] for _ in range(5)]
    blobs = [S.dump_ciphertext(Ciphertext(b=poly(b), a=poly(a), scale=1, level=lvl), digest)
             for b, a in cts]
    key = synth.switching_key(rng, p.chain.q, p.chain.p, p.n, p.dnum)
    swk = SwitchingKey(pairs=tuple((poly(key[j, 0], ext), poly(key[j, 1], ext))
                                   for j in range(p.dnum)))
    kblob = S.dump_switching_key(swk, digest)

    cb = S.load_ciphertext_batch(blobs, digest)
    host = np.stack([np.stack([c[0] for c in cts], axis=1), np.stack([c[1] for c in cts], axis=1)])
    assert cb.level == lvl and np.array_equal(cb.data.cpu().numpy().view(np.uint32), host)
    kd = S.load_switching_key_device(kblob, digest, ext)
    assert torch.equal(kd, ck.device_key(swk))

    out = ck.hmult_batch(cb, cb, kd).data.cpu().numpy().view(np.uint32)
    hb, ha = O.hmult(host[0], host[1], host[0], host[1], basis, key, p.chain.q, p.chain.p,
                     p.alpha, p.dnum)
    assert np.array_equal(out[0], hb) and np.array_equal(out[1], ha)
    again = S.dump_ciphertext_batch(cb, basis, digest)
    assert again == blobs
