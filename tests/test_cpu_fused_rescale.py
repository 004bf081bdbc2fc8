"""CPU check of the fused HMULT+rescale algebra (capi.cu moddown_rescale):
its oracle restatement equals the reference-order rescale(hmult(.)) oracle bit
for bit, for K = 1 and K > 1, alpha = 1 and alpha > 1, full and reduced levels."""

import numpy as np
import pytest

from oracle import oracle as O


@pytest.mark.parametrize("l_max,k,dnum,level", [(3, 1, 4, 3), (5, 3, 3, 5), (5, 2, 3, 2),
                                                (5, 2, 6, 1), (3, 2, 2, 3)])
def test_fused_hmult_rescale_matches_two_step(l_max, k, dnum, level):
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.generate(n=64, l_max=l_max, k=k, dnum=dnum, bit_size=28)
    rng = np.random.default_rng(31 + level + 7 * k)
    basis = tuple(p.chain.q[:level + 1])
    ext = tuple(p.chain.q) + tuple(p.chain.p)
    key = np.stack([np.stack([O.uniform_rows(rng, ext, (p.n,)) for _ in range(2)])
                    for _ in range(p.dnum)])
    c0 = [O.uniform_rows(rng, basis, (2, p.n)) for _ in range(2)]
    c1 = [O.uniform_rows(rng, basis, (2, p.n)) for _ in range(2)]
    hb, ha = O.hmult(c0[0], c0[1], c1[0], c1[1], basis, key, p.chain.q, p.chain.p,
                     p.alpha, p.dnum)
    rb, ra = O.rescale(hb, ha, basis)
    fb, fa = O.hmult_rescale_fused(c0[0], c0[1], c1[0], c1[1], basis, key, p.chain.q,
                                   p.chain.p, p.alpha, p.dnum)
    assert np.array_equal(fb, rb) and np.array_equal(fa, ra)
