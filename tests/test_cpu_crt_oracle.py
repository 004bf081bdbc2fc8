"""The oracle's CRT restatement (oracle.crt_decompose / encode_ints /
crt_compose_centered) against the reference's own functions
(rns.crt_decompose / crt_compose, CkksContext._centered), imported
read-only when /root/reference is present, and against its SPEC known answer
(CRT 23 <-> (6, 10) over {17, 13})."""
import os
import sys

import numpy as np
import pytest

from oracle import oracle as O

REF = "/root/reference/pkg/src"


def test_spec_known_answer():
    assert O.crt_decompose([23], (17, 13)).ravel().tolist() == [6, 10]
    assert O.crt_compose_centered(np.array([[6], [10]]), (17, 13)) == [23]        # 23 <= 110
    assert O.crt_compose_centered(np.array([[200 % 17], [200 % 13]]), (17, 13)) == [200 - 221]


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")
def test_against_reference_functions():
    sys.path.insert(0, REF)
    try:
        from rnsckks import rns as R
        from rnsckks.params import generate_primes
    finally:
        sys.path.remove(REF)
    basis = tuple(generate_primes(64, [30, 29, 28, 31]))
    rng = np.random.default_rng(3)
    ints = [int(v) for v in rng.integers(-(2 ** 62), 2 ** 62, 64)] + [3 ** 80, -(5 ** 50), 0]
    ints = ints[:64]
    assert np.array_equal(O.crt_decompose(ints, basis), R.crt_decompose(ints, basis).rows)
    rows = np.stack([rng.integers(0, q, 64, dtype=np.uint64).astype(np.uint32) for q in basis])
    poly = R.RnsPolynomial(rows=rows, basis=basis, domain=R.COEFF)
    big_q = 1
    for q in basis:
        big_q *= q
    want = [c - big_q if c > big_q // 2 else c for c in R.crt_compose(poly)]
    assert O.crt_compose_centered(rows, basis) == want
    x = rng.normal(0, 2.0 ** 40, 64)
    x[:4] = [0.5, 1.5, -2.5, 2.0 ** 70]
    assert O.encode_ints(x) == [int(c) for c in np.rint(x)]
