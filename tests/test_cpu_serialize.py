"""TFHE1 wire format (ref `serialize.py`) on CPU: blobs written by the
reference itself (tests/golden/tfhe1.npz, make_golden.py) load, and re-dump
byte for byte; header checks raise ParameterError like the reference
(`test_ckks.py:217-255`)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def blobs():
    d = np.load(os.path.join(GOLDEN, "tfhe1.npz"))
    return {k: d[k].tobytes() for k in d.files}


def _params():
    from paper_2212_14191_b200.params import CkksParams
    return CkksParams.generate(n=64, l_max=3, k=2, dnum=2, bit_size=28)


def test_digest_matches_reference(blobs):
    assert _params().digest() == blobs["digest"]


@pytest.mark.parametrize("kind", ["poly", "ct", "pt", "pk", "sk", "swk"])
def test_reference_blobs_roundtrip_bytewise(blobs, kind):
    from paper_2212_14191_b200 import serialize as S
    load, dump = {"poly": (S.load_polynomial, S.dump_polynomial),
                  "ct": (S.load_ciphertext, S.dump_ciphertext),
                  "pt": (S.load_plaintext, S.dump_plaintext),
                  "pk": (S.load_public_key, S.dump_public_key),
                  "sk": (S.load_secret_key, S.dump_secret_key),
                  "swk": (S.load_switching_key, S.dump_switching_key)}[kind]
    digest = blobs["digest"]
    obj = load(blobs[kind], digest)
    assert dump(obj, digest) == blobs[kind]


def test_ciphertext_fields(blobs):
    from fractions import Fraction
    from paper_2212_14191_b200 import serialize as S
    p = _params()
    ct = S.load_ciphertext(blobs["ct"], blobs["digest"])
    assert ct.level == 2 and ct.scale == Fraction(2 ** 40, 3)
    assert ct.b.basis == tuple(p.chain.q[:3]) and ct.b.domain == "ntt"
    assert ct.b.rows.shape == (3, 64) and ct.b.rows.dtype == np.uint32


def test_header_errors(blobs):
    from paper_2212_14191_b200 import serialize as S
    from paper_2212_14191_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        S.load_ciphertext(blobs["ct"], b"\x00" * 8)          # digest mismatch
    with pytest.raises(ParameterError):
        S.load_ciphertext(b"NOPE1" + b"\x00" * 20, blobs["digest"])
    with pytest.raises(ParameterError):
        S.load_ciphertext(blobs["swk"], blobs["digest"])      # wrong kind
    with pytest.raises(ParameterError):
        S.load_ciphertext(blobs["ct"][:200], blobs["digest"])  # truncated
    with pytest.raises(ParameterError):
        S.dump_polynomial(S.load_polynomial(blobs["poly"], blobs["digest"]), b"123")
