"""Client-side ops (keygen / relin / rotation / conjugation keys, encode,
encrypt, decrypt, decode) on the device path reproduce the reference's
outputs for the same seed bit for bit (tests/golden/client.json, written by
make_golden.py from the reference itself), and a full
encrypt -> hmult -> rescale -> decrypt round trip decodes to the same slots."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def _params(name):
    from paper_2212_14191_b200.params import CkksParams
    if name == "small":
        return CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30)
    return CkksParams.from_preset(name)


@pytest.mark.parametrize("name", ["small", "default", "set_a"])
def test_client_ops_match_reference(name):
    from paper_2212_14191_b200.ckks import CkksContext
    with open(os.path.join(GOLDEN, "client.json")) as fh:
        r = json.load(fh)[name]
    params = _params(name)
    ctx = CkksContext(params, backend="butterfly", seed=99)
    z = np.random.default_rng(5).uniform(-1, 1, params.slots) \
        + 1j * np.random.default_rng(6).uniform(-1, 1, params.slots)
    sk, pk = ctx.keygen()
    rlk = ctx.make_relin_key(sk)
    rk = ctx.make_rotation_key(sk, 1)
    ck = ctx.make_conjugation_key(sk)
    pt = ctx.encode(z)
    ct = ctx.encrypt(pk, pt)
    dec = ctx.decrypt_decode(sk, ct)
    assert _sha(sk.s.rows) == r["sk"]
    assert (_sha(pk.b.rows), _sha(pk.a.rows)) == (r["pk_b"], r["pk_a"])
    assert _sha(pt.poly.rows) == r["pt"]
    assert [pt.scale.numerator, pt.scale.denominator] == r["scale"]
    assert (_sha(ct.b.rows), _sha(ct.a.rows)) == (r["ct_b"], r["ct_a"])
    for kname, key in (("rlk", rlk), ("rk", rk), ("ck", ck)):
        assert [[_sha(b.rows), _sha(a.rows)] for b, a in key.pairs] == r[kname], kname
    np.testing.assert_allclose(dec.real[:16], r["dec_re"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(dec.imag[:16], r["dec_im"], rtol=0, atol=1e-12)
    assert np.max(np.abs(dec - z)) < 2 ** -20
    m = ctx.rescale(ctx.hmult(ct, ct, rlk))
    assert (_sha(m.b.rows), _sha(m.a.rows)) == (r["hmult_rescale_b"], r["hmult_rescale_a"])
    dm = ctx.decrypt_decode(sk, m)
    np.testing.assert_allclose(dm.real[:16], r["dec_sq_re"], rtol=0, atol=1e-12)
    if name != "set_a":   # Set_A's 54-bit Q cannot hold a 2^80-scaled product
        assert np.max(np.abs(dm - z * z)) < 2 ** -15
