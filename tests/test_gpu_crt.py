"""Device CRT decomposition / composition (the integer steps of the client-side
encode / decode) against the reference's big-integer
algorithm (rns.py:77-115, ckks.py:194-213) restated in Python ints."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ctx(n, primes):
    from paper_2212_14191_b200.device import DeviceContext
    return DeviceContext.get(n, tuple(primes))


from oracle import oracle as O  # noqa: E402

_ref_decompose = O.crt_decompose          # rns.py:77-90
_ref_centered = O.crt_compose_centered    # rns.py:93-115 + ckks.py:207-213


@pytest.mark.parametrize("limbs", [1, 3, 45])
def test_crt_decompose_float64_rint(limbs):
    """encode: ints = [int(c) for c in np.rint(coeffs)], then c % q per prime;
    ties round to even, magnitudes far past 2^64 reduce exactly."""
    from paper_2212_14191_b200.params import generate_primes
    n = 1 << 12
    primes = generate_primes(n, [30, 29, 28] * 15)[:limbs]
    rng = np.random.default_rng(limbs)
    x = rng.normal(0, 2.0 ** 40, n)
    x[:16] = [0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 0.0, -0.0, 2.0 ** 63, -2.0 ** 63,
              2.0 ** 64, 3.0 * 2.0 ** 200, -(2.0 ** 900), 2.0 ** 1023, 123456789.5, -7.5]
    x[16:32] = rng.normal(0, 1, 16) * 2.0 ** rng.integers(60, 1000, 16)
    got = _ctx(n, primes).crt_decompose(torch.from_numpy(x).cuda(), primes).cpu().numpy()
    want = _ref_decompose([int(c) for c in np.rint(x)], primes)
    assert np.array_equal(got.view(np.uint32), want)


def test_crt_decompose_int64_extremes():
    from paper_2212_14191_b200.params import generate_primes
    n = 1 << 10
    primes = generate_primes(n, [31, 30, 29])
    rng = np.random.default_rng(3)
    x = rng.integers(-(2 ** 63), 2 ** 63 - 1, n, dtype=np.int64)
    x[:6] = [np.iinfo(np.int64).min, np.iinfo(np.int64).max, -1, 0, 1, -19]
    got = _ctx(n, primes).crt_decompose(torch.from_numpy(x).cuda(), primes).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), _ref_decompose([int(c) for c in x], primes))


@pytest.mark.parametrize("preset_limbs", [1, 2, 7, 45, 46])
def test_crt_compose_centered_words_and_float(preset_limbs):
    """decode: the centred CRT value in (-Q/2, Q/2] bit for bit (two's
    complement words) and float(c) exactly (round half to even; +-inf where
    Python's float(int) overflows)."""
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.from_preset("p_default")
    basis = (tuple(p.chain.q) + tuple(p.chain.p))[:preset_limbs]
    n = 1 << 11
    big_q = 1
    for q in basis:
        big_q *= q
    rng = np.random.default_rng(preset_limbs)
    rows = np.stack([rng.integers(0, q, n, dtype=np.uint64).astype(np.uint32) for q in basis])
    # constructed values: small, ties at the 53-bit boundary, +-(Q-1)/2, powers of two
    special = [0, 1, -1, 2 ** 53 + 1, -(2 ** 53 + 1), 2 ** 60 + 2 ** 7, 2 ** 60 + 3 * 2 ** 7,
               2 ** 61 - 1, (big_q - 1) // 2, -((big_q - 1) // 2), 3 ** 200, -(5 ** 300),
               2 ** 1023 + 2 ** 970, 2 ** 1024 - 2 ** 970, 2 ** 1100]
    for j, v in enumerate(special):
        if abs(v) <= (big_q - 1) // 2:
            rows[:, j] = [v % q for q in basis]
    ctx = _ctx(p.n, tuple(p.chain.q) + tuple(p.chain.p))
    t = torch.from_numpy(rows.view(np.int32)).cuda()
    f, w = ctx.crt_compose(t, basis, words=True)
    want = _ref_centered(rows, basis)
    words = w.cpu().numpy().view(np.uint32).astype(object)
    got_ints = []
    for j in range(n):
        v = sum(int(words[k, j]) << (32 * k) for k in range(words.shape[0]))
        if v >> (32 * words.shape[0] - 1):
            v -= 1 << (32 * words.shape[0])
        got_ints.append(v)
    assert got_ints == want
    fl = f.cpu().numpy()
    for j in range(n):
        try:
            ref = float(want[j])
        except OverflowError:
            ref = np.inf if want[j] > 0 else -np.inf
        assert fl[j] == ref or (np.isinf(ref) and fl[j] == ref), (j, want[j], fl[j], ref)


def test_client_encode_decode_roundtrip_device_crt():
    """encode -> decode through the device CRT steps recovers the slots, and
    encode's residues equal the reference's host formula bit for bit."""
    from paper_2212_14191_b200.ckks import CkksContext
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.from_preset("set_a")
    ck = CkksContext(p, seed=11)
    z = np.random.default_rng(2).normal(size=p.n // 2) + 1j * np.random.default_rng(3).normal(
        size=p.n // 2)
    pt = ck.encode(z)
    back = ck.decode(pt)
    assert np.max(np.abs(back - z)) < 1e-6
    # the reference's host path for the same slots
    n = p.n
    idx, cidx = ck._rot_index()
    evals = np.zeros(n, dtype=np.complex128)
    evals[idx] = z * float(p.default_scale)
    evals[cidx] = np.conj(z) * float(p.default_scale)
    coeffs = np.real(np.fft.fft(evals) / n * np.exp(1j * np.pi / n) ** (-np.arange(n)))
    ref_rows = _ref_decompose([int(c) for c in np.rint(coeffs)], p.q_basis(p.l_max))
    coeff_poly = ck.to_coeff(pt.poly)
    assert np.array_equal(coeff_poly.host_rows(), ref_rows)
