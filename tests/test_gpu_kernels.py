"""GPU parity of the element-wise, automorphism and base-conversion operators.

`kernels.*` and `rns.fast_basis_conv` run on the device (tfhe_eltwise,
tfhe_automorphism, tfhe_bconv = the int8 tensor-core base conversion) and
must equal the reference's outputs recorded in tests/golden/kernels.npz
(make_golden.py, reference `kernels.py:33-117`, `rns.py:118-152`) bit for
bit; wider base conversions (up to 16 sources x 128 targets, ragged
coefficient counts, shared primes) are checked against the CPU oracle.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def k():
    return np.load(os.path.join(GOLDEN, "kernels.npz"))


def test_eltwise_and_automorphism_golden(k):
    from paper_2212_14191_b200 import kernels as K
    from paper_2212_14191_b200.rns import RnsPolynomial
    basis = tuple(int(q) for q in k["basis"])
    a = RnsPolynomial(rows=k["a"], basis=basis, domain="ntt")
    b = RnsPolynomial(rows=k["b"], basis=basis, domain="ntt")
    assert np.array_equal(K.ele_add(a, b).rows, k["add"])
    assert np.array_equal(K.ele_sub(a, b).rows, k["sub"])
    assert np.array_equal(K.hada_mult(a, b).rows, k["mul"])
    assert np.array_equal(K.scalar_rows_mult(a, [3, 5, 1 << 29]).rows, k["scal"])
    assert np.array_equal(K.negate(a).rows, k["neg"])
    n = a.n
    c = RnsPolynomial(rows=k["a"], basis=basis, domain="coeff")
    for t in (5, 25, 2 * n - 1, K.galois_element(3, n)):
        assert np.array_equal(K.apply_automorphism(a, t).rows, k[f"aut_ntt_{t}"]), t
        assert np.array_equal(K.apply_automorphism(c, t).rows, k[f"aut_coeff_{t}"]), t


def test_fast_basis_conv_golden(k):
    from paper_2212_14191_b200.rns import RnsPolynomial, fast_basis_conv
    for i in range(4):
        src = tuple(int(v) for v in k[f"bconv_src_{i}"])
        tgt = tuple(int(v) for v in k[f"bconv_tgt_{i}"])
        got = fast_basis_conv(RnsPolynomial(rows=k[f"bconv_in_{i}"], basis=src, domain="coeff"),
                              tgt)
        assert np.array_equal(got.rows, k[f"bconv_out_{i}"]), i


@pytest.mark.parametrize("n,batch,n_src,n_dst,shared", [
    (1 << 16, 3, 1, 45, 0), (1 << 16, 2, 2, 40, 2), (1 << 14, 5, 8, 16, 1),
    (1 << 12, 7, 9, 54, 3), (1 << 12, 3, 16, 128, 4), (256, 3, 5, 33, 0), (64, 1, 3, 7, 1)])
def test_bconv_tensor_core_vs_oracle(n, batch, n_src, n_dst, shared):
    """tfhe_bconv over (n_src, batch, n) -> (n_dst, batch, n); `shared` of the
    targets are source primes (copied through)."""
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    widths = [30] * 10 + [29] * 50 + [28] * 50 + [27] * 40
    primes = generate_primes(n, widths[:n_src + n_dst])
    src = primes[:n_src]
    dst = list(src[:shared]) + list(primes[n_src:n_src + n_dst - shared])
    ctx = DeviceContext.get(n, tuple(primes[:n_src + n_dst]))
    rng = np.random.default_rng(n + n_src * 131 + n_dst)
    x = O.uniform_rows(rng, src, (batch, n))
    out = ctx.bconv(torch.from_numpy(x.view(np.int32)).cuda(), src, dst)
    got = out.cpu().numpy().view(np.uint32)
    want = O.fast_basis_conv(x, tuple(src), tuple(dst))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,batch,n_src,n_dst,shared,bad", [
    (1 << 12, 7, 9, 54, 3, "one"), (1 << 12, 7, 9, 54, 3, "none"), (1 << 14, 4, 4, 40, 4, "all"),
    (1 << 16, 2, 9, 54, 9, "one")])
def test_bconv_copy_through_non_canonical(n, batch, n_src, n_dst, shared, bad):
    """rns.py:140-142 copies a shared prime's row as is, even residues >= q
    (RnsPolynomial does not enforce the bound).  The tensor-store kernel
    computes copies as a mod q and a fixup launch restores the raw rows when a
    copy source was non-canonical: bit-exact either way."""
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    widths = [30] * 10 + [29] * 50 + [28] * 50 + [27] * 40
    primes = generate_primes(n, widths[:n_src + n_dst])
    src = primes[:n_src]
    dst = list(primes[n_src:n_src + n_dst - shared]) + list(src[:shared])   # copies last
    ctx = DeviceContext.get(n, tuple(primes[:n_src + n_dst]))
    rng = np.random.default_rng(7 * n + n_src)
    x = O.uniform_rows(rng, src, (batch, n))
    if bad == "one":
        x[1, batch - 1, n - 3] = 0xFFFFFFF0          # one residue >= q in a copy source
    elif bad == "all":
        x[:shared] |= np.uint32(1 << 31)             # every copy-source residue >= q
    out = ctx.bconv(torch.from_numpy(x.view(np.int32)).cuda(), src, dst)
    got = out.cpu().numpy().view(np.uint32)
    want = O.fast_basis_conv(x, tuple(src), tuple(dst))
    assert np.array_equal(got, want)
    # the next launch (canonical input) must not see a stale fixup flag
    x2 = O.uniform_rows(rng, src, (batch, n))
    got2 = ctx.bconv(torch.from_numpy(x2.view(np.int32)).cuda(), src, dst).cpu().numpy()
    assert np.array_equal(got2.view(np.uint32), O.fast_basis_conv(x2, tuple(src), tuple(dst)))


@pytest.mark.parametrize("n,t", [(1 << 16, 5), (1 << 16, 25), (1 << 16, 63), (1 << 16, 5 + (1 << 16)),
                                 (1 << 12, 5), (1 << 13, 61), (1 << 16, 625), (1 << 16, (1 << 17) - 1)])
def test_ntt_automorphism_vs_oracle(n, t):
    """NTT-domain automorphism at full size: small multipliers take the
    smem-window kernel, others the gather; both equal the oracle's gather."""
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.params import generate_primes
    primes = generate_primes(n, [29, 28])
    ctx = DeviceContext.get(n, tuple(primes))
    rng = np.random.default_rng(t % 1000 + n)
    x = O.uniform_rows(rng, primes, (3, n))
    got = ctx.automorphism(torch.from_numpy(x.view(np.int32)).cuda(), t, True, primes)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), O.apply_automorphism(x, t, tuple(primes), "ntt"))
