"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) runs: tools/sanitize.sh.  Each op is
checked against the CPU oracle so a silent corruption also fails."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2212_14191_b200 import _lib  # noqa: E402
from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext  # noqa: E402
from paper_2212_14191_b200.device import DeviceContext  # noqa: E402
from paper_2212_14191_b200.params import CkksParams, generate_primes  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def main():
    rng = np.random.default_rng(1)
    # NTT: resident small-n (2^12), TS stage-2-only (2^13), TS (2^14)
    for n, B in ((1 << 12, 3), (1 << 13, 2), (1 << 14, 2)):
        qs = generate_primes(n, [30, 31])
        ctx = DeviceContext.get(n, tuple(qs))
        x = O.uniform_rows(rng, qs, (B, n))
        f = ctx.ntt(dev(x), qs)
        assert np.array_equal(host(f), O.ntt(x, qs)), n
        assert np.array_equal(host(ctx.ntt(f, qs, inverse=True)), x), n
        y = O.uniform_rows(rng, qs, (B, n))
        assert np.array_equal(host(ctx.eltwise(_lib.OP_MUL, dev(x), dev(y), qs)),
                              O.hada_mult(x, y, qs))
        assert np.array_equal(host(ctx.automorphism(dev(x), 5, True, qs)),
                              O.apply_automorphism(x, 5, qs))
        print("ntt/eltwise/automorphism ok", n, flush=True)
    # CKKS pipelines: small-n (set_a) and TS (set_c: alpha = 2, K = 8, tensor-core bconv)
    for preset, level in (("set_a", 1), ("set_c", 3)):
        p = CkksParams.from_preset(preset)
        ck = CkksContext(p)
        basis = tuple(p.chain.q[:level + 1])
        ext = tuple(p.chain.q) + tuple(p.chain.p)
        c0 = np.stack([O.uniform_rows(rng, basis, (2, p.n)) for _ in range(2)])
        c1 = np.stack([O.uniform_rows(rng, basis, (2, p.n)) for _ in range(2)])
        key = np.stack([np.stack([O.uniform_rows(rng, ext, (p.n,)) for _ in range(2)])
                        for _ in range(p.dnum)])
        got = host(ck.hmult_rescale_batch(CiphertextBatch(dev(c0), level),
                                          CiphertextBatch(dev(c1), level), dev(key)).data)
        for m in range(2):
            hb, ha = O.hmult(c0[0][:, m], c0[1][:, m], c1[0][:, m], c1[1][:, m], basis, key,
                             p.chain.q, p.chain.p, p.alpha, p.dnum)
            rb, ra = O.rescale(hb, ha, basis)
            assert np.array_equal(got[0][:, m], rb) and np.array_equal(got[1][:, m], ra)
        got = host(ck.hrotate_batch(CiphertextBatch(dev(c0), level), 1, dev(key)).data)
        rb, ra = O.hrotate(c0[0][:, 0], c0[1][:, 0], 1, basis, key, p.chain.q, p.chain.p,
                           p.alpha, p.dnum)
        assert np.array_equal(got[0][:, 0], rb) and np.array_equal(got[1][:, 0], ra)
        print("ckks ok", preset, flush=True)
    # N = 2^16 three-factor passes (column + row) and the grouped key switch
    # (column pass + EPI_KS_ACC row pass) on a 4-limb chain at level 3
    n = 1 << 16
    qs = generate_primes(n, [29, 30, 31])
    ctx = DeviceContext.get(n, tuple(qs))
    x = O.uniform_rows(rng, qs, (1, n))
    f = ctx.ntt(dev(x), qs)
    assert np.array_equal(host(f), O.ntt(x, qs))
    assert np.array_equal(host(ctx.ntt(f, qs, inverse=True)), x)
    print("ntt p3 ok", flush=True)
    from paper_2212_14191_b200.params import generate_chain_widths
    p = CkksParams(n=n, l_max=3, k=1, dnum=4, chain=generate_chain_widths(n, [29] * 4, [30]))
    if True:
        ck = CkksContext(p)
        level = p.l_max
        basis = tuple(p.chain.q[:level + 1])
        ext = tuple(p.chain.q) + tuple(p.chain.p)
        c0 = np.stack([O.uniform_rows(rng, basis, (1, p.n)) for _ in range(2)])
        c1 = np.stack([O.uniform_rows(rng, basis, (1, p.n)) for _ in range(2)])
        key = np.stack([np.stack([O.uniform_rows(rng, ext, (p.n,)) for _ in range(2)])
                        for _ in range(p.dnum)])
        got = host(ck.hmult_rescale_batch(CiphertextBatch(dev(c0), level),
                                          CiphertextBatch(dev(c1), level), dev(key)).data)
        hb, ha = O.hmult(c0[0][:, 0], c0[1][:, 0], c1[0][:, 0], c1[1][:, 0], basis, key,
                         p.chain.q, p.chain.p, p.alpha, p.dnum)
        rb, ra = O.rescale(hb, ha, basis)
        assert np.array_equal(got[0][:, 0], rb) and np.array_equal(got[1][:, 0], ra)
        print("ckks p3 ok", flush=True)
    # tensor-core base conversion (chunk pairs, TMA tensor stores), incl. a
    # non-canonical copy source (fixup launch)
    n = 1 << 12
    primes = generate_primes(n, [30] * 10 + [29] * 50)[:9 + 45]
    src, dst = primes[:9], primes[9:] + primes[:9]
    ctx = DeviceContext.get(n, tuple(primes))
    x = O.uniform_rows(rng, src, (2, n))
    x[3, 1, 7] = 0xFFFFFFF0
    got = host(ctx.bconv(dev(x), src, dst))
    assert np.array_equal(got, O.fast_basis_conv(x, tuple(src), tuple(dst)))
    print("bconv ok", flush=True)
    # client-side CRT
    c = rng.normal(0, 2.0 ** 50, n)
    rows = host(ctx.crt_decompose(torch.from_numpy(c).cuda(), primes[:5]))
    assert np.array_equal(rows, np.array([[int(v) % q for v in np.rint(c)] for q in primes[:5]],
                                         dtype=np.uint32))
    fl = ctx.crt_compose(dev(rows), primes[:5]).cpu().numpy()
    assert np.array_equal(fl, np.rint(c))
    print("crt ok", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE_SMOKE_OK")


if __name__ == "__main__":
    main()
