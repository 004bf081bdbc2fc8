"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `rnsckks` read-only, evaluates the hot-path operators on seeded
synthetic inputs and writes small fixtures next to this script:

* params.json     primes, psi and plans of every preset (+ p_default, the
                  paper-Default shape) and of the test fixtures' ad-hoc chains
* ntt_small.npz   transform_rows fwd/inv at n = 16..4096 (butterfly backend;
                  ntt.py:347) plus ntt_oracle rows, full arrays
* ntt_large.json  n = 2^15, 2^16 rows: seed + sha256 of the reference outputs
* kernels.npz     ele_add/ele_sub/hada_mult/scalar_rows_mult/negate,
                  automorphisms (ntt + coeff domain), fast_basis_conv
* ckks_small.npz  hmult / key_switch / rescale / hrotate / hconjugate / hadd /
                  hsub / cmult with synthetic uniform keys, at small_params
                  (conftest.py:13-18), the `default` and `set_a` presets, and a
                  reduced level (ragged GKS slices, test_ckks.py:179-186)
* ckks_large.json the same ops at N=2^16 (a reduced-level resnet20 chain and
                  a 3-limb N=2^16 chain): seed + sha256 of the outputs

The GPU box has no /root/reference; tests there regenerate inputs from the
recorded seeds (tests/golden/synth.py) and compare against these files.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import synth  # noqa: E402

from rnsckks import kernels as K  # noqa: E402
from rnsckks import ntt as RN  # noqa: E402
from rnsckks import params as RP  # noqa: E402
from rnsckks.ckks import Ciphertext, CkksContext, SwitchingKey  # noqa: E402
from rnsckks.rns import COEFF, NTT, RnsPolynomial, fast_basis_conv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def chain_doc(params):
    c = params.chain
    return {"n": params.n, "l_max": params.l_max, "k": params.k, "dnum": params.dnum,
            "q": list(c.q), "p": list(c.p),
            "psi": {str(r): c.roots[r].psi for r in c.q + c.p},
            "plan": [params.plan.n1, params.plan.n2]}


def p_default():
    chain = RP.generate_chain_widths(1 << 16, [29] * 17 + [28] * 28, [29])
    return RP.CkksParams(n=1 << 16, l_max=44, k=1, dnum=45, chain=chain)


def p_dnum5():
    chain = RP.generate_chain_widths(1 << 16, [29] * 17 + [28] * 28, [30] * 9)
    return RP.CkksParams(n=1 << 16, l_max=44, k=9, dnum=5, chain=chain)


def make_params():
    doc = {"presets": {}, "adhoc": {}}
    for name in RP.PRESETS:
        doc["presets"][name] = chain_doc(RP.CkksParams.from_preset(name))
    doc["presets"]["p_default"] = chain_doc(p_default())
    doc["presets"]["p_dnum5"] = chain_doc(p_dnum5())
    doc["adhoc"]["small_params"] = chain_doc(
        RP.CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30))
    for n in (16, 64, 256, 1024, 4096, 1 << 13, 1 << 14, 1 << 15, 1 << 16):
        qs = RP.generate_primes(n, [30, 24, 26, 28, 31])
        doc["adhoc"][f"primes_{n}"] = {
            "q": qs, "psi": [RP.find_negacyclic_root(q, n) for q in qs],
            "plan": [RP.build_ntt_plan(n).n1, RP.build_ntt_plan(n).n2]}
    doc["known_answers"] = {
        "find_negacyclic_root_17_4": RP.find_negacyclic_root(17, 4),
        "galois_1_64": K.galois_element(1, 64),
        "split_0x12345678": [int(v) for v in RP.split_bytes(np.array([0x12345678]))[:, 0]],
    }
    with open(os.path.join(HERE, "params.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    return doc


def make_ntt_small(doc):
    out = {}
    for n in (16, 64, 256, 1024, 4096):
        qs = doc["adhoc"][f"primes_{n}"]["q"]
        table = RN.TwiddleTable(n, qs)
        for q in qs:
            rng = np.random.default_rng(synth.seed_for("ntt", n, q))
            x = rng.integers(0, q, (3, n), dtype=np.uint64)
            out[f"x_{n}_{q}"] = x.astype(np.uint32)
            out[f"fwd_{n}_{q}"] = RN.transform_rows(x, q, table, "butterfly").astype(np.uint32)
            out[f"inv_{n}_{q}"] = RN.transform_rows(x, q, table, "butterfly",
                                                   inverse=True).astype(np.uint32)
            if n <= 256:
                psi = table.entry(q).psi
                out[f"direct_{n}_{q}"] = RN.ntt_oracle(x[0], q, psi).astype(np.uint32)
    np.savez_compressed(os.path.join(HERE, "ntt_small.npz"), **out)


def make_ntt_large(doc):
    rec = {}
    for n in (1 << 13, 1 << 14, 1 << 15, 1 << 16):
        qs = doc["adhoc"][f"primes_{n}"]["q"]
        table = RN.TwiddleTable(n, qs)
        for q in qs[:3]:
            x = synth.ntt_rows(n, q, rows=2)
            f = RN.transform_rows(x, q, table, "butterfly").astype(np.uint32)
            i = RN.transform_rows(x, q, table, "butterfly", inverse=True).astype(np.uint32)
            rec[f"{n}_{q}"] = {"fwd": sha(f), "inv": sha(i),
                               "fwd_head": f[0, :8].tolist(), "inv_head": i[0, :8].tolist()}
    with open(os.path.join(HERE, "ntt_large.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


def add_ntt_large_all():
    """Record every prime of primes_{n} (incl. the 31-bit qs[4]) at 2^13..2^16,
    keeping the existing records (test_acceptance.py:97-121 sweeps them all)."""
    with open(os.path.join(HERE, "params.json")) as fh:
        doc = json.load(fh)
    path = os.path.join(HERE, "ntt_large.json")
    with open(path) as fh:
        rec = json.load(fh)
    for n in (1 << 13, 1 << 14, 1 << 15, 1 << 16):
        qs = doc["adhoc"][f"primes_{n}"]["q"]
        table = RN.TwiddleTable(n, qs)
        for q in qs:
            if f"{n}_{q}" in rec:
                continue
            x = synth.ntt_rows(n, q, rows=2)
            f = RN.transform_rows(x, q, table, "butterfly").astype(np.uint32)
            i = RN.transform_rows(x, q, table, "butterfly", inverse=True).astype(np.uint32)
            rec[f"{n}_{q}"] = {"fwd": sha(f), "inv": sha(i),
                               "fwd_head": f[0, :8].tolist(), "inv_head": i[0, :8].tolist()}
    with open(path, "w") as fh:
        json.dump(rec, fh, indent=1)


def make_kernels(doc):
    n = 64
    basis = tuple(doc["adhoc"]["primes_64"]["q"][:3])
    rng = np.random.default_rng(4242)
    out = {"basis": np.array(basis, dtype=np.uint32)}

    def poly(domain):
        rows = np.stack([rng.integers(0, q, n).astype(np.uint32) for q in basis])
        return RnsPolynomial(rows=rows, basis=basis, domain=domain)

    a, b = poly(NTT), poly(NTT)
    out["a"], out["b"] = a.rows, b.rows
    out["add"] = K.ele_add(a, b).rows
    out["sub"] = K.ele_sub(a, b).rows
    out["mul"] = K.hada_mult(a, b).rows
    out["scal"] = K.scalar_rows_mult(a, [3, 5, 1 << 29]).rows
    out["neg"] = K.negate(a).rows
    for t in (5, 25, 2 * n - 1, K.galois_element(3, n)):
        out[f"aut_ntt_{t}"] = K.apply_automorphism(a, t).rows
        c = RnsPolynomial(rows=a.rows, basis=basis, domain=COEFF)
        out[f"aut_coeff_{t}"] = K.apply_automorphism(c, t).rows
    # fast_basis_conv: several (src, tgt) shapes incl. shared primes
    allq = tuple(doc["adhoc"]["primes_64"]["q"])
    for k, (src, tgt) in enumerate([(allq[:1], allq[1:]), (allq[:2], allq[2:]),
                                    (allq[:3], allq[3:]), (allq[1:4], allq[:2] + allq[4:])]):
        rows = np.stack([rng.integers(0, q, n).astype(np.uint32) for q in src])
        out[f"bconv_in_{k}"] = rows
        out[f"bconv_src_{k}"] = np.array(src, dtype=np.uint32)
        out[f"bconv_tgt_{k}"] = np.array(tgt, dtype=np.uint32)
        out[f"bconv_out_{k}"] = fast_basis_conv(
            RnsPolynomial(rows=rows, basis=src, domain=COEFF), tgt).rows
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def ref_ops(params, seed, level, with_rot=(1,)):
    """Run the reference scheme ops on synth inputs; return dict of outputs."""
    ctx = CkksContext(params, backend="butterfly", seed=0)
    ins = synth.ckks_inputs(params.chain.q, params.chain.p, params.n, params.dnum,
                            level, seed)
    basis = tuple(params.chain.q[:level + 1])
    ext_full = tuple(params.chain.q) + tuple(params.chain.p)

    def poly(rows, b=basis):
        return RnsPolynomial(rows=rows, basis=b, domain=NTT)

    def swk(arr):
        return SwitchingKey(pairs=tuple((poly(arr[j][0], ext_full), poly(arr[j][1], ext_full))
                                        for j in range(params.dnum)))

    c0 = Ciphertext(b=poly(ins["b0"]), a=poly(ins["a0"]), scale=1, level=level)
    c1 = Ciphertext(b=poly(ins["b1"]), a=poly(ins["a1"]), scale=1, level=level)
    rlk, rk = swk(ins["rlk"]), swk(ins["rotk"])
    res = {}
    m = ctx.hmult(c0, c1, rlk)
    res["hmult"] = np.stack([m.b.rows, m.a.rows])
    ksb, ksa = ctx.key_switch(poly(ins["a0"]), rlk)
    res["keyswitch"] = np.stack([ksb.rows, ksa.rows])
    if level >= 1:
        r = ctx.rescale(m)
        res["hmult_rescale"] = np.stack([r.b.rows, r.a.rows])
        r0 = ctx.rescale(c0)
        res["rescale"] = np.stack([r0.b.rows, r0.a.rows])
    for rot in with_rot:
        h = ctx.hrotate(c0, rot, rk)
        res[f"hrotate_{rot}"] = np.stack([h.b.rows, h.a.rows])
    hc = ctx.hconjugate(c0, rk)
    res["hconjugate"] = np.stack([hc.b.rows, hc.a.rows])
    s = ctx.hadd(c0, c1)
    res["hadd"] = np.stack([s.b.rows, s.a.rows])
    s = ctx.hsub(c0, c1)
    res["hsub"] = np.stack([s.b.rows, s.a.rows])
    return res


SMALL_CASES = [
    # (case name, params factory, level, seed)
    ("small_full", lambda: RP.CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30), 5, 11),
    ("small_l4", lambda: RP.CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30), 4, 12),
    ("small_l2", lambda: RP.CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30), 2, 13),
    ("default_full", lambda: RP.CkksParams.from_preset("default"), 5, 14),
    ("set_a_full", lambda: RP.CkksParams.from_preset("set_a"), 1, 15),
    ("set_b_full", lambda: RP.CkksParams.from_preset("set_b"), 2, 16),
]

LARGE_CASES = [
    # N=2^16 shapes; outputs recorded as sha256 (inputs regenerate from seed)
    ("n16_l3", lambda: RP.CkksParams.generate(n=1 << 16, l_max=3, k=1, dnum=4, bit_size=28), 3, 21),
    ("resnet20_l3", lambda: RP.CkksParams.from_preset("resnet20"), 3, 22),
    ("set_c_full", lambda: RP.CkksParams.from_preset("set_c"), 7, 23),
    # ragged GKS slices on the tensor-core (n >= 2^14) path: alpha = 2, the
    # last slice holds one limb (level 4) / groups mix 2- and 1-limb slices
    ("set_c_l4", lambda: RP.CkksParams.from_preset("set_c"), 4, 24),
    ("set_c_l2", lambda: RP.CkksParams.from_preset("set_c"), 2, 25),
    # dnum-reduced N=2^16 set (alpha = K = 9): 9-term tensor-core base
    # conversions in ModUp and ModDown; level 12 = one full + one ragged slice
    ("p_dnum5_l12", p_dnum5, 12, 26),
    # the bench's own configuration: P-Default at the top level (45 one-limb
    # GKS slices, so the device key switch runs several slice groups)
    ("p_default_l44", p_default, 44, 27),
    # 31-bit primes through the large-n (n1 >= 128) tensor-core path: the
    # tightest lazy [0, 2q) intermediates (params.py:17-19)
    ("n16_31b_l3", lambda: RP.CkksParams.generate(n=1 << 16, l_max=3, k=1, dnum=4, bit_size=31),
     3, 28),
    ("n14_31b_l5", lambda: RP.CkksParams.generate(n=1 << 14, l_max=5, k=2, dnum=3, bit_size=31),
     5, 29),
]


def make_ckks():
    out = {}
    for name, fac, level, seed in SMALL_CASES:
        t = time.time()
        res = ref_ops(fac(), seed, level)
        for k, v in res.items():
            out[f"{name}/{k}"] = v.astype(np.uint32)
        print(name, f"{time.time() - t:.1f}s")
    np.savez_compressed(os.path.join(HERE, "ckks_small.npz"), **out)
    rec = {}
    for name, fac, level, seed in LARGE_CASES:
        t = time.time()
        res = ref_ops(fac(), seed, level)
        rec[name] = {k: {"sha256": sha(v), "head": v.reshape(-1)[:8].tolist()}
                     for k, v in res.items()}
        print(name, f"{time.time() - t:.1f}s")
    with open(os.path.join(HERE, "ckks_large.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


def make_tfhe1():
    """Reference-written TFHE1 blobs of synthetic objects (small params)."""
    from fractions import Fraction
    from rnsckks import serialize as RS
    from rnsckks.ckks import Plaintext, PublicKey, SecretKey
    params = RP.CkksParams.generate(n=64, l_max=3, k=2, dnum=2, bit_size=28)
    digest = params.digest()
    rng = np.random.default_rng(9090)
    basis = tuple(params.chain.q[:3])
    ext = tuple(params.chain.q) + tuple(params.chain.p)

    def poly(b, dom=NTT):
        return RnsPolynomial(rows=synth.rows(rng, b, (params.n,)), basis=b, domain=dom)

    ct = Ciphertext(b=poly(basis), a=poly(basis), scale=Fraction(2 ** 40, 3), level=2)
    swk = SwitchingKey(pairs=tuple((poly(ext), poly(ext)) for _ in range(params.dnum)))
    out = {"digest": np.frombuffer(digest, np.uint8),
           "poly": np.frombuffer(RS.dump_polynomial(poly(basis, COEFF), digest), np.uint8),
           "ct": np.frombuffer(RS.dump_ciphertext(ct, digest), np.uint8),
           "pt": np.frombuffer(RS.dump_plaintext(Plaintext(poly=poly(basis), scale=Fraction(7),
                                                           level=2), digest), np.uint8),
           "pk": np.frombuffer(RS.dump_public_key(PublicKey(b=poly(ext), a=poly(ext)), digest),
                               np.uint8),
           "sk": np.frombuffer(RS.dump_secret_key(SecretKey(s=poly(ext)), digest), np.uint8),
           "swk": np.frombuffer(RS.dump_switching_key(swk, digest), np.uint8)}
    np.savez_compressed(os.path.join(HERE, "tfhe1.npz"), **out)


CLIENT_CASES = [
    ("small", lambda: RP.CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30)),
    ("default", lambda: RP.CkksParams.from_preset("default")),
    ("set_a", lambda: RP.CkksParams.from_preset("set_a")),
]


def make_client():
    """Reference keygen / encode / encrypt / decrypt on fixed seeds: sha256 of
    every key and ciphertext row set, and the decoded slots (client.json)."""
    rec = {}
    for name, fac in CLIENT_CASES:
        params = fac()
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
        r = {"sk": sha(sk.s.rows), "pk_b": sha(pk.b.rows), "pk_a": sha(pk.a.rows),
             "pt": sha(pt.poly.rows), "ct_b": sha(ct.b.rows), "ct_a": sha(ct.a.rows),
             "scale": [pt.scale.numerator, pt.scale.denominator],
             "dec_re": [float(v) for v in dec.real[:16]], "dec_im": [float(v) for v in dec.imag[:16]]}
        for kname, key in (("rlk", rlk), ("rk", rk), ("ck", ck)):
            r[kname] = [[sha(b.rows), sha(a.rows)] for b, a in key.pairs]
        # one evaluated product through the reference, for an end-to-end check
        m = ctx.rescale(ctx.hmult(ct, ct, rlk))
        r["hmult_rescale_b"], r["hmult_rescale_a"] = sha(m.b.rows), sha(m.a.rows)
        dm = ctx.decrypt_decode(sk, m)
        r["dec_sq_re"] = [float(v) for v in dm.real[:16]]
        rec[name] = r
        print("client", name)
    with open(os.path.join(HERE, "client.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


def add_large(names):
    """Append selected LARGE_CASES to ckks_large.json (keeps existing records)."""
    path = os.path.join(HERE, "ckks_large.json")
    with open(path) as fh:
        rec = json.load(fh)
    for name, fac, level, seed in LARGE_CASES:
        if name not in names:
            continue
        t = time.time()
        res = ref_ops(fac(), seed, level)
        rec[name] = {k: {"sha256": sha(v), "head": v.reshape(-1)[:8].tolist()}
                     for k, v in res.items()}
        print(name, f"{time.time() - t:.1f}s")
    with open(path, "w") as fh:
        json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "add-preset-p_dnum5":
        path = os.path.join(HERE, "params.json")
        with open(path) as fh:
            doc = json.load(fh)
        doc["presets"]["p_dnum5"] = chain_doc(p_dnum5())
        with open(path, "w") as fh:
            json.dump(doc, fh, indent=1)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "ntt-large-all":
        add_ntt_large_all()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "client":
        make_client()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "tfhe1":
        make_tfhe1()
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "add-large":
        add_large(sys.argv[2:])
        sys.exit(0)
    d = make_params()
    make_ntt_small(d)
    make_ntt_large(d)
    make_kernels(d)
    make_ckks()
    make_tfhe1()
    make_client()
    print("golden fixtures written to", HERE)
