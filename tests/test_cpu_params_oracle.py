"""CPU tests: host parameter layer and the CPU oracle, pinned to the golden
vectors that tests/golden/make_golden.py produced by running the reference."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
import synth
from oracle import oracle as O
from paper_2212_14191_b200 import params as P


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


# --------------------------------------------------------------------- params

@pytest.mark.parametrize("name", sorted(P.PRESETS))
def test_presets_match_reference(name, golden_params):
    doc = golden_params["presets"][name]
    p = P.CkksParams.from_preset(name)
    assert list(p.chain.q) == doc["q"] and list(p.chain.p) == doc["p"]
    assert (p.l_max, p.k, p.dnum) == (doc["l_max"], doc["k"], doc["dnum"])
    assert [p.plan.n1, p.plan.n2] == doc["plan"]
    for r in p.chain.q + p.chain.p:
        assert p.chain.roots[r].psi == doc["psi"][str(r)]


def test_p_default_is_paper_shape(golden_params):
    p = P.CkksParams.from_preset("p_default")
    assert (p.n, p.l_max, p.k, p.dnum, p.alpha) == (1 << 16, 44, 1, 45, 1)
    assert sum(r.bit_length() for r in p.chain.q + p.chain.p) == P.PRESET_LOG_PQ["p_default"]


def test_small_params_and_adhoc_primes(golden_params):
    sp = golden_params["adhoc"]["small_params"]
    p = P.CkksParams.generate(n=256, l_max=5, k=3, dnum=3, bit_size=30)
    assert list(p.chain.q) == sp["q"] and list(p.chain.p) == sp["p"]
    for n in (16, 64, 256, 1024, 4096, 1 << 13, 1 << 14, 1 << 15, 1 << 16):
        d = golden_params["adhoc"][f"primes_{n}"]
        assert P.generate_primes(n, [30, 24, 26, 28, 31]) == d["q"]
        assert [P.find_negacyclic_root(q, n) for q in d["q"]] == d["psi"]
        assert [P.build_ntt_plan(n).n1, P.build_ntt_plan(n).n2] == d["plan"]


def test_known_answers(golden_params):
    ka = golden_params["known_answers"]
    assert P.find_negacyclic_root(17, 4) == ka["find_negacyclic_root_17_4"] == 9
    assert [int(v) for v in P.split_bytes(np.array([0x12345678]))[:, 0]] == \
        ka["split_0x12345678"] == [0x78, 0x56, 0x34, 0x12]
    assert np.array_equal(P.fuse_bytes(P.split_bytes(np.arange(1000) * 4294967)),
                          (np.arange(1000) * 4294967).astype(np.uint32))


def test_is_prime_matches_sympy():
    sympy = pytest.importorskip("sympy")
    rng = np.random.default_rng(0)
    for v in list(rng.integers(2, 1 << 32, 3000)) + list(range(2, 2000)):
        assert P.is_prime(int(v)) == bool(sympy.isprime(int(v)))


def test_twiddle_closed_forms():
    n = 256
    q = P.generate_primes(n, [30])[0]
    psi = P.find_negacyclic_root(q, n)
    plan = P.build_ntt_plan(n)
    tw = P.build_twiddles(plan, q, psi, "fwd")
    for i in range(plan.n1):
        for j in range(plan.n2):
            assert tw.w2[i, j] == pow(psi, 2 * i * j + j, q)
    inv = P.build_twiddles(plan, q, psi, "inv")
    ipsi = pow(psi, q - 2, q)
    assert inv.w3[3, 5] == pow(ipsi, plan.n1 * (2 * 3 * 5 + 5), q)


def test_parameter_errors():
    with pytest.raises(P.ParameterError if hasattr(P, "ParameterError") else ValueError):
        P.generate_primes(100, [30])
    from paper_2212_14191_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        P.CkksParams.from_preset("nope")
    with pytest.raises(ParameterError):
        P.CkksParams.generate(n=256, l_max=5, k=3, dnum=4)
    with pytest.raises(ParameterError):  # GKS: P must exceed each slice product
        P.CkksParams.generate(n=256, l_max=5, k=1, dnum=2)


# --------------------------------------------------------------------- oracle

def test_oracle_frozen_vector():
    # test_ntt.py:45-54: n=4, q=17, psi=2, a=[1,2,3,4] -> [15,13,11,16]
    want = [15, 13, 11, 16]
    got = [sum(a * pow(2, 2 * m * k + m, 17) for m, a in enumerate([1, 2, 3, 4])) % 17
           for k in range(4)]
    assert got == want
    # the C oracle's direct O(n^2) path uses psi = smallest-root psi; check
    # it against the same closed form on a real table
    q = P.generate_primes(16, [24])[0]
    psi = O.negacyclic_root(q, 16)
    a = np.arange(16, dtype=np.uint32) * 7 % q
    direct = [sum(int(a[m]) * pow(psi, 2 * m * k + m, q) for m in range(16)) % q
              for k in range(16)]
    assert O.ntt_direct(a, q).tolist() == direct


@pytest.fixture(scope="module")
def ntt_small():
    return np.load(os.path.join(GOLDEN, "ntt_small.npz"))


@pytest.mark.parametrize("n", [16, 64, 256, 1024, 4096])
def test_oracle_ntt_golden(n, ntt_small, golden_params):
    for q in golden_params["adhoc"][f"primes_{n}"]["q"]:
        x = ntt_small[f"x_{n}_{q}"]
        if q >= 1 << 31:
            continue
        assert np.array_equal(O.transform_rows(x, q), ntt_small[f"fwd_{n}_{q}"])
        assert np.array_equal(O.transform_rows(x, q, inverse=True), ntt_small[f"inv_{n}_{q}"])
        if n <= 256:
            assert np.array_equal(O.ntt_direct(x[0], q), ntt_small[f"direct_{n}_{q}"])


@pytest.mark.parametrize("n", [1 << 13, 1 << 14])
def test_oracle_ntt_golden_large(n, golden_params):
    with open(os.path.join(GOLDEN, "ntt_large.json")) as fh:
        rec = json.load(fh)
    for q in golden_params["adhoc"][f"primes_{n}"]["q"]:   # incl. the 31-bit qs[4]
        x = synth.ntt_rows(n, q, rows=2)
        assert _sha(O.transform_rows(x, q)) == rec[f"{n}_{q}"]["fwd"]
        assert _sha(O.transform_rows(x, q, inverse=True)) == rec[f"{n}_{q}"]["inv"]


def test_oracle_kernels_golden():
    k = np.load(os.path.join(GOLDEN, "kernels.npz"))
    basis = tuple(int(v) for v in k["basis"])
    a, b = k["a"], k["b"]
    assert np.array_equal(O.ele_add(a, b, basis), k["add"])
    assert np.array_equal(O.ele_sub(a, b, basis), k["sub"])
    assert np.array_equal(O.hada_mult(a, b, basis), k["mul"])
    assert np.array_equal(O.scalar_rows_mult(a, [3, 5, 1 << 29], basis), k["scal"])
    assert np.array_equal(O.negate(a, basis), k["neg"])
    n = a.shape[-1]
    for t in (5, 25, 2 * n - 1, O.galois_element(3, n)):
        assert np.array_equal(O.apply_automorphism(a, t, basis, "ntt"), k[f"aut_ntt_{t}"])
        assert np.array_equal(O.apply_automorphism(a, t, basis, "coeff"), k[f"aut_coeff_{t}"])
    for i in range(4):
        src = tuple(int(v) for v in k[f"bconv_src_{i}"])
        tgt = tuple(int(v) for v in k[f"bconv_tgt_{i}"])
        assert np.array_equal(O.fast_basis_conv(k[f"bconv_in_{i}"], src, tgt), k[f"bconv_out_{i}"])


def _oracle_ops(params, level, seed):
    p = params
    ins = synth.ckks_inputs(p.chain.q, p.chain.p, p.n, p.dnum, level, seed)
    basis = tuple(p.chain.q[:level + 1])
    cq, cp = tuple(p.chain.q), tuple(p.chain.p)
    out = {}
    hb, ha = O.hmult(ins["b0"], ins["a0"], ins["b1"], ins["a1"], basis, ins["rlk"], cq, cp,
                     p.alpha, p.dnum)
    out["hmult"] = np.stack([hb, ha])
    out["keyswitch"] = np.stack(O.key_switch(ins["a0"], basis, ins["rlk"], cq, cp, p.alpha, p.dnum))
    if level >= 1:
        out["hmult_rescale"] = np.stack(O.rescale(hb, ha, basis))
        out["rescale"] = np.stack(O.rescale(ins["b0"], ins["a0"], basis))
    out["hrotate_1"] = np.stack(O.hrotate(ins["b0"], ins["a0"], 1, basis, ins["rotk"], cq, cp,
                                          p.alpha, p.dnum))
    out["hconjugate"] = np.stack(O.hconjugate(ins["b0"], ins["a0"], basis, ins["rotk"], cq, cp,
                                              p.alpha, p.dnum))
    out["hadd"] = np.stack([O.ele_add(ins["b0"], ins["b1"], basis),
                            O.ele_add(ins["a0"], ins["a1"], basis)])
    out["hsub"] = np.stack([O.ele_sub(ins["b0"], ins["b1"], basis),
                            O.ele_sub(ins["a0"], ins["a1"], basis)])
    return out


@pytest.mark.parametrize("case,level,seed,factory", [
    ("small_full", 5, 11, lambda: P.CkksParams.generate(n=256, l_max=5, k=3, dnum=3)),
    ("small_l4", 4, 12, lambda: P.CkksParams.generate(n=256, l_max=5, k=3, dnum=3)),
    ("small_l2", 2, 13, lambda: P.CkksParams.generate(n=256, l_max=5, k=3, dnum=3)),
    ("default_full", 5, 14, lambda: P.CkksParams.from_preset("default")),
    ("set_a_full", 1, 15, lambda: P.CkksParams.from_preset("set_a")),
    ("set_b_full", 2, 16, lambda: P.CkksParams.from_preset("set_b")),
])
def test_oracle_ckks_golden(case, level, seed, factory):
    g = np.load(os.path.join(GOLDEN, "ckks_small.npz"))
    for op, arr in _oracle_ops(factory(), level, seed).items():
        assert np.array_equal(arr, g[f"{case}/{op}"]), (case, op)


def test_oracle_ckks_golden_n16():
    with open(os.path.join(GOLDEN, "ckks_large.json")) as fh:
        rec = json.load(fh)["n16_l3"]
    p = P.CkksParams.generate(n=1 << 16, l_max=3, k=1, dnum=4, bit_size=28)
    for op, arr in _oracle_ops(p, 3, 21).items():
        assert _sha(arr) == rec[op]["sha256"], op


def test_oracle_ckks_golden_31bit():
    """A 31-bit chain (the tightest lazy bounds) at n = 2^14: the oracle
    reproduces the reference's outputs recorded in ckks_large.json."""
    with open(os.path.join(GOLDEN, "ckks_large.json")) as fh:
        rec = json.load(fh)["n14_31b_l5"]
    p = P.CkksParams.generate(n=1 << 14, l_max=5, k=2, dnum=3, bit_size=31)
    for op, arr in _oracle_ops(p, 5, 29).items():
        assert _sha(arr) == rec[op]["sha256"], op


def test_oracle_batched_equals_per_member():
    # batched (L, B, n) oracle calls equal the per-member calls (batch.py:78)
    p = P.CkksParams.from_preset("set_a")
    rng = np.random.default_rng(3)
    basis = tuple(p.chain.q)
    ext = basis + tuple(p.chain.p)
    key = np.stack([np.stack([O.uniform_rows(rng, ext, (p.n,)) for _ in range(2)])
                    for _ in range(p.dnum)])
    c = np.stack([O.uniform_rows(rng, basis, (3, p.n)) for _ in range(4)])
    hb, ha = O.hmult(c[0], c[1], c[2], c[3], basis, key, basis, tuple(p.chain.p), p.alpha, p.dnum)
    for m in range(3):
        b1, a1 = O.hmult(c[0][:, m], c[1][:, m], c[2][:, m], c[3][:, m], basis, key, basis,
                         tuple(p.chain.p), p.alpha, p.dnum)
        assert np.array_equal(hb[:, m], b1) and np.array_equal(ha[:, m], a1)


@pytest.mark.parametrize("n", [16, 256, 4096])
def test_numpy_butterfly_restatement_matches_goldens(n, golden_params):
    """oracle/butterfly_np.py (the numpy restatement bench.py times as the
    Python reference's cost profile) reproduces the reference's butterfly
    outputs recorded in ntt_small.npz."""
    from oracle import butterfly_np as BF
    small = np.load(os.path.join(GOLDEN, "ntt_small.npz"))
    for q in golden_params["adhoc"][f"primes_{n}"]["q"]:
        x = small[f"x_{n}_{q}"]
        assert np.array_equal(BF.forward(x, q).astype(np.uint32), small[f"fwd_{n}_{q}"])
        assert np.array_equal(BF.inverse(x, q).astype(np.uint32), small[f"inv_{n}_{q}"])
