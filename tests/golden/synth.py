"""Deterministic synthetic inputs shared by make_golden.py and the tests.

Pure numpy (no reference import), so the GPU box can regenerate exactly the
inputs the golden outputs were computed from.  Residues are uniform per limb,
drawn as `rng.integers(0, q, shape, dtype=uint64)` like the reference's
`cli._random_batch` (cli.py:59-64).  Switching keys are synthetic uniform
NTT-domain pairs over the full extended basis chain.q ++ chain.p
(ckks.py:57-60); bit-exactness does not need valid keys.
"""

import zlib

import numpy as np


def seed_for(*parts):
    return zlib.crc32(repr(parts).encode()) & 0x7FFFFFFF


def rows(rng, basis, tail):
    out = np.empty((len(basis),) + tuple(tail), dtype=np.uint32)
    for i, q in enumerate(basis):
        out[i] = rng.integers(0, q, tail, dtype=np.uint64)
    return out


def ntt_rows(n, q, rows=2):
    rng = np.random.default_rng(seed_for("ntt_large", n, q))
    return rng.integers(0, q, (rows, n), dtype=np.uint64).astype(np.uint32)


def switching_key(rng, chain_q, chain_p, n, dnum):
    ext = tuple(chain_q) + tuple(chain_p)
    key = np.empty((dnum, 2, len(ext), n), dtype=np.uint32)
    for j in range(dnum):
        for c in range(2):
            key[j, c] = rows(rng, ext, (n,))
    return key


def ckks_inputs(chain_q, chain_p, n, dnum, level, seed):
    """Two ciphertexts at `level` plus a relin key and a rotation key."""
    rng = np.random.default_rng(seed)
    basis = tuple(chain_q[:level + 1])
    d = {}
    for name in ("b0", "a0", "b1", "a1"):
        d[name] = rows(rng, basis, (n,))
    d["rlk"] = switching_key(rng, chain_q, chain_p, n, dnum)
    d["rotk"] = switching_key(rng, chain_q, chain_p, n, dnum)
    return d
