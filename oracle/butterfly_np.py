"""CPU ORACLE -- test / baseline infrastructure only (see oracle/oracle.py).

A numpy restatement of the reference's fastest CPU backend, the radix-2
butterfly transform (ref `ntt.py:172-205`, dispatched by `transform_rows`
`ntt.py:347-363` and `batched_apply` `batch.py:78-97`): uint64 ufuncs over a
(B, n) block of one prime, every product `(u * w) % q`, exactly the cost
profile of the reference's numpy code.  `bench.py` times it on one host core
and over a `multiprocessing.Pool` of every core beside the
C/OpenMP port; tests check it bit for bit against the C oracle.

* forward: Cooley-Tukey decimation in time with the bit-reversed powers of
  psi, natural-order output by a final bit-reversal gather (`ntt.py:172-186`);
* inverse: bit-reversal gather, Gentleman-Sande decimation in frequency with
  the bit-reversed powers of psi^-1, then n^-1 (`ntt.py:189-205`).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from .oracle import negacyclic_root


def _bit_reverse(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    out = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


@lru_cache(maxsize=None)
def _plan(q: int, n: int):
    """(bit-reversal permutation, psi^rev(i), psi^-rev(i), n^-1) for (q, n)
    (the reference's TwiddleTable.butterfly entry, ntt.py:158-165)."""
    rev = _bit_reverse(n)
    psi = negacyclic_root(q, n)

    def powers(root):
        p = np.empty(n, dtype=np.uint64)
        acc = 1
        for i in range(n):
            p[i] = acc
            acc = acc * root % q
        return p[rev]
    return rev, powers(psi), powers(pow(psi, q - 2, q)), pow(n, q - 2, q)


def forward(x, q: int) -> np.ndarray:
    """(B, n) residues mod q -> NTT (uint64), natural order."""
    a = np.asarray(x, dtype=np.uint64) % np.uint64(q)
    bsz, n = a.shape
    rev, wf, _, _ = _plan(q, n)
    qq = np.uint64(q)
    groups, span = 1, n
    while groups < n:
        span //= 2
        blk = a.reshape(bsz, groups, 2, span)
        w = wf[groups:2 * groups].reshape(1, groups, 1)
        top = blk[:, :, 0, :]
        bot = blk[:, :, 1, :] * w % qq
        a = np.stack(((top + bot) % qq, (top + qq - bot) % qq), axis=2).reshape(bsz, n)
        groups *= 2
    return a[:, rev]


def inverse(x, q: int) -> np.ndarray:
    """(B, n) NTT-domain residues mod q -> coefficients (uint64)."""
    a = np.asarray(x, dtype=np.uint64) % np.uint64(q)
    bsz, n = a.shape
    rev, _, wi, n_inv = _plan(q, n)
    qq = np.uint64(q)
    a = a[:, rev]
    groups, span = n // 2, 1
    while groups >= 1:
        blk = a.reshape(bsz, groups, 2, span)
        w = wi[groups:2 * groups].reshape(1, groups, 1)
        top, bot = blk[:, :, 0, :], blk[:, :, 1, :]
        a = np.stack(((top + bot) % qq, (top + qq - bot) * w % qq), axis=2).reshape(bsz, n)
        groups //= 2
        span *= 2
    return a * np.uint64(n_inv) % qq


def fwd_inv_rows(task):
    """Pool worker: fwd + inv of `members` seeded rows mod q; returns the
    number of limb-NTTs done (2 * members)."""
    q, n, members, seed = task
    x = np.random.default_rng(seed).integers(0, q, (members, n), dtype=np.uint64)
    inverse(forward(x, q), q)
    return 2 * members
