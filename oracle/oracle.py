"""CPU ORACLE -- test infrastructure only.

Imported ONLY by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline
leg and `--impl reference`).  The product package never imports it; the
product's own path is the sm_100a extension and fails loudly without it.

A numpy restatement of the reference's hot-path semantics
(/root/reference/pkg/src/rnsckks), with the transforms delegated to the
plain-C restatement in tfhe_oracle.c.  Arrays are level-major: axis 0 is the
RNS limb (one prime per row), the last axis is the coefficient/slot index and
any axes in between are batch axes, so the same function serves an
RnsPolynomial's (L+1, N) rows and a BatchBuffer's (L+1, B, N) data
(batch.py:22-47).  Every function cites the reference lines it restates.

Parity is PINNED: tests/test_oracle_golden.py checks this module against the
golden vectors in tests/golden/, which tests/golden/make_golden.py produced by
importing the reference itself, plus the reference's own known-answer tests
(test_ntt.py:45-54).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile tfhe_oracle.c with gcc (-O3 -fopenmp) into oracle/_build/."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.orc_ntt_tables.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, u32p]
        L.orc_ntt_rows.argtypes = [u32p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32,
                                   u32p, ctypes.c_int, ctypes.c_int]
        L.orc_ntt_direct.argtypes = [u32p, u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_mulmod_rows.argtypes = [u32p, u32p, u32p, ctypes.c_int64, ctypes.c_int64,
                                      u32p, ctypes.c_int]
        L.orc_mulmod_rows.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


#: host threads the transform loop may use (None = all)
THREADS = 0


# ---------------------------------------------------------------------------
# roots (params.py:40-62)
# ---------------------------------------------------------------------------

def _factors(m):
    out, f = [], 2
    while f * f <= m:
        if m % f == 0:
            out.append(f)
            while m % f == 0:
                m //= f
        f += 1
    if m > 1:
        out.append(m)
    return out


@lru_cache(maxsize=None)
def negacyclic_root(q: int, n: int) -> int:
    """psi = g^((q-1)/2n), g the smallest primitive root (params.py:40-62)."""
    fs = _factors(q - 1)
    g = 2
    while not all(pow(g, (q - 1) // f, q) != 1 for f in fs):
        g += 1
    return pow(g, (q - 1) // (2 * n), q)


@lru_cache(maxsize=None)
def _tables(q: int, n: int) -> np.ndarray:
    t = np.empty(4 * n + 2, dtype=np.uint32)
    rc = lib().orc_ntt_tables(q, negacyclic_root(q, n), n.bit_length() - 1, _p(t))
    if rc:
        raise ValueError(f"oracle cannot build tables for q={q}")
    return t


# ---------------------------------------------------------------------------
# transforms (ntt.py:172-205, 347-385; batch.py:95-97)
# ---------------------------------------------------------------------------

def transform_rows(x, q: int, inverse: bool = False, threads: int | None = None) -> np.ndarray:
    """(..., n) residues mod q -> transformed copy (ntt.transform_rows)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint64) % np.uint64(q), dtype=np.uint32).copy()
    n = a.shape[-1]
    rows = a.size // n
    lib().orc_ntt_rows(_p(a), rows, n.bit_length() - 1, q, _p(_tables(q, n)),
                       int(inverse), THREADS if threads is None else threads)
    return a


def ntt_direct(a, q: int) -> np.ndarray:
    """O(n^2) ntt_oracle (ntt.py:44-59)."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    n = a.shape[-1]
    out = np.empty(n, dtype=np.uint32)
    lib().orc_ntt_direct(_p(a), _p(out), n.bit_length() - 1, q, negacyclic_root(q, n))
    return out


def ntt(rows, basis, threads=None) -> np.ndarray:
    """Per-limb forward transform of (L, ..., n) (ntt_forward ntt.py:366-374,
    batched_apply 'ntt' batch.py:95-97)."""
    rows = np.asarray(rows, dtype=np.uint32)
    return np.stack([transform_rows(rows[i], q, False, threads) for i, q in enumerate(basis)]) \
        if len(basis) else rows.copy()


def transform_inplace(rows, basis, inverse: bool = False, threads=None) -> np.ndarray:
    """In-place per-limb transform of a C-contiguous uint32 (L, ..., n) array
    whose rows are already reduced mod their prime: the C kernel only, no
    upcast / copy / stack glue (the CPU-baseline timing path)."""
    if rows.dtype != np.uint32 or not rows.flags.c_contiguous:
        raise ValueError("transform_inplace needs a C-contiguous uint32 array")
    n = rows.shape[-1]
    per = rows[0].size // n if len(basis) else 0
    for i, q in enumerate(basis):
        lib().orc_ntt_rows(_p(rows[i]), per, n.bit_length() - 1, q, _p(_tables(q, n)),
                           int(inverse), THREADS if threads is None else threads)
    return rows


def intt(rows, basis, threads=None) -> np.ndarray:
    rows = np.asarray(rows, dtype=np.uint32)
    return np.stack([transform_rows(rows[i], q, True, threads) for i, q in enumerate(basis)]) \
        if len(basis) else rows.copy()


# ---------------------------------------------------------------------------
# element-wise kernels (kernels.py:24-67, batch.py:116-127)
# ---------------------------------------------------------------------------

def _q(basis, ndim):
    return np.array(basis, dtype=np.uint64).reshape((-1,) + (1,) * (ndim - 1))


def ele_add(a, b, basis):
    q = _q(basis, np.ndim(a))
    return ((np.asarray(a, np.uint64) + np.asarray(b, np.uint64)) % q).astype(np.uint32)


def ele_sub(a, b, basis):
    q = _q(basis, np.ndim(a))
    return ((np.asarray(a, np.uint64) + q - np.asarray(b, np.uint64)) % q).astype(np.uint32)


def hada_mult(a, b, basis):
    q = _q(basis, np.ndim(a))
    return (np.asarray(a, np.uint64) * np.asarray(b, np.uint64) % q).astype(np.uint32)


def scalar_rows_mult(a, scalars, basis):
    q = _q(basis, np.ndim(a))
    s = np.array([int(c) % int(p) for c, p in zip(scalars, basis)],
                 dtype=np.uint64).reshape(q.shape)
    return (np.asarray(a, np.uint64) * s % q).astype(np.uint32)


def negate(a, basis):
    q = _q(basis, np.ndim(a))
    return ((q - np.asarray(a, np.uint64)) % q).astype(np.uint32)


# ---------------------------------------------------------------------------
# automorphisms (kernels.py:70-117)
# ---------------------------------------------------------------------------

def galois_element(r: int, n: int, conj: bool = False) -> int:
    return 2 * n - 1 if conj else pow(5, r % n, 2 * n)


def ntt_permutation(t: int, n: int) -> np.ndarray:
    k = np.arange(n, dtype=np.int64)
    return ((t * (2 * k + 1)) % (2 * n) - 1) // 2


def apply_automorphism(a, t: int, basis, domain: str = "ntt"):
    a = np.asarray(a, dtype=np.uint32)
    n = a.shape[-1]
    t %= 2 * n
    if domain == "ntt":
        return np.ascontiguousarray(a[..., ntt_permutation(t, n)])
    i = np.arange(n, dtype=np.int64)
    e = (t * i) % (2 * n)
    dest, neg = e % n, e >= n
    out = np.zeros_like(a)
    vals = np.where(neg, negate(a, basis), a)
    out[..., dest] = vals
    return out


# ---------------------------------------------------------------------------
# base conversion (rns.py:118-152)
# ---------------------------------------------------------------------------

def fast_basis_conv(rows, src, tgt) -> np.ndarray:
    """b_j = sum_i [a_i * (Q/q_i)^-1]_{q_i} * ((Q/q_i) mod p_j) mod p_j;
    shared primes are copied (rns.py:118-152).  rows: (len(src), ..., n)."""
    rows = np.asarray(rows, dtype=np.uint32)
    big_q = 1
    for q in src:
        big_q *= q
    ys = [(rows[i].astype(np.uint64) * np.uint64(pow(big_q // q, -1, q))) % np.uint64(q)
          for i, q in enumerate(src)]
    out = np.empty((len(tgt),) + rows.shape[1:], dtype=np.uint32)
    for j, p in enumerate(tgt):
        if p in src:
            out[j] = rows[src.index(p)]
            continue
        acc = np.zeros(rows.shape[1:], dtype=np.uint64)
        pj = np.uint64(p)
        for i, q in enumerate(src):
            acc = (acc + ys[i] * np.uint64((big_q // q) % p) % pj) % pj
        out[j] = acc
    return out


# ---------------------------------------------------------------------------
# CKKS evaluation ops (ckks.py:246-381); a ciphertext is (b, a) level-major
# arrays over `basis` = chain primes q_0..q_level.  `chain_q`/`chain_p` are
# the full chain and specials; `alpha`, `dnum` as CkksParams.  Switching keys
# are (dnum, 2, L+1+K, n) arrays over chain_q ++ chain_p (ckks.py:57-60).
# Batch axes between limb and coefficient are carried through unchanged.
# ---------------------------------------------------------------------------

def _key_rows(key_poly, full_ext, ext):
    idx = [full_ext.index(r) for r in ext]
    return key_poly[idx]


def mod_up(part, part_basis, ext, threads=None):
    """ckks.py:354-365"""
    coeff = intt(part, part_basis, threads)
    missing = tuple(q for q in ext if q not in part_basis)
    conv = ntt(fast_basis_conv(coeff, tuple(part_basis), missing), missing, threads)
    out = np.empty((len(ext),) + part.shape[1:], dtype=np.uint32)
    for i, q in enumerate(ext):
        out[i] = part[part_basis.index(q)] if q in part_basis else conv[missing.index(q)]
    return out


def mod_down(x, x_basis, target, specials, threads=None):
    """ckks.py:367-381"""
    sp_idx = [x_basis.index(r) for r in specials]
    special_part = intt(x[sp_idx], specials, threads)
    conv = ntt(fast_basis_conv(special_part, tuple(specials), tuple(target)), target, threads)
    big_p = 1
    for r in specials:
        big_p *= r
    out = np.empty((len(target),) + x.shape[1:], dtype=np.uint32)
    for i, q in enumerate(target):
        qq = np.uint64(q)
        xi = x[x_basis.index(q)].astype(np.uint64)
        y = conv[i].astype(np.uint64)
        out[i] = (xi + qq - y) % qq * np.uint64(pow(big_p, -1, q)) % qq
    return out


def key_switch_acc(d, basis, key, chain_q, chain_p, alpha, dnum, threads=None):
    """ckks.py:321-351: the key switch's inner-product accumulators over
    ext = basis ++ specials, before ModDown."""
    basis = tuple(basis)
    level = len(basis) - 1
    ext = basis + tuple(chain_p)
    full_ext = tuple(chain_q) + tuple(chain_p)
    acc_b = np.zeros((len(ext),) + d.shape[1:], dtype=np.uint32)
    acc_a = np.zeros_like(acc_b)
    for j in range(dnum):
        lo = j * alpha
        if lo > level:
            break
        hi = min((j + 1) * alpha, level + 1)
        raised = mod_up(d[lo:hi], basis[lo:hi], ext, threads)
        kb = _key_rows(key[j][0], full_ext, ext)
        ka = _key_rows(key[j][1], full_ext, ext)
        if raised.ndim > 2:
            kb = kb.reshape(kb.shape[:1] + (1,) * (raised.ndim - 2) + kb.shape[1:])
            ka = ka.reshape(kb.shape)
        acc_b = ele_add(acc_b, hada_mult(raised, kb, ext), ext)
        acc_a = ele_add(acc_a, hada_mult(raised, ka, ext), ext)
    return acc_b, acc_a


def key_switch(d, basis, key, chain_q, chain_p, alpha, dnum, threads=None):
    """ckks.py:321-352.  d: (level+1, ..., n) NTT domain over `basis`."""
    basis = tuple(basis)
    acc_b, acc_a = key_switch_acc(d, basis, key, chain_q, chain_p, alpha, dnum, threads)
    ext = basis + tuple(chain_p)
    return (mod_down(acc_b, ext, basis, tuple(chain_p), threads),
            mod_down(acc_a, ext, basis, tuple(chain_p), threads))


def key_switch_part(d_local, y_full, basis, lo, key, chain_q, chain_p, alpha, dnum,
                    threads=None):
    """Limb-partitioned key switch restated on the CPU: the rank
    owning chain rows [lo, lo + len(d_local)) of `basis` raises every GKS
    slice of the gathered coefficient rows y_full to its own primes plus the
    specials, accumulates against the key and does ModDown to its own rows.
    Equals key_switch(...)[:, lo:lo+n] (ckks.py:321-381)."""
    basis = tuple(basis)
    level = len(basis) - 1
    n_loc = d_local.shape[0]
    own = basis[lo:lo + n_loc]
    tgt = own + tuple(chain_p)
    full_ext = tuple(chain_q) + tuple(chain_p)
    acc_b = np.zeros((len(tgt),) + d_local.shape[1:], dtype=np.uint32)
    acc_a = np.zeros_like(acc_b)
    for j in range(dnum):
        s0 = j * alpha
        if s0 > level:
            break
        s1 = min((j + 1) * alpha, level + 1)
        sl_basis = basis[s0:s1]
        raised = np.empty_like(acc_b)
        for t, q in enumerate(tgt):
            if q in sl_basis:          # slice rows reused unchanged (ckks.py:361-364)
                raised[t] = d_local[own.index(q)]
            else:
                conv = fast_basis_conv(y_full[s0:s1], sl_basis, (q,))
                raised[t] = ntt(conv, (q,), threads)[0]
        kb = _key_rows(key[j][0], full_ext, tgt)
        ka = _key_rows(key[j][1], full_ext, tgt)
        if raised.ndim > 2:
            kb = kb.reshape(kb.shape[:1] + (1,) * (raised.ndim - 2) + kb.shape[1:])
            ka = ka.reshape(kb.shape)
        acc_b = ele_add(acc_b, hada_mult(raised, kb, tgt), tgt)
        acc_a = ele_add(acc_a, hada_mult(raised, ka, tgt), tgt)
    return (mod_down(acc_b, tgt, own, tuple(chain_p), threads),
            mod_down(acc_a, tgt, own, tuple(chain_p), threads))


def hmult(b0, a0, b1, a1, basis, rlk, chain_q, chain_p, alpha, dnum, threads=None):
    """ckks.py:265-274 -> (b, a)"""
    d0 = hada_mult(b0, b1, basis)
    d1 = ele_add(hada_mult(a0, b1, basis), hada_mult(a1, b0, basis), basis)
    d2 = hada_mult(a0, a1, basis)
    ksb, ksa = key_switch(d2, basis, rlk, chain_q, chain_p, alpha, dnum, threads)
    return ele_add(d0, ksb, basis), ele_add(d1, ksa, basis)


def hmult_rescale_fused(b0, a0, b1, a1, basis, rlk, chain_q, chain_p, alpha, dnum,
                        threads=None):
    """The build's fused HMULT+rescale (capi.cu moddown_rescale) restated, so
    the CPU suite can check its algebra against rescale(hmult(.)) (ckks.py
    :265-274 then :291-311): with X_i = acc_i P^-1 + d_i, conv_i the converted
    special rows and T = INTT_top(ModDown_top + d_top),
        rescale_i = (X_i - NTT_i(conv_i P^-1 + T)) q_top^-1."""
    basis = tuple(basis)
    sp = tuple(chain_p)
    ext = basis + sp
    q_top = basis[-1]
    d0 = hada_mult(b0, b1, basis)
    d1 = ele_add(hada_mult(a0, b1, basis), hada_mult(a1, b0, basis), basis)
    d2 = hada_mult(a0, a1, basis)
    accs = key_switch_acc(d2, basis, rlk, chain_q, chain_p, alpha, dnum, threads)
    big_p = 1
    for r in sp:
        big_p *= r
    outs = []
    for acc, dd in zip(accs, (d0, d1)):
        conv = fast_basis_conv(intt(acc[len(basis):], sp, threads), sp, basis)
        # the top row's ModDown alone, then its coefficient form
        qq = np.uint64(q_top)
        pinv = np.uint64(pow(big_p, -1, q_top))
        y = ntt(conv[-1:], (q_top,), threads)[0].astype(np.uint64)
        top = ((acc[len(basis) - 1].astype(np.uint64) + qq - y) % qq * pinv
               + dd[-1].astype(np.uint64)) % qq
        t = intt(top[None].astype(np.uint32), (q_top,), threads)[0].astype(np.uint64)
        w = np.empty((len(basis) - 1,) + acc.shape[1:], dtype=np.uint32)
        x = np.empty_like(w)
        for i, q in enumerate(basis[:-1]):
            qi = np.uint64(q)
            pi = np.uint64(pow(big_p, -1, q))
            x[i] = (acc[i].astype(np.uint64) * pi + dd[i].astype(np.uint64)) % qi
            w[i] = (conv[i].astype(np.uint64) % qi * pi + t % qi) % qi
        nw = ntt(w, basis[:-1], threads)
        out = np.empty_like(w)
        for i, q in enumerate(basis[:-1]):
            qi = np.uint64(q)
            out[i] = (x[i].astype(np.uint64) + qi - nw[i]) % qi * np.uint64(pow(q_top, -1, q)) % qi
        outs.append(out)
    return outs[0], outs[1]


def rescale_poly(c, basis, threads=None):
    """ckks.py:301-311 (all limbs to coeff, subtract top, scale, back to ntt)."""
    basis = tuple(basis)
    q_top = basis[-1]
    coeff = intt(c, basis, threads)
    top = coeff[-1].astype(np.uint64)
    out = np.empty((len(basis) - 1,) + c.shape[1:], dtype=np.uint32)
    for i, q in enumerate(basis[:-1]):
        qq = np.uint64(q)
        diff = (coeff[i].astype(np.uint64) + qq - top % qq) % qq
        out[i] = diff * np.uint64(pow(q_top, -1, q)) % qq
    return ntt(out, basis[:-1], threads)


def rescale(b, a, basis, threads=None):
    """ckks.py:291-299 -> (b', a') over basis[:-1]"""
    return rescale_poly(b, basis, threads), rescale_poly(a, basis, threads)


def hrotate(b, a, r, basis, rot_key, chain_q, chain_p, alpha, dnum, threads=None):
    """ckks.py:276-282"""
    n = b.shape[-1]
    t = galois_element(r, n)
    bt = apply_automorphism(b, t, basis)
    at = apply_automorphism(a, t, basis)
    ksb, ksa = key_switch(at, basis, rot_key, chain_q, chain_p, alpha, dnum, threads)
    return ele_add(bt, ksb, basis), ksa


def hconjugate(b, a, basis, conj_key, chain_q, chain_p, alpha, dnum, threads=None):
    """ckks.py:284-289"""
    n = b.shape[-1]
    t = 2 * n - 1
    bt = apply_automorphism(b, t, basis)
    at = apply_automorphism(a, t, basis)
    ksb, ksa = key_switch(at, basis, conj_key, chain_q, chain_p, alpha, dnum, threads)
    return ele_add(bt, ksb, basis), ksa


# ---------------------------------------------------------------------------
# client-side CRT (rns.py:77-115, ckks.py:194-213): Python big integers
# ---------------------------------------------------------------------------

def crt_decompose(coeffs, basis) -> np.ndarray:
    """Arbitrary-precision signed ints -> canonical residue rows (len(basis),
    len(coeffs)) (rns.py:77-90)."""
    return np.array([[int(c) % q for c in coeffs] for q in basis], dtype=np.uint32)


def encode_ints(coeffs) -> list:
    """encode's rounding of the float64 embedding (ckks.py:194-196):
    [int(c) for c in np.rint(coeffs)]."""
    return [int(c) for c in np.rint(np.asarray(coeffs, dtype=np.float64))]


def crt_compose_centered(rows, basis) -> list:
    """CRT representative in [0, Q) (rns.py:93-115) centred into (-Q/2, Q/2]
    (ckks.py:207-213 _centered)."""
    rows = np.asarray(rows)
    big_q = 1
    for q in basis:
        big_q *= q
    terms = [(big_q // q) * pow(big_q // q, -1, q) for q in basis]
    out = []
    for j in range(rows.shape[-1]):
        v = sum(f * int(rows[i, j]) for i, f in enumerate(terms)) % big_q
        out.append(v - big_q if v > big_q // 2 else v)
    return out


def uniform_rows(rng, basis, shape_tail):
    """cli._random_batch (cli.py:59-64): rng.integers(0, q, shape) per limb."""
    out = np.empty((len(basis),) + tuple(shape_tail), dtype=np.uint32)
    for i, q in enumerate(basis):
        out[i] = rng.integers(0, q, shape_tail, dtype=np.uint64)
    return out
