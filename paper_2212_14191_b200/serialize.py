"""`TFHE1` serialization (ref `serialize.py:1-157`), byte-compatible, plus
loaders straight into device batches.

Wire layout (little-endian), as the reference writes it:

    "TFHE1" | u8 kind | 8-byte params digest
    poly    = u8 domain (0 coeff, 1 ntt) | u32 L | L x u32 primes | u32 n | L*n x u32 rows
    kinds   : 1 polynomial | 2 ciphertext (poly b, poly a, u64 num, u64 den, u32 level)
              3 switching key (u32 count, count x (poly b, poly a)) | 4 public key
              5 secret key | 6 plaintext (poly, u64 num, u64 den, u32 level)

A digest mismatch, wrong kind or bad magic raises ParameterError before any
payload is decoded (ref `serialize.py:66-74`).

New here: `load_ciphertext_batch` assembles many ciphertext blobs into one
`CiphertextBatch` (2, level+1, B, N) and `load_switching_key_device` a key
blob into the (dnum, 2, L+1+K, N) tensor the key switch reads -- the
residue rows are gathered into one pinned host buffer and moved with a
single host-to-device copy, so cached keys / ciphertext fixtures land in HBM
without per-polynomial round trips.
"""

from __future__ import annotations

import struct
from fractions import Fraction

import numpy as np
import torch

from .ckks import Ciphertext, CiphertextBatch, Plaintext, PublicKey, SecretKey, SwitchingKey
from .errors import ParameterError
from .rns import COEFF, NTT, RnsPolynomial

MAGIC = b"TFHE1"
KIND_POLY, KIND_CT, KIND_SWK, KIND_PK, KIND_SK, KIND_PT = 1, 2, 3, 4, 5, 6
DOMAINS = (COEFF, NTT)


class _Writer:
    def __init__(self, kind, digest):
        if len(digest) != 8:
            raise ParameterError("params digest must be 8 bytes")
        self.parts = [MAGIC, bytes([kind]), bytes(digest)]

    def u32(self, v):
        self.parts.append(struct.pack("<I", v))

    def poly(self, poly):
        rows = poly.host_rows() if hasattr(poly, "host_rows") else np.asarray(poly.rows)
        self.parts.append(struct.pack("<BI", DOMAINS.index(poly.domain), len(poly.basis)))
        self.parts.append(np.asarray(poly.basis, dtype="<u4").tobytes())
        self.parts.append(struct.pack("<I", poly.n))
        self.parts.append(np.ascontiguousarray(rows, dtype="<u4").tobytes())

    def scale(self, s):
        f = Fraction(s)
        self.parts.append(struct.pack("<QQ", f.numerator, f.denominator))

    def bytes(self):
        return b"".join(self.parts)


class _Reader:
    """Cursor over one blob; `rows=False` skips copying row data (index only)."""

    def __init__(self, buf, kind, digest):
        self.buf = memoryview(buf)
        if bytes(self.buf[:5]) != MAGIC:
            raise ParameterError("bad magic bytes")
        if self.buf[5] != kind:
            raise ParameterError(f"wrong payload kind {self.buf[5]}, wanted {kind}")
        if bytes(self.buf[6:14]) != bytes(digest):
            raise ParameterError("params digest mismatch")
        self.off = 14

    def u32(self):
        (v,) = struct.unpack_from("<I", self.buf, self.off)
        self.off += 4
        return v

    def poly_span(self):
        """(domain, basis, n, byte offset of the rows) and advance past the poly."""
        dom, blen = struct.unpack_from("<BI", self.buf, self.off)
        self.off += 5
        basis = tuple(int(x) for x in np.frombuffer(self.buf, "<u4", blen, self.off))
        self.off += 4 * blen
        (n,) = struct.unpack_from("<I", self.buf, self.off)
        self.off += 4
        start = self.off
        self.off += 4 * blen * n
        if self.off > len(self.buf):
            raise ParameterError("truncated payload")
        return DOMAINS[dom], basis, n, start

    def poly(self):
        dom, basis, n, start = self.poly_span()
        rows = np.frombuffer(self.buf, "<u4", len(basis) * n, start).reshape(len(basis), n)
        return RnsPolynomial(rows=rows.astype(np.uint32), basis=basis, domain=dom)

    def scale(self):
        num, den = struct.unpack_from("<QQ", self.buf, self.off)
        self.off += 16
        return Fraction(num, den)


# -- reference API (same names and behaviour) --------------------------------

def dump_polynomial(poly, digest):
    w = _Writer(KIND_POLY, digest)
    w.poly(poly)
    return w.bytes()


def load_polynomial(buf, digest):
    return _Reader(buf, KIND_POLY, digest).poly()


def dump_ciphertext(ct, digest):
    w = _Writer(KIND_CT, digest)
    w.poly(ct.b)
    w.poly(ct.a)
    w.scale(ct.scale)
    w.u32(ct.level)
    return w.bytes()


def load_ciphertext(buf, digest):
    r = _Reader(buf, KIND_CT, digest)
    b, a = r.poly(), r.poly()
    scale = r.scale()
    return Ciphertext(b=b, a=a, scale=scale, level=r.u32())


def dump_plaintext(pt, digest):
    w = _Writer(KIND_PT, digest)
    w.poly(pt.poly)
    w.scale(pt.scale)
    w.u32(pt.level)
    return w.bytes()


def load_plaintext(buf, digest):
    r = _Reader(buf, KIND_PT, digest)
    poly = r.poly()
    scale = r.scale()
    return Plaintext(poly=poly, scale=scale, level=r.u32())


def dump_public_key(pk, digest):
    w = _Writer(KIND_PK, digest)
    w.poly(pk.b)
    w.poly(pk.a)
    return w.bytes()


def load_public_key(buf, digest):
    r = _Reader(buf, KIND_PK, digest)
    return PublicKey(b=r.poly(), a=r.poly())


def dump_secret_key(sk, digest):
    w = _Writer(KIND_SK, digest)
    w.poly(sk.s)
    return w.bytes()


def load_secret_key(buf, digest):
    return SecretKey(s=_Reader(buf, KIND_SK, digest).poly())


def dump_switching_key(swk, digest):
    w = _Writer(KIND_SWK, digest)
    w.u32(len(swk.pairs))
    for b, a in swk.pairs:
        w.poly(b)
        w.poly(a)
    return w.bytes()


def load_switching_key(buf, digest):
    r = _Reader(buf, KIND_SWK, digest)
    return SwitchingKey(pairs=tuple((r.poly(), r.poly()) for _ in range(r.u32())))


# -- device loaders ---------------------------------------------------------------

def _to_device(host_u32, device):
    pinned = torch.from_numpy(host_u32.view(np.int32)).pin_memory()
    return pinned.to(device, non_blocking=True)


def load_ciphertext_batch(bufs, digest, device=None):
    """B ciphertext blobs (same level, basis, scale) -> CiphertextBatch with
    data (2, level+1, B, N) on the device (one H2D copy)."""
    if not bufs:
        raise ParameterError("empty ciphertext batch")
    spans, meta = [], None
    for buf in bufs:
        r = _Reader(buf, KIND_CT, digest)
        pb, pa = r.poly_span(), r.poly_span()
        scale = r.scale()
        level = r.u32()
        m = (pb[0], pb[1], pb[2], scale, level)
        if pb[:3] != pa[:3] or pb[0] != NTT:
            raise ParameterError("ciphertext components must share an ntt-domain basis")
        if meta is None:
            meta = m
        elif m != meta:
            raise ParameterError("batch members must share basis, level and scale")
        spans.append((r.buf, pb[3], pa[3]))
    _, basis, n, scale, level = meta
    L, B = len(basis), len(bufs)
    host = np.empty((2, L, B, n), dtype=np.uint32)
    for i, (mv, ob, oa) in enumerate(spans):
        host[0, :, i] = np.frombuffer(mv, "<u4", L * n, ob).reshape(L, n)
        host[1, :, i] = np.frombuffer(mv, "<u4", L * n, oa).reshape(L, n)
    dev = torch.device(device) if device is not None else torch.device("cuda")
    return CiphertextBatch(data=_to_device(host, dev), level=level, scale=scale)


def dump_ciphertext_batch(cb, basis, digest):
    """CiphertextBatch -> one TFHE1 ciphertext blob per member."""
    data = cb.data.cpu().numpy().view(np.uint32)
    out = []
    for i in range(cb.batch_size):
        ct = Ciphertext(b=RnsPolynomial(rows=data[0, :, i], basis=tuple(basis), domain=NTT),
                        a=RnsPolynomial(rows=data[1, :, i], basis=tuple(basis), domain=NTT),
                        scale=cb.scale, level=cb.level)
        out.append(dump_ciphertext(ct, digest))
    return out


def load_switching_key_device(buf, digest, ext_basis, device=None):
    """Switching-key blob -> (dnum, 2, len(ext_basis), N) device tensor, rows
    restricted / reordered to `ext_basis` (chain.q ++ chain.p), the layout
    tfhe_keyswitch reads (ckks.py:57-60)."""
    r = _Reader(buf, KIND_SWK, digest)
    count = r.u32()
    ext_basis = tuple(int(q) for q in ext_basis)
    host = None
    for j in range(count):
        for c in range(2):
            dom, basis, n, start = r.poly_span()
            if dom != NTT:
                raise ParameterError("switching keys are ntt-domain")
            idx = {q: i for i, q in enumerate(basis)}
            missing = [q for q in ext_basis if q not in idx]
            if missing:
                raise ParameterError(f"key lacks primes {missing[:3]}")
            if host is None:
                host = np.empty((count, 2, len(ext_basis), n), dtype=np.uint32)
            rows = np.frombuffer(r.buf, "<u4", len(basis) * n, start).reshape(len(basis), n)
            host[j, c] = rows[[idx[q] for q in ext_basis]]
    if host is None:
        raise ParameterError("empty switching key")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    return _to_device(host, dev)
