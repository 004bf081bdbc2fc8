"""RNS-CKKS evaluation operators on the B200 (operator API of ref `ckks.py`).

`CkksContext` keeps the reference's evaluation interface (`ckks.py:63-381`):
``to_ntt``, ``to_coeff``, ``hadd``, ``hsub``, ``cmult``, ``hmult``,
``hrotate``, ``hconjugate``, ``rescale`` and ``key_switch`` over
`Ciphertext` / `RnsPolynomial` objects, with the same checks and exceptions.
Every call is bit-identical to the reference's.

New here (TensorFHE operation-level batching): the ``*_batch`` methods take a
`CiphertextBatch` -- a (2, level+1, B, N) device tensor, component b then a,
level-major -- and run ONE native pipeline for the whole batch
(tfhe_hmult / tfhe_rescale / tfhe_hrotate / tfhe_keyswitch in csrc/capi.cu).
Each member equals the reference's per-member call (cli.py:175-191).

Key generation, encoding and encryption (the client side) come
from `client.ClientMixin`: host sampling / FFT / CRT exactly as the
reference (same seed -> same keys and ciphertexts), device transforms.  Keys
made by the reference itself (any `SwitchingKey` whose pairs cover
chain.q ++ chain.p) are accepted directly too.
"""

from __future__ import annotations

import weakref
from collections import OrderedDict
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _lib, kernels
from .client import ClientMixin
from .device import DeviceContext, to_device
from .errors import DomainError, ParameterError
from .ntt import BACKENDS, TwiddleTable, ntt_forward, ntt_inverse
from .rns import NTT, RnsPolynomial


@dataclass(frozen=True)
class Plaintext:
    poly: RnsPolynomial
    scale: Fraction
    level: int


@dataclass(frozen=True)
class Ciphertext:
    b: RnsPolynomial
    a: RnsPolynomial
    scale: Fraction
    level: int

    def __post_init__(self):
        if self.b.basis != self.a.basis:
            raise ParameterError("ciphertext component bases differ")


@dataclass(frozen=True)
class SecretKey:
    s: RnsPolynomial


@dataclass(frozen=True)
class PublicKey:
    b: RnsPolynomial
    a: RnsPolynomial


@dataclass(frozen=True)
class SwitchingKey:
    """dnum pairs (b_j, a_j) over the extended basis, ntt domain (ref `ckks.py:57-60`)."""
    pairs: tuple


@dataclass
class CiphertextBatch:
    """B ciphertexts at one level: data (2, level+1, B, N) int32 on the device."""
    data: torch.Tensor
    level: int
    scale: Fraction = Fraction(1)

    @property
    def batch_size(self):
        return int(self.data.shape[2])

    @property
    def n(self):
        return int(self.data.shape[3])


class CkksContext(ClientMixin):
    """Evaluation engine bound to one parameter set (ref `ckks.py:63-83`)."""

    def __init__(self, params, backend="segmented", seed=0, workers=None, device=None):
        if backend not in BACKENDS:
            raise ParameterError(f"unknown backend {backend!r}")
        self.params = params
        self.backend = backend
        self.workers = workers
        self.rng = np.random.default_rng(seed)
        self.ext_basis = tuple(params.chain.q) + tuple(params.chain.p)
        self.dev = DeviceContext.get(params.n, self.ext_basis, n_chain=len(params.chain.q),
                                     n_special=len(params.chain.p), device=device)
        self.table = TwiddleTable(params.n, self.ext_basis)
        self.table._ctx = self.dev
        # device copies of host switching keys: a small LRU keyed by the host
        # object's id, evicted when the host key is garbage-collected
        self._keys = OrderedDict()
        self.max_cached_keys = 4
        # the device path's limits (poly_ops.h): base conversions of at most
        # kMaxBconvSrc sources, primes below 2^31 (tfhe_ctx_create)
        if max(params.alpha, len(params.chain.p)) > _lib.MAX_BCONV_SRC:
            raise ParameterError(
                f"alpha={params.alpha} / K={len(params.chain.p)}: the device base conversion "
                f"takes at most {_lib.MAX_BCONV_SRC} source limbs")
        if max(self.ext_basis) >= 1 << 31:
            raise ParameterError("the device path needs primes below 2^31")

    # -- transforms -----------------------------------------------------------
    def to_ntt(self, poly):
        return ntt_forward(poly, self.table, self.backend)

    def to_coeff(self, poly):
        return ntt_inverse(poly, self.table, self.backend)

    # -- device layout helpers ------------------------------------------------
    def device_key(self, swk) -> torch.Tensor:
        """(dnum, 2, L+1+K, N) device copy of a switching key (cached per key)."""
        if isinstance(swk, torch.Tensor):
            return swk
        hit = self._keys.get(id(swk))
        if hit is not None and hit[0]() is swk:
            self._keys.move_to_end(id(swk))
            return hit[1]
        p = self.params
        if isinstance(swk, SwitchingKey):
            if len(swk.pairs) != p.dnum:
                raise ParameterError("switching key must hold dnum pairs")
            arr = np.empty((p.dnum, 2, len(self.ext_basis), p.n), dtype=np.uint32)
            for j, (kb, ka) in enumerate(swk.pairs):
                arr[j, 0] = kb.restrict(self.ext_basis).host_rows()
                arr[j, 1] = ka.restrict(self.ext_basis).host_rows()
        else:
            arr = np.asarray(swk, dtype=np.uint32)
        t, _ = to_device(arr, self.dev.device)
        try:
            ref = weakref.ref(swk)
            weakref.finalize(swk, self._keys.pop, id(swk), None)
        except TypeError:   # not weak-referenceable (e.g. a list): do not cache
            return t
        self._keys[id(swk)] = (ref, t)
        while len(self._keys) > self.max_cached_keys:
            self._keys.popitem(last=False)
        return t

    def _ct_tensor(self, ct):
        b, _ = to_device(ct.b.rows, self.dev.device)
        a, _ = to_device(ct.a.rows, self.dev.device)
        return torch.stack([b, a]).unsqueeze(2).contiguous()

    def _from_tensor(self, t, basis, scale, level, host):
        rows = [t[0, :, 0], t[1, :, 0]]
        if host:
            rows = [r.cpu().numpy().view(np.uint32) for r in rows]
        return Ciphertext(b=RnsPolynomial(rows=rows[0], basis=basis, domain=NTT),
                          a=RnsPolynomial(rows=rows[1], basis=basis, domain=NTT),
                          scale=scale, level=level)

    def _check_aligned(self, c0, c1, scale=True):
        if c0.level != c1.level:
            raise ParameterError("ciphertext levels differ")
        if scale and c0.scale != c1.scale:
            raise ParameterError("ciphertext scales differ")

    # -- homomorphic operations (single ciphertext, reference semantics) -----
    def hadd(self, c0, c1):
        self._check_aligned(c0, c1)
        return Ciphertext(b=kernels.ele_add(c0.b, c1.b), a=kernels.ele_add(c0.a, c1.a),
                          scale=c0.scale, level=c0.level)

    def hsub(self, c0, c1):
        self._check_aligned(c0, c1)
        return Ciphertext(b=kernels.ele_sub(c0.b, c1.b), a=kernels.ele_sub(c0.a, c1.a),
                          scale=c0.scale, level=c0.level)

    def cmult(self, ct, pt):
        if pt.level != ct.level:
            raise ParameterError("plaintext level does not match ciphertext")
        return Ciphertext(b=kernels.hada_mult(ct.b, pt.poly), a=kernels.hada_mult(ct.a, pt.poly),
                          scale=ct.scale * pt.scale, level=ct.level)

    def hmult(self, c0, c1, rlk):
        """Tensor product + relinearising key switch (ref `ckks.py:265-274`)."""
        self._check_aligned(c0, c1, scale=False)
        out = self.dev.hmult(self._ct_tensor(c0), self._ct_tensor(c1), c0.level,
                             self.device_key(rlk), self.params.dnum)
        return self._from_tensor(out, c0.b.basis, c0.scale * c1.scale, c0.level,
                                 not c0.b.on_device)

    def key_switch(self, d, swk):
        """(ksb, ksa) over d's basis (ref `ckks.py:321-352`)."""
        if d.domain != NTT:
            raise DomainError("key_switch needs an ntt-domain input")
        level = d.level_count - 1
        x, host = to_device(d.rows, self.dev.device)
        out = self.dev.keyswitch(x.view(level + 1, 1, d.n), level, self.device_key(swk),
                                 self.params.dnum)
        ct = self._from_tensor(out, d.basis, Fraction(1), level, host)
        return ct.b, ct.a

    def hrotate(self, ct, r, rot_key):
        """Rotate slots left by r (ref `ckks.py:276-282`)."""
        t = kernels.galois_element(r, self.params.n)
        out = self.dev.hrotate(self._ct_tensor(ct), ct.level, t, self.device_key(rot_key),
                               self.params.dnum)
        return self._from_tensor(out, ct.b.basis, ct.scale, ct.level, not ct.b.on_device)

    def hconjugate(self, ct, conj_key):
        """Complex conjugation (ref `ckks.py:284-289`)."""
        t = 2 * self.params.n - 1
        out = self.dev.hrotate(self._ct_tensor(ct), ct.level, t, self.device_key(conj_key),
                               self.params.dnum)
        return self._from_tensor(out, ct.b.basis, ct.scale, ct.level, not ct.b.on_device)

    def rescale(self, ct):
        """Drop the top prime, divide the scale by it (ref `ckks.py:291-299`)."""
        if ct.level < 1:
            raise ParameterError("no levels left to rescale")
        q_top = ct.b.basis[-1]
        out = self.dev.rescale(self._ct_tensor(ct), ct.level)
        return self._from_tensor(out, ct.b.basis[:-1], ct.scale / q_top, ct.level - 1,
                                 not ct.b.on_device)

    # -- batched operations (one native pipeline per call) -------------------
    def batch_from_ciphertexts(self, cts) -> CiphertextBatch:
        if not cts:
            raise ParameterError("empty ciphertext batch")
        lvl = cts[0].level
        for c in cts:
            if c.level != lvl:
                raise ParameterError("batch members must share a level")
        data = torch.cat([self._ct_tensor(c) for c in cts], dim=2).contiguous()
        return CiphertextBatch(data=data, level=lvl, scale=cts[0].scale)

    def batch_to_ciphertexts(self, cb: CiphertextBatch, host=True):
        basis = self.params.q_basis(cb.level)
        return [self._from_tensor(cb.data[:, :, b:b + 1], basis, cb.scale, cb.level, host)
                for b in range(cb.batch_size)]

    def hmult_batch(self, c0: CiphertextBatch, c1: CiphertextBatch, rlk, out=None):
        if c0.level != c1.level or c0.data.shape != c1.data.shape:
            raise ParameterError("batch operands must match in level and shape")
        d = self.dev.hmult(c0.data, c1.data, c0.level, self.device_key(rlk), self.params.dnum,
                           out=out)
        return CiphertextBatch(data=d, level=c0.level, scale=c0.scale * c1.scale)

    def hmult_rescale_batch(self, c0: CiphertextBatch, c1: CiphertextBatch, rlk, out=None):
        """`rescale_batch(hmult_batch(c0, c1, rlk))` in one pipeline, bit-identical:
        ModDown's and the rescale's forward NTTs merge by linearity (2*level
        fewer limb-NTTs; capi.cu moddown_rescale)."""
        if c0.level != c1.level or c0.data.shape != c1.data.shape:
            raise ParameterError("batch operands must match in level and shape")
        if c0.level < 1:
            raise ParameterError("no levels left to rescale")
        q_top = self.params.chain.q[c0.level]
        d = self.dev.hmult_rescale(c0.data, c1.data, c0.level, self.device_key(rlk),
                                   self.params.dnum, out=out)
        return CiphertextBatch(data=d, level=c0.level - 1, scale=c0.scale * c1.scale / q_top)

    def rescale_batch(self, cb: CiphertextBatch, out=None):
        if cb.level < 1:
            raise ParameterError("no levels left to rescale")
        q_top = self.params.chain.q[cb.level]
        d = self.dev.rescale(cb.data, cb.level, out=out)
        return CiphertextBatch(data=d, level=cb.level - 1, scale=cb.scale / q_top)

    def hrotate_batch(self, cb: CiphertextBatch, r, rot_key, out=None):
        t = kernels.galois_element(r, self.params.n)
        d = self.dev.hrotate(cb.data, cb.level, t, self.device_key(rot_key), self.params.dnum,
                             out=out)
        return CiphertextBatch(data=d, level=cb.level, scale=cb.scale)

    def hconjugate_batch(self, cb: CiphertextBatch, conj_key, out=None):
        d = self.dev.hrotate(cb.data, cb.level, 2 * self.params.n - 1,
                             self.device_key(conj_key), self.params.dnum, out=out)
        return CiphertextBatch(data=d, level=cb.level, scale=cb.scale)

    def key_switch_batch(self, d: torch.Tensor, level: int, swk, out=None):
        """d: (level+1, B, N) NTT domain -> (2, level+1, B, N) = (ksb, ksa)."""
        return self.dev.keyswitch(d, level, self.device_key(swk), self.params.dnum, out=out)

    def _binary_batch(self, op, c0: CiphertextBatch, c1: CiphertextBatch):
        """ele_add / ele_sub of both components of every member: one launch
        over the (2 (level+1), B, N) rows, row i mod q_{i mod (level+1)}."""
        if c0.level != c1.level or c0.data.shape != c1.data.shape:
            raise ParameterError("batch operands must match in level and shape")
        if c0.scale != c1.scale:
            raise ParameterError("ciphertext scales differ")
        basis = self.params.q_basis(c0.level)
        l1, B, n = len(basis), c0.batch_size, c0.n
        if tuple(c0.data.shape) != (2, l1, B, n):
            raise ParameterError("ciphertext batch must be (2, level+1, B, N)")
        a = c0.data.reshape(2 * l1, B, n)
        b = c1.data.reshape(2 * l1, B, n)
        d = self.dev.eltwise(op, a, b, basis * 2)
        return CiphertextBatch(data=d.view(2, l1, B, n), level=c0.level, scale=c0.scale)

    def hadd_batch(self, c0: CiphertextBatch, c1: CiphertextBatch):
        """hadd (ref `ckks.py:246-250`) of every member."""
        return self._binary_batch(_lib.OP_ADD, c0, c1)

    def hsub_batch(self, c0: CiphertextBatch, c1: CiphertextBatch):
        """hsub (ref `ckks.py:252-256`) of every member."""
        return self._binary_batch(_lib.OP_SUB, c0, c1)

    def cmult_batch(self, cb: CiphertextBatch, pt, pt_scale=None):
        """Plaintext product (ref `ckks.py:258-263`) of every member: pt is a
        (level+1, B, N) NTT-domain tensor (one plaintext per member) or a
        single `Plaintext` / (level+1, N) tensor shared by the batch.  A raw
        tensor carries no scale, so `pt_scale` is required with it (the result
        scale is cb.scale * pt_scale, as the reference's)."""
        basis = self.params.q_basis(cb.level)
        l1, B, n = len(basis), cb.batch_size, cb.n
        if isinstance(pt, Plaintext):
            if pt.level != cb.level:
                raise ParameterError("plaintext level does not match ciphertext")
            scale = cb.scale * pt.scale
            pt = pt.poly.rows
        else:
            if pt_scale is None:
                raise ParameterError("cmult_batch of a raw plaintext tensor needs pt_scale")
            scale = cb.scale * Fraction(pt_scale)
        t, _ = to_device(pt, self.dev.device)
        if tuple(t.shape) == (l1, n):
            t = t.unsqueeze(1).expand(l1, B, n).contiguous()
        if tuple(t.shape) != (l1, B, n):
            raise ParameterError("plaintext batch must be (level+1, B, N) or (level+1, N)")
        out = torch.empty_like(cb.data)
        for c in range(2):
            self.dev.eltwise(_lib.OP_MUL, cb.data[c], t, basis, out=out[c])
        return CiphertextBatch(data=out, level=cb.level, scale=scale)

