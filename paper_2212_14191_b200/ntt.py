"""Negacyclic NTT / INTT on the B200 tensor cores (operator API of ref `ntt.py`).

Same entry points as the reference (`ntt.py:347-385`):

* ``transform_rows(x, q, table, backend, inverse=False, workers=None)``
* ``ntt_forward(poly, table, backend, workers)`` / ``ntt_inverse(...)``
* ``TwiddleTable(n, primes)``

The reference's plugin point is the backend string (`ntt.py:30`).  Its three
backends are bit-identical by construction, and all three names are accepted
here for drop-in compatibility; every one of them runs the single sm_100a
implementation -- TensorFHE's "segmented" formulation on int8 tcgen05 MMAs
(csrc/ntt_tc.cu).  ``"tcgen05"`` names it explicitly.  There is no CPU path:
without the extension every call raises DeviceError.

Outputs are bit-identical to the reference on the same inputs (tests/).
Host numpy inputs return host numpy outputs (uint64 like the reference's
transform_rows); CUDA tensor inputs return CUDA int32 tensors (u32 bits).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import params as par
from .device import HOST_NUMPY, DeviceContext, like_input, to_device
from .errors import DomainError, ParameterError
from .rns import COEFF, NTT, RnsPolynomial

#: reference names (all bit-identical, all served by the tensor-core kernel) + native name
BACKENDS = ("butterfly", "gemm", "segmented", "tcgen05")


def _check_backend(backend):
    if backend not in BACKENDS:
        raise ParameterError(f"unknown backend {backend!r}")


@dataclass
class PrimeEntry:
    q: int
    psi: int
    n_inv: int


class TwiddleTable:
    """Per-prime NTT constants for one degree (ref `ntt.py:115-165`).

    Host side it records psi / n^-1 per prime exactly like the reference;
    the device tables (byte-split twiddle tiles, Hadamard twiddles, Barrett
    constants) are built once by the extension and cached in a
    DeviceContext shared with every other operator on these primes.
    """

    def __init__(self, n, primes, device=None):
        self.n = int(n)
        self.plan = par.build_ntt_plan(self.n)
        self._entries = {}
        for q in primes:
            q = int(q)
            self._entries[q] = PrimeEntry(q=q, psi=par.find_negacyclic_root(q, self.n),
                                          n_inv=pow(self.n, q - 2, q))
        self._device = device
        self._ctx = None

    @property
    def primes(self):
        return tuple(self._entries)

    def entry(self, q):
        try:
            return self._entries[int(q)]
        except KeyError:
            raise ParameterError(f"no twiddles prepared for prime {q}") from None

    def twiddles(self, q, direction):
        """Host copy of W1/W2/W3 (params.build_twiddles), for inspection."""
        e = self.entry(q)
        return par.build_twiddles(self.plan, q, e.psi, direction)

    def context(self) -> DeviceContext:
        if self._ctx is None:
            self._ctx = DeviceContext.get_for(self.n, self.primes, self._device)
        return self._ctx


def transform_rows(x, q, table, backend="segmented", inverse=False, workers=None):
    """Transform a (batch, n) block of residues for a single prime (ref `ntt.py:347-363`).

    ``workers`` is accepted for signature compatibility (the reference uses
    it to thread its 16 partial GEMMs); the device schedule is fixed.
    """
    _check_backend(backend)
    table.entry(q)
    ctx = table.context()
    t, host = to_device(x, ctx.device)
    shape = t.shape
    n = int(shape[-1])
    if n != table.n:
        raise ParameterError(f"row length {n} does not match table degree {table.n}")
    rows = t.reshape(1, -1, n)
    out = ctx.ntt(rows, [int(q)], inverse=inverse).reshape(shape)
    if host == HOST_NUMPY:  # reference returns uint64 rows (ntt.py:351)
        return out.cpu().numpy().view(np.uint32).astype(np.uint64)
    return like_input(out, host)


def _poly_transform(poly, table, inverse):
    ctx = table.context()
    for q in poly.basis:
        table.entry(q)
    t, host = to_device(poly.rows, ctx.device)
    L = len(poly.basis)
    out = ctx.ntt(t.view(L, 1, poly.n), list(poly.basis), inverse=inverse).view(L, poly.n)
    return RnsPolynomial(rows=like_input(out, host), basis=poly.basis,
                         domain=COEFF if inverse else NTT)


def ntt_forward(poly, table, backend="segmented", workers=None):
    """Forward transform of every residue row; flips domain to ntt (ref `ntt.py:366-374`)."""
    _check_backend(backend)
    if poly.domain != COEFF:
        raise DomainError("ntt_forward needs a coefficient-domain input")
    return _poly_transform(poly, table, inverse=False)


def ntt_inverse(poly, table, backend="segmented", workers=None):
    """Inverse transform with n^-1; flips domain to coeff (ref `ntt.py:377-385`)."""
    _check_backend(backend)
    if poly.domain != NTT:
        raise DomainError("ntt_inverse needs an ntt-domain input")
    return _poly_transform(poly, table, inverse=True)
