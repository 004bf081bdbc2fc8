"""Device contexts and buffer plumbing between the operator API and the C ABI.

PyTorch is used here only as the device-memory / stream plumbing: residues
live in int32 CUDA tensors (bit-identical views of u32), raw pointers and the
current stream go to the extension, and nothing is computed by torch.

`DeviceContext` owns one `TfheCtx` (twiddle and constant tables on one GPU)
for a degree n and an ordered prime list.  Contexts are cached per
(device, n, primes, n_chain, n_special) so every operator reuses them.
"""

from __future__ import annotations

import ctypes
import threading
import warnings

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, ParameterError
from .params import find_negacyclic_root

_CTX_CACHE: dict = {}
_LOCK = threading.Lock()


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


#: residency tags returned by to_device (host tags are truthy)
ON_DEVICE, HOST_NUMPY, HOST_TORCH = "", "numpy", "torch"


def to_device(x, device=None):
    """numpy / torch (u32 or i32) -> (contiguous int32 CUDA tensor, residency tag).

    Host torch tensors in pinned memory are copied asynchronously on the
    current stream; numpy arrays go through a staging copy.
    """
    device = device or default_device()
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.uint32:
            x = x.view(torch.int32)
        elif x.dtype != torch.int32:
            x = x.to(torch.int64).to(torch.int32)
        tag = ON_DEVICE if x.device.type == "cuda" else HOST_TORCH
        return x.to(device, non_blocking=True).contiguous(), tag
    a = np.asarray(x)
    if a.dtype != np.uint32:
        a = a.astype(np.uint32)
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a.view(np.int32)).to(device), HOST_NUMPY


def to_host(t) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


def like_input(t, tag):
    """Return a device result with the residency of the caller's input."""
    if tag == HOST_NUMPY:
        return to_host(t)
    if tag == HOST_TORCH:
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return out
    return t


class DeviceContext:
    """Constant tables for degree n over `primes` (chain first, then specials)."""

    def __init__(self, n: int, primes, n_chain: int | None = None, n_special: int = 0,
                 device=None):
        self.lib = _lib.load()
        self.device = torch.device(device) if device is not None else default_device()
        self.n = int(n)
        self.log_n = self.n.bit_length() - 1
        self.primes = tuple(int(q) for q in primes)
        self.n_chain = len(self.primes) - n_special if n_chain is None else int(n_chain)
        self.n_special = int(n_special)
        if self.n_chain + self.n_special != len(self.primes):
            raise ParameterError("n_chain + n_special must equal the prime count")
        self.index = {q: i for i, q in enumerate(self.primes)}
        psis = [find_negacyclic_root(q, self.n) for q in self.primes]
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.tfhe_ctx_create(
                self.device.index or 0, self.log_n, _lib.u32_array(self.primes),
                _lib.u32_array(psis), self.n_chain, self.n_special, ctypes.byref(handle)),
                "tfhe_ctx_create")
        self.handle = handle
        n1, n2 = ctypes.c_int(), ctypes.c_int()
        self.lib.tfhe_ctx_plan(self.handle, ctypes.byref(n1), ctypes.byref(n2))
        self.plan = (n1.value, n2.value)
        k = [ctypes.c_int() for _ in range(3)]
        self.lib.tfhe_ctx_transform_plan(self.handle, *[ctypes.byref(v) for v in k])
        #: contraction lengths of the device factorisation (tfhe_ctx_transform_plan)
        self.transform_plan = tuple(v.value for v in k)
        self._ws = {}          # stream handle -> byte workspace
        self._staging = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and getattr(self, "lib", None) is not None:
            try:
                self.lib.tfhe_ctx_destroy(h)
            except Exception:
                pass

    @classmethod
    def get(cls, n, primes, n_chain=None, n_special=0, device=None) -> "DeviceContext":
        dev = torch.device(device) if device is not None else default_device()
        key = (str(dev), int(n), tuple(int(q) for q in primes), n_chain, n_special)
        with _LOCK:
            ctx = _CTX_CACHE.get(key)
            if ctx is None:
                ctx = cls(n, primes, n_chain, n_special, dev)
                _CTX_CACHE[key] = ctx
        return ctx

    @classmethod
    def get_for(cls, n, primes, device=None) -> "DeviceContext":
        """Any cached context of degree n on `device` whose primes cover
        `primes` (e.g. the CkksContext's extended basis), else a new one."""
        dev = torch.device(device) if device is not None else default_device()
        need = set(int(q) for q in primes)
        with _LOCK:
            for key, ctx in _CTX_CACHE.items():
                if key[0] == str(dev) and key[1] == int(n) and need <= set(ctx.primes):
                    return ctx
        return cls.get(n, tuple(sorted(need, reverse=True)), device=dev)

    # -- helpers --------------------------------------------------------------
    def prime_ids(self, primes):
        try:
            return [self.index[int(q)] for q in primes]
        except KeyError as e:
            raise ParameterError(f"no twiddles prepared for prime {e.args[0]}") from None

    def workspace(self, nbytes: int) -> torch.Tensor:
        """Byte workspace of the CURRENT stream (grown on demand, reused by the
        calls stream-ordered behind each other).  Every operator enqueues on
        the current stream, so ops issued on different streams (threads or
        `torch.cuda.stream` scopes) get disjoint scratch and cannot race."""
        nbytes = max(int(nbytes), 256)
        key = torch.cuda.current_stream(self.device).cuda_stream
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            self._ws.pop(key, None)
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def empty(self, *shape):
        return torch.empty(shape, dtype=torch.int32, device=self.device)

    # -- operators ------------------------------------------------------------
    def ntt(self, x, limb_primes, inverse=False, in_rows=None, out_rows=None, out=None,
            out_rows_total=None):
        """x: (rows, batch, n) int32 CUDA tensor.  Output row l = transform of
        x[in_rows[l]] mod limb_primes[l] (prime values)."""
        L = len(limb_primes)
        batch = x.shape[1]
        if out is None:
            out = self.empty(out_rows_total or L, batch, self.n)
        ws_bytes = self.lib.tfhe_ntt_workspace_bytes(self.handle, L, batch)
        ws = self.workspace(ws_bytes)
        _lib.check(self.lib.tfhe_ntt(
            self.handle, _ptr(x), _ptr(out), _lib.i32_array(self.prime_ids(limb_primes)),
            _lib.i32_array(in_rows) if in_rows is not None else None,
            _lib.i32_array(out_rows) if out_rows is not None else None,
            L, batch, int(bool(inverse)), _ptr(ws), ws.numel(), _stream(self.device)),
            "tfhe_ntt")
        return out

    def ntt_host(self, x, limb_primes, inverse=False):
        """Host-to-host batched transform of x (rows, batch, n) -- a CPU torch
        tensor (pinned for full overlap) or a numpy array -- streamed through
        the device in chunks with H2D / transform / D2H overlapped
        (tfhe_ntt_host).  Returns the same kind of host buffer (pinned)."""
        numpy_in = not isinstance(x, torch.Tensor)
        if numpy_in:
            a = np.ascontiguousarray(x, dtype=np.uint32)
            with warnings.catch_warnings():   # read-only input: only ever read
                warnings.simplefilter("ignore")
                xt = torch.from_numpy(a.view(np.int32))
        else:
            xt = (x.view(torch.int32) if x.dtype == torch.uint32
                  else x.to(torch.int32)).contiguous()
        if xt.ndim != 3:
            raise ParameterError("ntt_host expects (rows, batch, n)")
        L, batch = int(xt.shape[0]), int(xt.shape[1])
        # the result lands in pinned memory from torch's caching host allocator
        # (reused across calls; a fresh pageable array would page-fault on
        # every call); a pageable numpy input is bounced by the library
        out = torch.empty(tuple(xt.shape), dtype=torch.int32, pin_memory=True)
        nbytes = max(int(self.lib.tfhe_ntt_host_staging_bytes(self.handle, L, batch)), 256)
        if self._staging is None or self._staging.numel() < nbytes:
            self._staging = None
            self._staging = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        _lib.check(self.lib.tfhe_ntt_host(
            self.handle, ctypes.c_void_p(xt.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            _lib.i32_array(self.prime_ids(limb_primes)), L, batch, int(bool(inverse)),
            _ptr(self._staging), self._staging.numel(), _stream(self.device)), "tfhe_ntt_host")
        torch.cuda.current_stream(self.device).synchronize()
        return out.numpy().view(np.uint32) if numpy_in else out

    def eltwise(self, op, a, b, row_primes, scalars=None, out=None):
        rows = a.shape[0]
        per_row = a.numel() // max(rows, 1)
        if out is None:
            out = torch.empty_like(a)
        _lib.check(self.lib.tfhe_eltwise(
            self.handle, op, _ptr(a), _ptr(b), _ptr(out),
            _lib.i32_array(self.prime_ids(row_primes)), rows, per_row,
            _lib.u32_array(scalars) if scalars is not None else None, _stream(self.device)),
            "tfhe_eltwise")
        return out

    def automorphism(self, x, t, ntt_domain, row_primes, out=None):
        rows, batch = x.shape[0], x.shape[1]
        if out is None:
            out = torch.empty_like(x)
        _lib.check(self.lib.tfhe_automorphism(
            self.handle, _ptr(x), _ptr(out), int(t), int(bool(ntt_domain)),
            _lib.i32_array(self.prime_ids(row_primes)), rows, batch, _stream(self.device)),
            "tfhe_automorphism")
        return out

    def bconv(self, x, src, dst, out=None):
        batch = x.shape[1]
        if out is None:
            out = self.empty(len(dst), batch, self.n)
        _lib.check(self.lib.tfhe_bconv(
            self.handle, _ptr(x), _ptr(out), _lib.i32_array(self.prime_ids(src)), len(src),
            _lib.i32_array(self.prime_ids(dst)), len(dst), batch, _stream(self.device)),
            "tfhe_bconv")
        return out

    def crt_decompose(self, coeffs, basis, out=None):
        """Signed coefficients (device int64, or float64 rounded half to even
        like np.rint) -> canonical residue rows (len(basis), n) (ref
        rns.py:77-90 crt_decompose)."""
        n = coeffs.numel()
        if coeffs.dtype == torch.int64:
            kind = 0
        elif coeffs.dtype == torch.float64:
            kind = 1
        else:
            raise ParameterError("crt_decompose takes int64 or float64 coefficients")
        if out is None:
            out = torch.empty((len(basis), n), dtype=torch.int32, device=self.device)
        _lib.check(self.lib.tfhe_crt_decompose(
            self.handle, _ptr(coeffs), kind, n, _lib.i32_array(self.prime_ids(basis)), len(basis),
            _ptr(out), _stream(self.device)), "tfhe_crt_decompose")
        return out

    def crt_compose(self, rows, basis, words=False):
        """Residue rows (len(basis), n) -> the CRT representative centred in
        (-Q/2, Q/2] (ref rns.py:93-115 + ckks._centered) as correctly rounded
        float64, and with words=True also as (n_words, n) two's-complement
        32-bit words."""
        n = rows.shape[-1]
        ids = _lib.i32_array(self.prime_ids(basis))
        out_f = torch.empty(n, dtype=torch.float64, device=self.device)
        w = None
        n_words = 0
        if words:
            n_words = self.lib.tfhe_crt_words(self.handle, ids, len(basis)) + 1
            w = torch.empty((n_words, n), dtype=torch.int32, device=self.device)
        _lib.check(self.lib.tfhe_crt_compose(
            self.handle, _ptr(rows), ids, len(basis), n, _ptr(out_f), _ptr(w), n_words,
            _stream(self.device)), "tfhe_crt_compose")
        return (out_f, w) if words else out_f

    def ckks_workspace(self, level, batch):
        return self.workspace(self.lib.tfhe_ckks_workspace_bytes(self.handle, level, batch))

    def keyswitch(self, d, level, key, dnum, add=None, out=None):
        batch = d.shape[1]
        if out is None:
            out = self.empty(2, level + 1, batch, self.n)
        ws = self.ckks_workspace(level, batch)
        _lib.check(self.lib.tfhe_keyswitch(
            self.handle, _ptr(d), level, batch, _ptr(key), dnum, _ptr(out), _ptr(add),
            _ptr(ws), ws.numel(), _stream(self.device)), "tfhe_keyswitch")
        return out

    def hmult(self, ct0, ct1, level, rlk, dnum, out=None):
        batch = ct0.shape[2]
        if out is None:
            out = self.empty(2, level + 1, batch, self.n)
        ws = self.ckks_workspace(level, batch)
        _lib.check(self.lib.tfhe_hmult(
            self.handle, _ptr(ct0), _ptr(ct1), level, batch, _ptr(rlk), dnum, _ptr(out),
            _ptr(ws), ws.numel(), _stream(self.device)), "tfhe_hmult")
        return out

    def hmult_rescale(self, ct0, ct1, level, rlk, dnum, out=None):
        """rescale(hmult(ct0, ct1)) in one native pipeline (bit-identical)."""
        batch = ct0.shape[2]
        if out is None:
            out = self.empty(2, level, batch, self.n)
        ws = self.ckks_workspace(level, batch)
        _lib.check(self.lib.tfhe_hmult_rescale(
            self.handle, _ptr(ct0), _ptr(ct1), level, batch, _ptr(rlk), dnum, _ptr(out),
            _ptr(ws), ws.numel(), _stream(self.device)), "tfhe_hmult_rescale")
        return out

    def rescale(self, ct, level, out=None):
        batch = ct.shape[2]
        if out is None:
            out = self.empty(2, level, batch, self.n)
        ws = self.ckks_workspace(level, batch)
        _lib.check(self.lib.tfhe_rescale(
            self.handle, _ptr(ct), level, batch, _ptr(out), _ptr(ws), ws.numel(),
            _stream(self.device)), "tfhe_rescale")
        return out

    def hrotate(self, ct, level, galois_t, key, dnum, out=None):
        batch = ct.shape[2]
        if out is None:
            out = self.empty(2, level + 1, batch, self.n)
        ws = self.ckks_workspace(level, batch)
        _lib.check(self.lib.tfhe_hrotate(
            self.handle, _ptr(ct), level, batch, int(galois_t), _ptr(key), dnum, _ptr(out),
            _ptr(ws), ws.numel(), _stream(self.device)), "tfhe_hrotate")
        return out
