"""ctypes binding of the sm_100a extension (libtfhe_b200.so, include/tfhe_b200.h).

There is no fallback: if the library is missing or cannot load, every
operator raises DeviceError.  The library is built in-tree by
`__graft_entry__.build()` (or `make -C paper_2212_14191_b200/csrc`).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import DeviceError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
#: in-tree build; TFHE_B200_LIB may point at another build of the same ABI
#: (A/B performance experiments)
LIB_PATH = os.environ.get("TFHE_B200_LIB") or os.path.join(_HERE, "libtfhe_b200.so")
ABI_VERSION = 3

EINVAL = 2
ECUDA = 3

OP_ADD, OP_SUB, OP_MUL, OP_NEG, OP_SCALAR = 0, 1, 2, 3, 4
#: widest base conversion one device launch takes (csrc/poly_ops.h kMaxBconvSrc)
MAX_BCONV_SRC = 16

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p

#: every symbol include/tfhe_b200.h declares, with (restype, argtypes)
SIGNATURES = {
    "tfhe_abi_version": (ctypes.c_int, []),
    "tfhe_last_error": (ctypes.c_char_p, []),
    "tfhe_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _u32p, _u32p, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(_vp)]),
    "tfhe_ctx_destroy": (None, [_vp]),
    "tfhe_ctx_plan": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int)]),
    "tfhe_ntt_workspace_bytes": (ctypes.c_size_t, [_vp, ctypes.c_int, ctypes.c_int]),
    "tfhe_ntt": (ctypes.c_int, [_vp, _vp, _vp, _i32p, _i32p, _i32p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, _vp, ctypes.c_size_t, _vp]),
    "tfhe_eltwise": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _i32p, ctypes.c_int,
                                    ctypes.c_int64, _u32p, _vp]),
    "tfhe_automorphism": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint32, ctypes.c_int, _i32p,
                                         ctypes.c_int, ctypes.c_int, _vp]),
    "tfhe_bconv": (ctypes.c_int, [_vp, _vp, _vp, _i32p, ctypes.c_int, _i32p, ctypes.c_int,
                                  ctypes.c_int, _vp]),
    "tfhe_ckks_workspace_bytes": (ctypes.c_size_t, [_vp, ctypes.c_int, ctypes.c_int]),
    "tfhe_keyswitch": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                                      _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "tfhe_hmult": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                                  _vp, _vp, ctypes.c_size_t, _vp]),
    "tfhe_hmult_rescale": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp,
                                          ctypes.c_int, _vp, _vp, ctypes.c_size_t, _vp]),
    "tfhe_rescale": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                    ctypes.c_size_t, _vp]),
    "tfhe_hrotate": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, _vp,
                                    ctypes.c_int, _vp, _vp, ctypes.c_size_t, _vp]),
    "tfhe_ntt_host_staging_bytes": (ctypes.c_size_t, [_vp, ctypes.c_int, ctypes.c_int]),
    "tfhe_ntt_host": (ctypes.c_int, [_vp, _vp, _vp, _i32p, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, _vp, ctypes.c_size_t, _vp]),
    "tfhe_tensor_product": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _vp, _vp]),
    "tfhe_keyswitch_part": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                           ctypes.c_int, _vp, ctypes.c_size_t, _vp]),
    "tfhe_rescale_part": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, _vp, _vp, ctypes.c_size_t, _vp]),
    "tfhe_debug_corrupt_twiddle": (ctypes.c_int, [_vp, ctypes.c_int]),
    "tfhe_ctx_transform_plan": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int),
                                               ctypes.POINTER(ctypes.c_int),
                                               ctypes.POINTER(ctypes.c_int)]),
    "tfhe_crt_decompose": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int64, _i32p,
                                          ctypes.c_int, _vp, _vp]),
    "tfhe_crt_words": (ctypes.c_int, [_vp, _i32p, ctypes.c_int]),
    "tfhe_crt_compose": (ctypes.c_int, [_vp, _vp, _i32p, ctypes.c_int, ctypes.c_int64, _vp, _vp,
                                        ctypes.c_int, _vp]),
    "tfhe_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "tfhe_profile_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t]),
}

_lib = None


def build(force: bool = False) -> str:
    """Compile the extension in-tree with nvcc for sm_100a."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-j4", "-C", os.path.join(_HERE, "csrc")])
    return LIB_PATH


def load():
    """Load and bind the extension; raises DeviceError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"sm_100a extension not built ({LIB_PATH} missing); run __graft_entry__.build()")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        raise DeviceError(f"cannot load {LIB_PATH}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.tfhe_abi_version() != ABI_VERSION:
        raise DeviceError("libtfhe_b200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(rc: int, what: str):
    if rc == 0:
        return
    msg = (load().tfhe_last_error() or b"").decode(errors="replace")
    if rc == EINVAL:
        raise ParameterError(f"{what}: {msg}")
    raise DeviceError(f"{what} failed ({rc}): {msg}")


def i32_array(values):
    vals = [int(v) for v in values]
    arr = (ctypes.c_int32 * max(len(vals), 1))(*vals)
    return arr


def u32_array(values):
    vals = [int(v) for v in values]
    return (ctypes.c_uint32 * max(len(vals), 1))(*vals)


class kernel_timer:
    """Per-kernel device timing (tfhe_profile_enable / tfhe_profile_read):
    inside the `with` block every NTT-pass, fused-NTT and base-conversion
    launch is bracketed by CUDA events on its own stream; `.times` then maps
    kernel family -> (launches, total device ms)."""

    def __enter__(self):
        L = load()
        L.tfhe_profile_read(None, 0)   # drop stale records
        L.tfhe_profile_enable(1)
        self.times = {}
        return self

    def __exit__(self, *exc):
        L = load()
        L.tfhe_profile_enable(0)
        buf = ctypes.create_string_buffer(1 << 16)
        n = L.tfhe_profile_read(buf, len(buf))
        if n < 0:
            raise DeviceError("tfhe_profile_read failed: " +
                              (L.tfhe_last_error() or b"").decode(errors="replace"))
        for line in buf.value.decode().splitlines():
            name, count, ms = line.split("\t")
            self.times[name] = (int(count), float(ms))
        return False
