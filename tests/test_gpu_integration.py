"""The reference-side ctypes binding shown in INTEGRATION.md, executed verbatim.

The ```python block of INTEGRATION.md §2 (what a reference maintainer would
add to rnsckks/ntt.py as a "b200" backend: tfhe_ctx_create +
tfhe_ntt_host over plain numpy host buffers, staging via cudaMalloc, no
torch) is extracted from the document and run against the golden vectors the
reference produced (tests/golden/ntt_small.npz, ntt_large.json), so the
documented integration is the tested one.
"""

import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
import synth

pytestmark = pytest.mark.gpu


def _stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# rnsckks/ntt\.py.*?)```", text, re.S).group(1)
    from paper_2212_14191_b200 import _lib
    from paper_2212_14191_b200.errors import ParameterError
    lib_path = _lib.LIB_PATH
    # the stub loads "libtfhe_b200.so" / "libcudart.so" by name: point them at
    # this build and at the CUDA runtime the build links against
    cudart = next(p for p in ("libcudart.so.12", "libcudart.so",
                              "/usr/local/cuda/lib64/libcudart.so") if _try_cdll(p))
    block = block.replace('"libtfhe_b200.so"', repr(lib_path)).replace('"libcudart.so"',
                                                                        repr(cudart))
    ns = {"ParameterError": ParameterError}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    return ns["_b200_transform"]


def _try_cdll(p):
    try:
        ctypes.CDLL(p)
        return True
    except OSError:
        return False


def test_integration_stub_small_golden(golden_params):
    from paper_2212_14191_b200 import ntt
    fn = _stub()
    small = np.load(os.path.join(GOLDEN, "ntt_small.npz"))
    for n in (16, 256, 4096):
        qs = golden_params["adhoc"][f"primes_{n}"]["q"]
        table = ntt.TwiddleTable(n, qs)
        for q in qs:
            x = small[f"x_{n}_{q}"]
            f = fn(x, q, table, False)
            assert f.dtype == np.uint64
            assert np.array_equal(f, small[f"fwd_{n}_{q}"]), (n, q)
            assert np.array_equal(fn(x, q, table, True), small[f"inv_{n}_{q}"]), (n, q)


def test_integration_stub_large_golden(golden_params):
    from paper_2212_14191_b200 import ntt
    fn = _stub()
    with open(os.path.join(GOLDEN, "ntt_large.json")) as fh:
        rec = json.load(fh)
    n = 1 << 16
    qs = golden_params["adhoc"][f"primes_{n}"]["q"][:2]
    table = ntt.TwiddleTable(n, qs)
    for q in qs:
        x = synth.ntt_rows(n, q, rows=2)
        f = fn(x, q, table, False).astype(np.uint32)
        assert hashlib.sha256(f.tobytes()).hexdigest() == rec[f"{n}_{q}"]["fwd"]
