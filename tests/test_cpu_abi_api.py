"""CPU tests of the C ABI library and the host-side operator API (no GPU).

* the shared library loads and exports every symbol include/tfhe_b200.h
  declares, with the declared ABI version;
* argument validation happens at the boundary (TFHE_EINVAL, no CUDA call);
* without a GPU every operator fails loudly (DeviceError) -- there is no CPU
  fallback -- while the reference's argument checks (ParameterError,
  DomainError, BatchError) fire first, exactly as in the reference.
"""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2212_14191_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib


def test_header_symbols_exported():
    lib = _lib()
    L = lib.load()
    header = open(os.path.join(ROOT, "include", "tfhe_b200.h")).read()
    declared = set(re.findall(r"\b(tfhe_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(L, name), f"{name} not exported"
    assert declared == set(lib.SIGNATURES), "ctypes binding out of sync with the header"
    assert L.tfhe_abi_version() == lib.ABI_VERSION


def test_ctx_create_validates_before_cuda():
    lib = _lib()
    L = lib.load()
    h = ctypes.c_void_p()
    # 97 is not 1 mod 2n for n = 2^6
    rc = L.tfhe_ctx_create(0, 6, lib.u32_array([97]), lib.u32_array([1]), 1, 0, ctypes.byref(h))
    assert rc == lib.EINVAL
    assert b"not 1 mod 2n" in L.tfhe_last_error()
    # bad psi for a valid prime
    rc = L.tfhe_ctx_create(0, 6, lib.u32_array([257]), lib.u32_array([2]), 1, 0, ctypes.byref(h))
    assert rc == lib.EINVAL and b"psi" in L.tfhe_last_error()
    assert L.tfhe_ntt(None, None, None, None, None, None, 0, 1, 0, None, 0, None) == lib.EINVAL


def _no_gpu():
    import torch
    return not torch.cuda.is_available()


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2212_14191_b200 import kernels, ntt
    from paper_2212_14191_b200.errors import DeviceError
    from paper_2212_14191_b200.rns import NTT, RnsPolynomial
    table = ntt.TwiddleTable(64, [257, 641])
    x = np.zeros((2, 64), dtype=np.uint64)
    with pytest.raises(DeviceError):
        ntt.transform_rows(x, 257, table, "segmented")
    p = RnsPolynomial(rows=np.zeros((2, 64), np.uint32), basis=(257, 641), domain=NTT)
    with pytest.raises(DeviceError):
        kernels.ele_add(p, p)


def test_reference_checks_fire_first():
    from paper_2212_14191_b200 import batch, kernels, ntt
    from paper_2212_14191_b200.errors import BatchError, DomainError, ParameterError
    from paper_2212_14191_b200.rns import COEFF, NTT, RnsPolynomial
    table = ntt.TwiddleTable(64, [257])
    with pytest.raises(ParameterError):
        ntt.transform_rows(np.zeros((1, 64)), 257, table, "fft")
    with pytest.raises(ParameterError):
        table.entry(97)
    c = RnsPolynomial(rows=np.zeros((1, 64), np.uint32), basis=(257,), domain=COEFF)
    with pytest.raises(DomainError):
        ntt.ntt_inverse(c, table)
    with pytest.raises(DomainError):
        kernels.hada_mult(c, c)
    with pytest.raises(ParameterError):
        kernels.apply_automorphism(c, 4)
    other = RnsPolynomial(rows=np.zeros((1, 64), np.uint32), basis=(641,), domain=COEFF)
    with pytest.raises(ParameterError):
        kernels.ele_add(c, other)
    buf = batch.pack([c, c])
    with pytest.raises(BatchError):
        batch.batched_apply(buf, "permute")
    with pytest.raises(BatchError):
        batch.batched_apply(buf, "intt", table=table)
    with pytest.raises(BatchError):
        batch.pack([])
    with pytest.raises(BatchError):
        batch.pack([c, RnsPolynomial(rows=np.zeros((1, 64), np.uint32), basis=(257,), domain=NTT)])


def test_batch_layout_helpers():
    from paper_2212_14191_b200 import batch
    from paper_2212_14191_b200.rns import COEFF, RnsPolynomial
    rng = np.random.default_rng(1)
    items = [RnsPolynomial(rows=rng.integers(0, 257, (2, 16)).astype(np.uint32),
                           basis=(257, 641), domain=COEFF) for _ in range(5)]
    buf = batch.pack(items)
    assert buf.data.shape == (2, 5, 16) and buf.data.flags.c_contiguous
    for x, y in zip(items, batch.unpack(buf)):
        assert np.array_equal(x.rows, y.rows)
    src = rng.integers(0, 99, (5, 3, 7)).astype(np.uint32)
    dst = batch.reorder_layout(src)
    assert dst.shape == (3, 5, 7) and dst[1, 4, 6] == src[4, 1, 6]
    assert np.array_equal(batch.reorder_layout(dst), src)


def test_planner_matches_reference_semantics():
    from paper_2212_14191_b200 import batch
    from paper_2212_14191_b200.errors import CapacityError
    from paper_2212_14191_b200.params import CkksParams
    p = CkksParams.generate(n=1 << 12, l_max=5, k=3, dnum=3)
    assert batch.plan_batch_size(batch.working_set_bytes(p, "ntt", 1), p, "ntt") == 1
    with pytest.raises(CapacityError):
        batch.plan_batch_size(1024, p, "ntt")
    assert batch.plan_batch_size(1 << 40, p, "ntt") == batch.MAX_BATCH


def test_shard_ranges_cover_batch():
    from paper_2212_14191_b200.shard import shard_range
    for b in (1, 7, 128, 1000):
        for w in (1, 2, 3, 8):
            spans = [shard_range(b, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == b
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
