"""B200-native batched RNS-CKKS hot path (TensorFHE, arXiv 2212.14191).

Drop-in for the reference `rnsckks` operator layer on the hot path: NTT/INTT
(int8 tcgen05 tensor-core formulation), element-wise and automorphism
kernels, fast base conversion, key switching, HMULT, RESCALE and HROTATE,
over RNS ciphertext batches.  Host-side parameter generation matches the
reference bit for bit; all compute runs in the sm_100a extension
(libtfhe_b200.so, C ABI in include/tfhe_b200.h).
"""

from .errors import BatchError, CapacityError, DeviceError, DomainError, ParameterError
from .params import CkksParams, ModulusChain, NttPlan, PRESETS
from .rns import COEFF, NTT, RnsPolynomial, crt_compose, crt_decompose, fast_basis_conv

__version__ = "0.1.0"


def __getattr__(name):
    # device-facing modules import torch lazily so `import paper_2212_14191_b200`
    # stays cheap for host-only use (parameters, CPU tests)
    if name in ("BACKENDS", "TwiddleTable", "ntt_forward", "ntt_inverse", "transform_rows"):
        from . import ntt
        return getattr(ntt, name)
    if name in ("Ciphertext", "CkksContext", "Plaintext", "PublicKey", "SecretKey",
                "SwitchingKey", "CiphertextBatch"):
        from . import ckks
        return getattr(ckks, name)
    if name in ("BatchBuffer", "batched_apply", "pack", "plan_batch_size", "reorder_layout",
                "unpack"):
        from . import batch
        return getattr(batch, name)
    raise AttributeError(name)


__all__ = [
    "BACKENDS", "BatchBuffer", "BatchError", "CapacityError", "Ciphertext", "CiphertextBatch",
    "CkksContext", "CkksParams", "COEFF", "DeviceError", "DomainError", "ModulusChain", "NTT",
    "NttPlan", "ParameterError", "Plaintext", "PRESETS", "PublicKey", "RnsPolynomial",
    "SecretKey", "SwitchingKey", "TwiddleTable", "batched_apply", "crt_compose",
    "crt_decompose", "fast_basis_conv", "ntt_forward", "ntt_inverse", "pack",
    "plan_batch_size", "reorder_layout", "transform_rows", "unpack",
]
