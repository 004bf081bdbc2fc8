"""Client-side CKKS operations (ref `ckks.py:85-239`): sampling, key
generation, encoding / decoding and encryption / decryption.

These run BEFORE and AFTER the evaluated path (the
lowest-priority row).  The random draws and the canonical-embedding FFT stay
host numpy exactly as in the reference -- same `numpy.random.default_rng(seed)`
stream, drawn in the same order with the same calls, same float64 FFT -- so a
given seed yields the reference's keys and ciphertexts bit for bit.  The
integer work runs on the device: rounding and CRT decomposition of the
encoded / sampled coefficients (`DeviceContext.crt_decompose`, exact for any
float64 magnitude), the CRT composition + centring + float conversion of
decode (`DeviceContext.crt_compose`, correctly rounded like Python's
float(int)), and every transform and element-wise product on the way
(`to_ntt`, `hada_mult`, `ele_add/sub`, automorphisms of the secret).

`ClientMixin` is mixed into `CkksContext`, so the context offers the
reference's full API (`keygen`, `make_relin_key`, `make_rotation_key`,
`make_conjugation_key`, `make_switching_key`, `encode`, `decode`, `encrypt`,
`decrypt`, `decrypt_decode`).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import torch

from . import kernels
from .errors import ParameterError
from .rns import crt_compose

SIGMA = 3.2          # ref ckks.py:23
NOISE_BOUND = 19     # ~6 sigma truncation (ref ckks.py:24)


class ClientMixin:
    """Needs: self.params, self.rng, self.ext_basis, self.to_ntt, self.to_coeff."""

    # -- sampling (ref ckks.py:87-109) -------------------------------------------
    def _sample_gaussian(self):
        e = np.rint(self.rng.normal(0.0, SIGMA, self.params.n)).astype(np.int64)
        return np.clip(e, -NOISE_BOUND, NOISE_BOUND)

    def _sample_ternary(self, hamming=None):
        n = self.params.n
        s = np.zeros(n, dtype=np.int64)
        if hamming is None:
            s[:] = self.rng.integers(-1, 2, n)
        else:
            pos = self.rng.choice(n, size=hamming, replace=False)
            s[pos] = self.rng.choice([-1, 1], size=hamming)
        return s

    def _sample_uniform(self, basis):
        from .rns import NTT, RnsPolynomial
        rows = np.empty((len(basis), self.params.n), dtype=np.uint32)
        for i, q in enumerate(basis):
            rows[i] = self.rng.integers(0, q, self.params.n, dtype=np.uint64)
        return RnsPolynomial(rows=rows, basis=tuple(basis), domain=NTT)

    def _device_rows(self, coeffs, basis):
        """Signed coefficients (int64 or float64 host array) -> COEFF-domain
        residue rows over `basis`, decomposed on the device (rns.py:77-90;
        float64 is rounded half to even first, as np.rint)."""
        from .rns import COEFF, RnsPolynomial
        t = torch.from_numpy(np.ascontiguousarray(coeffs)).to(self.dev.device)
        return RnsPolynomial(rows=self.dev.crt_decompose(t, tuple(basis)), basis=tuple(basis),
                             domain=COEFF)

    def _encode_signed(self, vals, basis):
        """Small signed integers (ternary / Gaussian samples) -> NTT-domain
        residue rows (ref ckks.py:100-109: crt_decompose then to_ntt)."""
        vals = np.asarray(vals)
        if vals.dtype.kind not in "iu":
            raise ParameterError("_encode_signed takes an integer array")
        return self.to_ntt(self._device_rows(vals.astype(np.int64), basis)).to_host()

    # -- keys (ref ckks.py:113-170) -------------------------------------------------
    def keygen(self):
        """Secret key (ternary, over the extended basis) and public key."""
        from .ckks import SecretKey
        s = self._sample_ternary(self.params.h)
        sk = SecretKey(s=self._encode_signed(s, self.ext_basis))
        return sk, self._make_encryption_key(sk)

    def _make_encryption_key(self, sk):
        from .ckks import PublicKey
        basis = tuple(self.params.q_basis())
        a = self._sample_uniform(basis)
        e = self._encode_signed(self._sample_gaussian(), basis)
        b = kernels.ele_sub(e, kernels.hada_mult(a, sk.s.restrict(basis)))
        return PublicKey(b=b, a=a)

    def make_switching_key(self, sk, target_s):
        """dnum pairs (b_j, a_j) over the extended basis; b_j = e - a_j s + P
        target_s on slice j's chain primes (ref ckks.py:126-151)."""
        from .ckks import SwitchingKey
        p = self.params
        big_p = p.special_modulus()
        ext = tuple(self.ext_basis)
        target = target_s.host_rows()
        pairs = []
        for j in range(p.dnum):
            a = self._sample_uniform(ext)
            e = self._encode_signed(self._sample_gaussian(), ext)
            b = kernels.ele_sub(e, kernels.hada_mult(a, sk.s))
            rows = b.host_rows().copy()
            for i in range(j * p.alpha, (j + 1) * p.alpha):
                q = np.uint64(ext[i])
                f = np.uint64(big_p % ext[i])
                rows[i] = ((rows[i].astype(np.uint64) + target[i].astype(np.uint64) * f % q)
                           % q).astype(np.uint32)
            pairs.append((b.with_rows(rows), a))
        return SwitchingKey(pairs=tuple(pairs))

    def make_relin_key(self, sk):
        return self.make_switching_key(sk, kernels.hada_mult(sk.s, sk.s))

    def make_rotation_key(self, sk, r):
        return self.make_switching_key(sk, kernels.forbenius_map(sk.s, r))

    def make_conjugation_key(self, sk):
        return self.make_switching_key(sk, kernels.conjugate(sk.s))

    # -- encoding (ref ckks.py:174-214) ----------------------------------------------
    def _rot_index(self):
        cached = getattr(self, "_rot_idx", None)
        if cached is not None:
            return cached
        n = self.params.n
        two_n = 2 * n
        g = np.empty(n // 2, dtype=np.int64)   # 5^j mod 2n
        acc = 1
        for j in range(n // 2):
            g[j] = acc
            acc = acc * kernels.GALOIS_GEN % two_n
        self._rot_idx = ((g - 1) // 2, (two_n - g - 1) // 2)
        return self._rot_idx

    def encode(self, values, level=None, scale=None):
        """Up to n/2 complex slots -> scaled integer polynomial (canonical
        embedding by FFT, rounded, CRT-decomposed, NTT on the device)."""
        from .ckks import Plaintext
        p = self.params
        level = p.l_max if level is None else level
        scale = p.default_scale if scale is None else scale
        n = p.n
        values = np.asarray(values)
        if values.size > n // 2:
            raise ParameterError(f"too many slots: {values.size} > {n // 2}")
        z = np.zeros(n // 2, dtype=np.complex128)
        z[:values.size] = values
        idx, cidx = self._rot_index()
        evals = np.zeros(n, dtype=np.complex128)
        evals[idx] = z * float(scale)
        evals[cidx] = np.conj(z) * float(scale)
        zeta = np.exp(1j * np.pi / n)
        coeffs = np.real(np.fft.fft(evals) / n * zeta ** (-np.arange(n)))
        # ref: ints = [int(c) for c in np.rint(coeffs)] -> crt_decompose; the
        # device rounds half to even and reduces every magnitude exactly
        if not np.all(np.isfinite(coeffs)):
            raise (ValueError if np.isnan(coeffs).any() else OverflowError)(
                "cannot convert float NaN/infinity to integer")
        poly = self.to_ntt(self._device_rows(coeffs, p.q_basis(level))).to_host()
        return Plaintext(poly=poly, scale=Fraction(scale), level=level)

    def decode(self, pt):
        """Slot values of a plaintext (ref ckks.py:200-213): INTT, CRT
        composition, centring and float conversion on the device, then the
        inverse canonical embedding (host float64 FFT)."""
        poly = self.to_coeff(pt.poly).to_device(self.dev.device)
        vals = self.dev.crt_compose(poly.rows, poly.basis).cpu().numpy()
        if not np.all(np.isfinite(vals)):   # Python's float(int) raises past the double range
            raise OverflowError("int too large to convert to float")
        return self._decode_floats(vals, pt.scale)

    def _decode_floats(self, vals, scale):
        n = self.params.n
        zeta = np.exp(1j * np.pi / n)
        evals = n * np.fft.ifft(vals * zeta ** np.arange(n))
        return evals[self._rot_index()[0]] / float(scale)

    def _decode_ints(self, coeffs, scale):
        """Reference form (ckks.py:203-213) over Python ints (host helper)."""
        return self._decode_floats(np.array([float(c) for c in coeffs]), scale)

    @staticmethod
    def _centered(poly):
        """Coefficients in (-Q/2, Q/2] of a coefficient-domain polynomial."""
        big_q = 1
        for q in poly.basis:
            big_q *= q
        half = big_q // 2
        return [c - big_q if c > half else c for c in crt_compose(poly)]

    # -- encryption (ref ckks.py:218-239) ----------------------------------------------
    def encrypt(self, pk, pt):
        from .ckks import Ciphertext
        basis = pt.poly.basis
        v = self._encode_signed(self._sample_ternary(), basis)
        e0 = self._encode_signed(self._sample_gaussian(), basis)
        e1 = self._encode_signed(self._sample_gaussian(), basis)
        b = kernels.ele_add(kernels.ele_add(kernels.hada_mult(v, pk.b.restrict(basis)), e0),
                            pt.poly)
        a = kernels.ele_add(kernels.hada_mult(v, pk.a.restrict(basis)), e1)
        return Ciphertext(b=b, a=a, scale=pt.scale, level=pt.level)

    def decrypt(self, sk, ct):
        from .ckks import Plaintext
        m = kernels.ele_add(ct.b, kernels.hada_mult(ct.a, sk.s.restrict(ct.b.basis)))
        return Plaintext(poly=m, scale=ct.scale, level=ct.level)

    def decrypt_decode(self, sk, ct):
        return self.decode(self.decrypt(sk, ct))
