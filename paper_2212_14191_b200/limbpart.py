"""Limb-partitioned CKKS evaluation over G GPUs (optional mode).

Batch sharding (`shard.py`) is the throughput mode: whole ciphertexts per
GPU, no collective.  This module is the latency / key-memory mode: every
ciphertext of the batch is split by RNS limb across the G ranks of a process
group -- rank g owns chain rows [g*per, (g+1)*per) (per = ceil((L+1)/G),
fixed at the top level so rows never move; the top rank simply loses rows as
rescale drops limbs).

Which steps need other ranks' rows (ref `ckks.py:265-381`):

* tensor product, automorphism (NTT-domain gather is per limb), hadd/hsub:
  local.
* key switch: ModUp raises every GKS slice to every target prime, so each
  rank needs the coefficient form of ALL chain rows.  Each rank INTTs its
  own rows of d, then ONE all-gather (NCCL over NVLink) assembles
  (level+1, B, N); the rank then raises all slices to its own rows plus the K
  special primes (specials computed redundantly on every rank, which avoids a
  second collective), does the inner product against its key rows and the
  ModDown locally (`tfhe_keyswitch_part`).
* rescale: every rank needs the top limb's coefficient rows (2 rows): the
  owner INTTs them and broadcasts; the rest is local (`tfhe_rescale_part`).

Each op is split into `*_prepare` (local work producing this rank's
contribution to the collective) and `*_finish` (local work after it), so
the same code runs under torch.distributed (`LimbPartitionedEvaluator.hmult`
etc.) and in the single-GPU rank simulation the parity tests use.
Concatenating the ranks' outputs along the limb axis equals the
unpartitioned batched op bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib, kernels
from .device import _ptr, _stream
from .errors import ParameterError


@dataclass(frozen=True)
class LimbPartition:
    """Contiguous split of the chain rows 0..l_max over `world` ranks."""
    n_chain: int
    world: int

    def __post_init__(self):
        if self.world < 1 or self.n_chain < 1:
            raise ParameterError("limb partition needs world >= 1 and at least one limb")

    @property
    def per(self) -> int:
        return -(-self.n_chain // self.world)

    def rows(self, rank: int, level: int) -> tuple[int, int]:
        """(row_lo, n_rows) owned by `rank` at `level` (n_rows may be 0)."""
        lo = min(rank * self.per, level + 1)
        hi = min(lo + self.per, level + 1)
        return lo, hi - lo

    def owner(self, row: int) -> int:
        return row // self.per

    def split(self, x: torch.Tensor, rank: int, level: int, axis: int) -> torch.Tensor:
        """This rank's rows of a full tensor (limb axis `axis`)."""
        lo, n = self.rows(rank, level)
        return x.narrow(axis, lo, n).contiguous()

    def pad(self, local: torch.Tensor) -> torch.Tensor:
        """(n_rows, B, N) -> (per, B, N): equal-size all-gather contributions."""
        if local.shape[0] == self.per:
            return local.contiguous()
        out = torch.zeros((self.per,) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        out[:local.shape[0]] = local
        return out

    def assemble(self, gathered: torch.Tensor, level: int) -> torch.Tensor:
        """(world*per, B, N) all-gather result -> the level+1 chain rows."""
        return gathered[:level + 1]

    # -- the two collectives of the mode (torch.distributed: NCCL on GPUs) ----
    def all_gather_rows(self, local: torch.Tensor, level: int, group=None) -> torch.Tensor:
        """Every rank's (n_rows, B, N) -> the (level+1, B, N) chain rows on all
        ranks: ONE all-gather of equal (per, B, N) contributions."""
        import torch.distributed as dist
        padded = self.pad(local)
        out = torch.empty((self.world * self.per,) + tuple(padded.shape[1:]),
                          dtype=padded.dtype, device=padded.device)
        dist.all_gather_into_tensor(out, padded, group=group)
        return self.assemble(out, level)

    def broadcast_top(self, top: torch.Tensor, level: int, group=None) -> torch.Tensor:
        """The top limb's (2, B, N) coefficient rows from their owner to all."""
        import torch.distributed as dist
        dist.broadcast(top, src=self.owner(level), group=group)
        return top


class LimbPartitionedEvaluator:
    """One rank's share of limb-partitioned HMULT / key switch / rescale /
    HROTATE over a CiphertextBatch split by limb (2, n_rows, B, N)."""

    def __init__(self, ckks_ctx, rank: int, world: int, group=None):
        self.ck = ckks_ctx
        self.dev = ckks_ctx.dev
        self.lib = self.dev.lib
        self.rank, self.world, self.group = int(rank), int(world), group
        self.part = LimbPartition(len(ckks_ctx.params.chain.q), self.world)

    # -- local pieces ---------------------------------------------------------
    def rows(self, level):
        return self.part.rows(self.rank, level)

    def ks_prepare(self, d_local: torch.Tensor, level: int) -> torch.Tensor:
        """INTT of the local rows of d (this rank's all-gather contribution)."""
        lo, n = self.rows(level)
        y = self.dev.empty(n, d_local.shape[1], self.dev.n)
        if n:
            self.dev.ntt(d_local, self.dev.primes[lo:lo + n], inverse=True, out=y)
        return y

    def ks_finish(self, d_local, y_full, level, swk, add=None, add_components=2):
        """Raise all slices to the local rows + specials, inner product, ModDown."""
        lo, n = self.rows(level)
        batch = y_full.shape[1]
        out = self.dev.empty(2, n, batch, self.dev.n)
        if n == 0:
            return out
        ws = self.dev.ckks_workspace(level, batch)
        key = self.ck.device_key(swk)
        _lib.check(self.lib.tfhe_keyswitch_part(
            self.dev.handle, _ptr(d_local), _ptr(y_full), level, batch, _ptr(key),
            self.ck.params.dnum, lo, n, _ptr(out), _ptr(add), add_components if add is not None
            else 0, _ptr(ws), ws.numel(),
            _stream(self.dev.device)), "tfhe_keyswitch_part")
        return out

    def tensor(self, c0_local, c1_local, level):
        lo, n = self.rows(level)
        batch = c0_local.shape[2]
        out = self.dev.empty(3, n, batch, self.dev.n)
        _lib.check(self.lib.tfhe_tensor_product(
            self.dev.handle, _ptr(c0_local), _ptr(c1_local), lo, n, batch, _ptr(out),
            _stream(self.dev.device)), "tfhe_tensor_product")
        return out

    def rescale_prepare(self, ct_local, level):
        """Owner of the top row: INTT of both components' top limb (2, B, N)."""
        lo, n = self.rows(level)
        batch = ct_local.shape[2]
        top = self.dev.empty(2, batch, self.dev.n)
        if lo <= level < lo + n:
            r = level - lo
            self.dev.ntt(ct_local.reshape(2 * n, batch, self.dev.n), [self.dev.primes[level]] * 2,
                         inverse=True, in_rows=[r, n + r], out=top)
        return top

    def rescale_finish(self, ct_local, top, level):
        lo, n = self.rows(level)
        batch = ct_local.shape[2]
        keep = max(0, min(lo + n, level) - lo)
        out = self.dev.empty(2, keep, batch, self.dev.n)
        if keep:
            ws = self.dev.ckks_workspace(level, batch)
            _lib.check(self.lib.tfhe_rescale_part(
                self.dev.handle, _ptr(ct_local), _ptr(top), level, batch, lo, n, _ptr(out),
                _ptr(ws), ws.numel(), _stream(self.dev.device)), "tfhe_rescale_part")
        return out

    def automorphism(self, ct_local, level, galois_t):
        lo, n = self.rows(level)
        if n == 0:
            return ct_local
        rows = list(self.dev.primes[lo:lo + n]) * 2
        x = ct_local.reshape(2 * n, ct_local.shape[2], self.dev.n)
        return self.dev.automorphism(x, galois_t, True, rows).view(ct_local.shape)

    # -- distributed operators ------------------------------------------------
    def key_switch(self, d_local, level, swk, add=None, add_components=2):
        y = self.part.all_gather_rows(self.ks_prepare(d_local, level), level, self.group)
        return self.ks_finish(d_local, y, level, swk, add, add_components)

    def hmult(self, c0_local, c1_local, level, rlk):
        """Relinearised product of the local rows (ckks.py:265-274)."""
        d = self.tensor(c0_local, c1_local, level)
        return self.key_switch(d[2], level, rlk, add=d[:2])

    def rescale(self, ct_local, level):
        if level < 1:
            raise ParameterError("no levels left to rescale")
        top = self.part.broadcast_top(self.rescale_prepare(ct_local, level), level, self.group)
        return self.rescale_finish(ct_local, top, level)

    def hrotate(self, ct_local, level, r, rot_key):
        """b' = phi(b) + ksb(phi(a)), a' = ksa(phi(a)) (ckks.py:276-282)."""
        t = kernels.galois_element(r, self.ck.params.n)
        phi = self.automorphism(ct_local, level, t)
        return self.key_switch(phi[1].contiguous(), level, rot_key, add=phi, add_components=1)


def simulate(ckks_ctx, world: int):
    """The `world` ranks' evaluators on ONE device, with the collectives done
    by concatenation (sequential rank simulation for parity tests)."""
    return [LimbPartitionedEvaluator(ckks_ctx, g, world) for g in range(world)]


def sim_key_switch(evs, d_full, level, swk, add_full=None, add_components=2):
    part = evs[0].part
    locs = [part.split(d_full, e.rank, level, 0) for e in evs]
    y = part.assemble(torch.cat([part.pad(e.ks_prepare(d, level)) for e, d in zip(evs, locs)]),
                      level)
    outs = []
    for e, d in zip(evs, locs):
        add = part.split(add_full, e.rank, level, 1) if add_full is not None else None
        outs.append(e.ks_finish(d, y, level, swk, add, add_components))
    return torch.cat(outs, dim=1)


def sim_hmult(evs, c0_full, c1_full, level, rlk):
    part = evs[0].part
    ds = [e.tensor(part.split(c0_full, e.rank, level, 1), part.split(c1_full, e.rank, level, 1),
                   level) for e in evs]
    d2 = torch.cat([d[2] for d in ds])
    add = torch.cat([d[:2] for d in ds], dim=1)
    return sim_key_switch(evs, d2, level, rlk, add)


def sim_rescale(evs, ct_full, level):
    part = evs[0].part
    locs = [part.split(ct_full, e.rank, level, 1) for e in evs]
    top = evs[part.owner(level)].rescale_prepare(locs[part.owner(level)], level)
    return torch.cat([e.rescale_finish(c, top, level) for e, c in zip(evs, locs)], dim=1)


def sim_hrotate(evs, ct_full, level, r, rot_key):
    part = evs[0].part
    t = kernels.galois_element(r, evs[0].ck.params.n)
    phis = [e.automorphism(part.split(ct_full, e.rank, level, 1), level, t) for e in evs]
    phi = torch.cat(phis, dim=1)
    return sim_key_switch(evs, phi[1].contiguous(), level, rot_key, phi, add_components=1)
