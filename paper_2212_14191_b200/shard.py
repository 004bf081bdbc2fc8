"""Batch sharding across GPUs (one process per GPU, torch.distributed plumbing).

Independent ciphertexts are the unit of work: rank g of G takes
members [g*B/G, (g+1)*B/G) of a level-major (L, B, N) batch and runs the
whole pipeline locally.  Twiddles and switching keys are replicated; there is
no collective on the hot path.  `gather_batch` reassembles results (off the
hot path, for checking / returning to a single host).
"""

from __future__ import annotations


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous member range of `rank` (balanced: sizes differ by at most 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return batch * rank // world, batch * (rank + 1) // world


def local_members(x, rank: int, world: int, axis: int = 1):
    """View of this rank's members of a level-major buffer (axis = batch axis)."""
    lo, hi = shard_range(x.shape[axis], rank, world)
    sl = [slice(None)] * x.ndim
    sl[axis] = slice(lo, hi)
    return x[tuple(sl)]


def gather_batch(local, group=None, axis: int = 1):
    """All-gather the per-rank shards back into the full batch (any backend)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [None] * world
    dist.all_gather_object(sizes, int(local.shape[axis]), group=group)
    parts = []
    for r in range(world):
        shape = list(local.shape)
        shape[axis] = sizes[r]
        parts.append(torch.empty(shape, dtype=local.dtype, device=local.device))
    if len(set(sizes)) == 1:
        dist.all_gather(parts, local.contiguous(), group=group)
    else:
        for r in range(world):
            src = local.contiguous() if r == dist.get_rank(group) else parts[r]
            dist.broadcast(src, src=r, group=group)
            parts[r] = src
    return torch.cat(parts, dim=axis)
