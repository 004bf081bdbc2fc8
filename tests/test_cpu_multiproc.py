"""World-size-2 gloo test of the batch-sharded (N>1) path on CPU.

Each rank takes its contiguous member range (paper_2212_14191_b200.shard),
transforms it (the CPU oracle stands in for the device, which this box does
not have), and the shards are all-gathered; the result must equal the
unsharded transform bit for bit -- batch sharding has no collective on the
hot path, so this is exactly the property the multi-GPU bench relies on.
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, q, n, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2212_14191_b200.shard import gather_batch, local_members, shard_range
    rng = np.random.default_rng(99)
    full = O.uniform_rows(rng, [q], (batch, n))          # (1, B, n), same on all ranks
    mine = local_members(full, rank, world)
    lo, hi = shard_range(batch, rank, world)
    assert mine.shape[1] == hi - lo
    local = O.ntt(mine, [q])
    got = gather_batch(torch.from_numpy(local.view(np.int32)), axis=1)
    if rank == 0:
        np.save(out_path, got.numpy().view(np.uint32))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [6, 7])
def test_sharded_equals_unsharded(tmp_path, batch):
    import torch.multiprocessing as mp
    from oracle import oracle as O
    from paper_2212_14191_b200.params import generate_primes
    n = 256
    q = generate_primes(n, [30])[0]
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), batch, q, n, out), nprocs=2, join=True)
    rng = np.random.default_rng(99)
    full = O.uniform_rows(rng, [q], (batch, n))
    assert np.array_equal(np.load(out), O.ntt(full, [q]))
