"""Limb-partitioned key switch / rescale host logic over gloo (world 2 and 3).

The N>1 limb-partitioned mode (paper_2212_14191_b200.limbpart)
exchanges data in exactly two places: one all-gather of every rank's INTT'd
rows per key switch and one broadcast of the top limb per rescale.  Here the
CPU oracle stands in for the device (no GPU on this box): each rank INTTs its
own rows, the real `LimbPartition.all_gather_rows` / `broadcast_top` run over
gloo, each rank computes its own output rows with the oracle's restatement of
the partitioned algorithm, and the gathered result must equal the
unpartitioned key switch / rescale bit for bit -- including ranks that own no
rows (world > rows at low levels) and uneven last shards.
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


def _params():
    from paper_2212_14191_b200.params import CkksParams
    return CkksParams.generate(n=64, l_max=5, k=2, dnum=3, bit_size=28)


def _inputs(p, level):
    import synth
    return synth.ckks_inputs(p.chain.q, p.chain.p, p.n, p.dnum, level, 4242 + level)


def _worker(rank, world, port, level, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2212_14191_b200.limbpart import LimbPartition
    p = _params()
    ins = _inputs(p, level)
    basis = tuple(p.chain.q[:level + 1])
    part = LimbPartition(len(p.chain.q), world)
    lo, n = part.rows(rank, level)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32))  # noqa: E731
    u = lambda x: x.numpy().view(np.uint32)                                # noqa: E731

    # key switch: INTT own rows -> all-gather -> raise to own rows + specials
    d_local = ins["a0"][lo:lo + n]
    y_local = O.intt(d_local, basis[lo:lo + n]) if n else d_local
    y_full = u(part.all_gather_rows(t(y_local), level))
    ksb, ksa = O.key_switch_part(d_local, y_full, basis, lo, ins["rlk"], p.chain.q, p.chain.p,
                                 p.alpha, p.dnum) if n else (d_local, d_local)
    gb = u(part.all_gather_rows(t(ksb), level))
    ga = u(part.all_gather_rows(t(ksa), level))

    # rescale: the owner INTTs the top limb of b and a, broadcast, local rest
    top = torch.zeros((2, p.n), dtype=torch.int32)
    if lo <= level < lo + n:
        q_top = basis[level]
        top = t(np.stack([O.intt(ins[c][level:level + 1], (q_top,))[0] for c in ("b0", "a0")]))
    top = u(part.broadcast_top(top, level))
    keep = max(0, min(lo + n, level) - lo)
    rs = []
    for ci, c in enumerate(("b0", "a0")):
        rows = []
        for i in range(lo, lo + keep):
            q = basis[i]
            x = ins[c][i].astype(np.uint64)
            y = O.ntt((top[ci] % np.uint32(q))[None], (q,))[0].astype(np.uint64)
            rows.append(((x + q - y) % q * pow(basis[level], -1, q) % q).astype(np.uint32))
        loc = np.stack(rows) if rows else np.zeros((0, p.n), np.uint32)
        rs.append(u(part.all_gather_rows(t(loc), level - 1)))
    if rank == 0:
        np.savez(out_path, y=y_full, ksb=gb, ksa=ga, rb=rs[0], ra=rs[1])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,level", [(2, 5), (3, 5), (2, 1), (4, 2)])
def test_limb_partitioned_equals_unpartitioned(tmp_path, world, level):
    """alpha = 2 slices straddle rank boundaries; (4, 2) leaves two ranks empty."""
    import torch.multiprocessing as mp
    from oracle import oracle as O
    out = str(tmp_path / "lp.npz")
    mp.spawn(_worker, args=(world, _free_port(), level, out), nprocs=world, join=True)
    got = np.load(out)
    p = _params()
    ins = _inputs(p, level)
    basis = tuple(p.chain.q[:level + 1])
    assert np.array_equal(got["y"], O.intt(ins["a0"], basis))
    wb, wa = O.key_switch(ins["a0"], basis, ins["rlk"], p.chain.q, p.chain.p, p.alpha, p.dnum)
    assert np.array_equal(got["ksb"], wb) and np.array_equal(got["ksa"], wa)
    rb, ra = O.rescale(ins["b0"], ins["a0"], basis)
    assert np.array_equal(got["rb"], rb) and np.array_equal(got["ra"], ra)


def test_partition_rows():
    from paper_2212_14191_b200.limbpart import LimbPartition
    part = LimbPartition(45, 8)
    assert part.per == 6
    assert [part.rows(g, 44) for g in range(8)] == [(0, 6), (6, 6), (12, 6), (18, 6),
                                                    (24, 6), (30, 6), (36, 6), (42, 3)]
    assert part.rows(7, 40) == (41, 0) and part.rows(6, 40) == (36, 5)
    assert part.owner(44) == 7 and part.owner(41) == 6
    covered = [r for g in range(8) for r in range(*(lambda lo, n: (lo, lo + n))(*part.rows(g, 30)))]
    assert covered == list(range(31))
