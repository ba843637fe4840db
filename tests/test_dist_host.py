"""Multi-rank host logic of the partitioned PageRank, on CPU with gloo
(world_size 2): the unique-id exchange and the partition rule."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2012_07990_b200.dist import partition_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_bounds_balance_in_edges():
    rng = np.random.default_rng(0)
    deg = rng.zipf(1.8, 5000).clip(max=2000)
    off = np.concatenate(([0], np.cumsum(deg)))
    for P in (1, 2, 4, 8):
        b = partition_bounds(off, P)
        assert b[0] == 0 and b[-1] == 5000 and all(x <= y for x, y in zip(b, b[1:]))
        loads = [off[b[r + 1]] - off[b[r]] for r in range(P)]
        assert sum(loads) == off[-1]
        assert max(loads) - off[-1] / P <= deg.max()


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the same byte exchange Comm.create performs for the NCCL unique id
    uid = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
    dist.broadcast(uid, 0)
    off = np.concatenate(([0], np.cumsum(np.arange(1, 101))))
    b = partition_bounds(off, world)
    t = torch.tensor([off[b[rank + 1]] - off[b[rank]]], dtype=torch.int64)
    dist.all_reduce(t)
    q.put((rank, bytes(uid.numpy()), int(t.item()), b))
    dist.destroy_process_group()


def test_two_rank_id_exchange_and_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == bytes(range(128)) for r in res)
    assert all(r[2] == sum(range(1, 101)) for r in res)
    assert res[0][3] == res[1][3]


def _worker_partitions(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2012_07990_b200.dist import (bfs_partition_bounds, degree_renumbering,
                                            eb_partition_bounds)
    from oracle import gen
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V, s, d = gen.rmat(12, 16, seed=5)  # every rank generates the same graph
    b = eb_partition_bounds(V, s, d, world)
    newid = degree_renumbering(V, s)
    indeg = np.bincount(newid[d], minlength=V)
    mine = int(indeg[b[rank]:b[rank + 1]].sum())  # in-edges this rank keeps
    t = torch.tensor([mine], dtype=torch.int64)
    dist.all_reduce(t)
    allb = [None] * world
    dist.all_gather_object(allb, b)
    off = np.concatenate(([0], np.cumsum(np.bincount(s, minlength=V))))
    bb = bfs_partition_bounds(off, world)
    allbb = [None] * world
    dist.all_gather_object(allbb, bb)
    q.put((rank, int(t.item()), len(s), allb, allbb))
    dist.destroy_process_group()


def test_two_rank_partitions_cover_and_agree():
    """World size 2 over gloo: the EdgeBlocking destination partition and the
    BFS vertex partition are computed identically on every rank, 32-aligned,
    and the ranks' kept in-edges add up to E."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_partitions, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, total, E, allb, allbb in res:
        assert total == E
        assert allb[0] == allb[1] and allbb[0] == allbb[1]
        for b in (allb[0], allbb[0]):
            assert b[0] == 0 and all(x % 32 == 0 for x in b[:-1]) and b == sorted(b)
