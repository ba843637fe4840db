"""Multi-GPU PageRank: 1-D destination partition over NCCL.

One process per GPU (torchrun).  ``Comm.create`` exchanges the NCCL unique id
through ``torch.distributed`` (any backend; gloo works for the exchange) and
builds a libgg communicator on this rank's device; ``pagerank_dist`` runs the
partitioned PageRank (csrc/dist.cu) and returns the full rank vector on every
rank.  ``partition_bounds`` is the host statement of the partition rule the
device uses (destination ranges balanced by in-edge count).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .runtime import RunStats


def partition_bounds(in_offsets, nranks):
    """bounds[r] = first v with in_off[v] >= r*E/P (bounds[0]=0, bounds[P]=V)."""
    off = np.asarray(in_offsets, dtype=np.int64)
    V = len(off) - 1
    E = int(off[-1])
    b = [0]
    for r in range(1, nranks):
        target = (E * r) // nranks
        b.append(int(np.searchsorted(off[:V], target, side="left")))
    b.append(V)
    return b


class Comm:
    def __init__(self, handle, rank, world, device):
        self._h = handle
        self.rank, self.world, self.device = rank, world, device

    @classmethod
    def create(cls, rank, world, device, group=None):
        import torch
        import torch.distributed as dist
        uid = (C.c_char * 128)()
        if rank == 0:
            _lib.call("gg_nccl_unique_id", uid)
        if world > 1:
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda(device)
            dist.broadcast(t, 0, group=group)
            uid = (C.c_char * 128)(*t.cpu().numpy().tobytes())
        h = C.c_void_p()
        _lib.call("gg_comm_init", device, world, rank, uid, C.byref(h))
        return cls(h, rank, world, device)

    def close(self):
        if self._h is not None:
            _lib.load().gg_comm_destroy(self._h)
            self._h = None


def _binding(program):
    from .algos import _plan
    from .engine import binding_pod
    plan = _plan(program, "pagerank")
    return binding_pod(plan.apply_schedule)


def pagerank_dist(comm, g, max_iters=100, tolerance=1e-9, damping=0.85, out=None,
                  program=None, contrib_fp32=False):
    """This rank's share of a partitioned PageRank; returns the full rank
    vector (gathered on every rank) and this rank's RunStats.  With an
    EDGE_ONLY + BLOCKED program the EdgeBlocking layout of the owned
    destinations runs; otherwise the PULL gather (no program = PULL)."""
    ranks = out if out is not None else np.empty(g.num_vertices, np.float64)
    st = _lib.new_stats()
    if program is None:
        _lib.call("gg_pagerank_dist", comm._h, g.handle, int(max_iters), float(tolerance),
                  float(damping), _lib.ptr(ranks), C.byref(st))
    else:
        pod = _binding(program)
        _lib.call("gg_pagerank_dist_ex", comm._h, g.handle, C.byref(pod),
                  1 if contrib_fp32 else 0, int(max_iters), float(tolerance), float(damping),
                  _lib.ptr(ranks), C.byref(st))
    return ranks, RunStats.from_pod(st)


def prepare_dist(nranks, rank, g, program, contrib_fp32=False, with_partition=False):
    """Build this rank's layout ahead of the timed runs; returns prep ms (and,
    with_partition, the destination bounds in renumbered ids + the
    renumbering original -> renumbered)."""
    pod = _binding(program)
    ms = C.c_double()
    bounds = np.empty(nranks + 1, np.int64) if with_partition else None
    newid = np.empty(g.num_vertices, np.int32) if with_partition else None
    _lib.call("gg_pagerank_dist_prepare", int(nranks), int(rank), g.handle, C.byref(pod),
              1 if contrib_fp32 else 0, C.byref(ms), _lib.ptr(bounds), _lib.ptr(newid))
    return (ms.value, bounds, newid) if with_partition else ms.value


def degree_renumbering(num_vertices, src):
    """Host statement of the EdgeBlocking renumbering (prblock.cu build_layout
    step 1): vertices by out-degree, descending, ties by id; returns newid."""
    deg = np.bincount(np.asarray(src, np.int64), minlength=num_vertices)
    order = np.argsort(-deg, kind="stable")
    newid = np.empty(num_vertices, np.int64)
    newid[order] = np.arange(num_vertices)
    return newid


def eb_partition_bounds(num_vertices, src, dst, nranks):
    """Host statement of the partitioned EdgeBlocking run's destination
    partition (prblock.cu k_part_bounds): renumbered destinations, balanced
    by in-edges, bounds rounded down to multiples of 32."""
    newid = degree_renumbering(num_vertices, src)
    indeg = np.bincount(newid[np.asarray(dst, np.int64)], minlength=num_vertices)
    off = np.concatenate(([0], np.cumsum(indeg)))
    E = int(off[-1])
    b = [0]
    for r in range(1, nranks):
        target = (E * r) // nranks
        b.append(int(np.searchsorted(off[:num_vertices], target, side="left")) & ~31)
    b.append(num_vertices)
    return b


def bfs_partition_bounds(out_offsets, nranks):
    """Host statement of the partitioned BFS's vertex partition (bfsdist.cu
    k_bfsd_bounds): balanced by out-degree, rounded down to multiples of 32."""
    off = np.asarray(out_offsets, dtype=np.int64)
    V = len(off) - 1
    E = int(off[-1])
    b = [0]
    for r in range(1, nranks):
        target = (E * r) // nranks
        b.append(int(np.searchsorted(off[:V], target, side="left")) & ~31)
    b.append(V)
    return b


def bfs_dist_bounds(g, nranks):
    """The device's BFS vertex partition (gg_bfs_dist_bounds)."""
    b = np.empty(nranks + 1, np.int64)
    _lib.call("gg_bfs_dist_bounds", g.handle, int(nranks), _lib.ptr(b))
    return b.tolist()


def pagerank_virtual(g, nparts, program, max_iters=100, tolerance=1e-9, damping=0.85,
                     out=None, contrib_fp32=False, fused_allgather=False):
    """The partitioned EdgeBlocking run with `nparts` virtual ranks on one
    device -- the test mode of the multi-GPU path: copy exchange, or the
    vertex pass storing into the other ranks' buffers (fused all-gather)."""
    ranks = out if out is not None else np.empty(g.num_vertices, np.float64)
    st = _lib.new_stats()
    pod = _binding(program)
    _lib.call("gg_pagerank_virtual", g.handle, int(nparts), C.byref(pod),
              1 if contrib_fp32 else 0, 1 if fused_allgather else 0, int(max_iters),
              float(tolerance), float(damping), _lib.ptr(ranks), C.byref(st))
    return ranks, RunStats.from_pod(st)


def bfs_dist(comm, g, source, threshold=0.05, out=None):
    """This rank's share of the partitioned direction-optimizing BFS; returns
    the full parent array (gathered on every rank) and this rank's RunStats."""
    if not 0 <= source < g.num_vertices:
        raise ValueError("invalid source %d for graph with %d vertices" % (source, g.num_vertices))
    parents = out if out is not None else np.empty(g.num_vertices, np.int32)
    st = _lib.new_stats()
    _lib.call("gg_bfs_dist", comm._h, g.handle, int(source), float(threshold), _lib.ptr(parents),
              C.byref(st))
    return parents, RunStats.from_pod(st)


def last_exchange_bytes():
    """Bytes one rank received through the exchange in the last bfs_dist /
    bfs_virtual call on this thread (gg_last_exchange_bytes)."""
    b = C.c_uint64(0)
    _lib.call("gg_last_exchange_bytes", C.byref(b))
    return int(b.value)


def bfs_virtual(g, nparts, source, threshold=0.05, out=None):
    """The partitioned BFS with `nparts` virtual ranks on one device (test mode)."""
    if not 0 <= source < g.num_vertices:
        raise ValueError("invalid source %d for graph with %d vertices" % (source, g.num_vertices))
    parents = out if out is not None else np.empty(g.num_vertices, np.int32)
    st = _lib.new_stats()
    _lib.call("gg_bfs_virtual", g.handle, int(nparts), int(source), float(threshold),
              _lib.ptr(parents), C.byref(st))
    return parents, RunStats.from_pod(st)
