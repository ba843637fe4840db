"""Partitioned PageRank through NCCL on one GPU (world size 1 communicator);
the multi-rank data path is exercised by bench.py under torchrun."""

import numpy as np
import pytest

import oracle
from oracle import gen

pytestmark = pytest.mark.gpu


def test_pagerank_dist_single_rank_matches_oracle():
    import torch
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import Comm, pagerank_dist
    V, s, d = gen.rmat(12, 16, seed=5)
    g = gg.Graph.from_coo(V, s, d)
    comm = Comm.create(0, 1, 0)
    ranks, st = pagerank_dist(comm, g, max_iters=20, tolerance=0.0)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    assert np.max(np.abs(ranks - want) / want) < 1e-6
    assert st.rounds == 20
    comm.close()


def _eb_program(gg, blocking_size=None):
    return gg.ScheduleProgram({"s0:s1": gg.Schedule(load_balance="EDGE_ONLY", blocking=True,
                                                    blocking_size=blocking_size)})


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 8])
def test_pagerank_virtual_ranks_match_oracle(nparts, fp32, fused):
    """The partitioned EdgeBlocking run (per-rank layouts over owned
    destinations + exchange) with virtual ranks on one device."""
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import pagerank_virtual
    V, s, d = gen.rmat(12, 16, seed=5)
    g = gg.Graph.from_coo(V, s, d)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    for bs in (None, 300):  # default window (hot segment only) and many cold segments
        ranks, st = pagerank_virtual(g, nparts, _eb_program(gg, bs), max_iters=20, tolerance=0.0,
                                     contrib_fp32=fp32, fused_allgather=fused)
        assert np.max(np.abs(ranks - want) / want) < 1e-6, (nparts, bs)
        assert st.rounds == 20
        assert st.edges_traversed == 20 * len(s)


def test_pagerank_virtual_ranks_tolerance_and_tiny_partitions():
    """More ranks than 32-vertex partition blocks (empty ranks) and the L1
    stop test summed over ranks."""
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import pagerank_virtual
    V, s, d = gen.rmat(6, 4, seed=9)
    g = gg.Graph.from_coo(V, s, d)
    want, it = oracle.pagerank(V, s, d, 100, 1e-9)
    ranks, st = pagerank_virtual(g, 8, _eb_program(gg), max_iters=100, tolerance=1e-9,
                                 fused_allgather=True)
    assert np.max(np.abs(ranks - want) / want) < 1e-6
    assert st.rounds == it


def test_pagerank_dist_ex_single_rank_edgeblocking():
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import Comm, pagerank_dist, prepare_dist
    V, s, d = gen.rmat(12, 16, seed=5)
    g = gg.Graph.from_coo(V, s, d)
    prog = _eb_program(gg)
    assert prepare_dist(1, 0, g, prog) >= 0.0
    comm = Comm.create(0, 1, 0)
    ranks, st = pagerank_dist(comm, g, max_iters=20, tolerance=0.0, program=prog)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    assert np.max(np.abs(ranks - want) / want) < 1e-6
    assert st.rounds == 20
    comm.close()


def _levels_and_tree(gg, g, parents, source, off, nbr):
    V = g.num_vertices
    want = oracle.bfs_levels(V, off, nbr, source).tolist()
    assert gg.bfs_levels(parents) == want
    assert parents[source] == source
    arcs = set(zip(g.coo_src.tolist(), g.coo_dst.tolist()))
    for v, p in enumerate(parents.tolist()):
        if v != source and p != -1:
            assert (p, v) in arcs


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
@pytest.mark.parametrize("theta", [1e-9, 0.05, 0.999999])
def test_bfs_virtual_ranks_levels_and_tree(nparts, theta):
    """Partitioned direction-optimizing BFS with virtual ranks: always-pull,
    hybrid and always-push thresholds; depths bit-exact vs the oracle,
    parents a legal BFS tree."""
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import bfs_virtual
    g = gg.generate_rmat(11, 8, seed=3, symmetrize=True)
    V = g.num_vertices
    off, nbr, _ = oracle.csr(V, g.coo_src, g.coo_dst)
    deg = np.diff(off)
    for source in [int(np.argmax(deg)), int(np.flatnonzero(deg == 1)[0]), int(np.flatnonzero(deg == 0)[0])]:
        parents, st = bfs_virtual(g, nparts, source, theta)
        _levels_and_tree(gg, g, parents, source, off, nbr)
        if theta == 1e-9:
            assert set(st.direction_log) <= {"PULL"}
        if theta == 0.999999:
            assert set(st.direction_log) == {"PUSH"}


@pytest.mark.parametrize("nparts", [2, 4, 8])
@pytest.mark.parametrize("theta", [1e-9, 0.999999])
def test_bfs_virtual_exchange_is_bitmaps(nparts, theta):
    """Per level one rank receives bitmap words only: top-down the owners'
    slices of the peers' discovered bitmaps, then everyone else's words of the
    next frontier -- at most 2 * V/8 bytes, never a V-long int32
    array -- plus the final V*4-byte parent all-gather."""
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import bfs_dist_bounds, bfs_virtual, last_exchange_bytes
    g = gg.generate_rmat(12, 8, seed=5, symmetrize=True)
    V = g.num_vertices
    off, nbr, _ = oracle.csr(V, g.coo_src, g.coo_dst)
    src = int(np.argmax(np.diff(off)))
    parents, st = bfs_virtual(g, nparts, src, theta)
    _levels_and_tree(gg, g, parents, src, off, nbr)
    got = last_exchange_bytes()
    b = [int(x) for x in bfs_dist_bounds(g, nparts)]
    W = (V + 31) // 32
    wb = [(x + 31) // 32 for x in b]
    wb[-1] = W
    own = wb[1] - wb[0]
    parent_bytes = (V - (b[1] - b[0])) * 4
    per_level = 4 * (W - own) + (4 * (nparts - 1) * own if theta > 0.5 else 0)
    assert got == parent_bytes + st.rounds * per_level
    assert per_level <= 2 * W * 4  # bitmap words, not 4 bytes per vertex


def test_bfs_dist_single_rank_matches_oracle():
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import Comm, bfs_dist
    g = gg.generate_rmat(11, 8, seed=3, symmetrize=True)
    V = g.num_vertices
    off, nbr, _ = oracle.csr(V, g.coo_src, g.coo_dst)
    comm = Comm.create(0, 1, 0)
    src = int(np.argmax(np.diff(off)))
    parents, st = bfs_dist(comm, g, src, 0.05)
    _levels_and_tree(gg, g, parents, src, off, nbr)
    comm.close()


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_device_partitions_equal_host_statements(nranks):
    """The device's partitions (EdgeBlocking destinations in renumbered ids,
    BFS vertices) equal the host statements in dist.py."""
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200 import dist
    V, s, d = gen.rmat(12, 16, seed=5)
    g = gg.Graph.from_coo(V, s, d)
    for r in (0, nranks - 1):
        _, bounds, newid = dist.prepare_dist(nranks, r, g, _eb_program(gg), with_partition=True)
        assert bounds.tolist() == dist.eb_partition_bounds(V, s, d, nranks)
        assert np.array_equal(newid, dist.degree_renumbering(V, s))
    gs = gg.generate_rmat(11, 8, seed=3, symmetrize=True)
    off = np.asarray(gs.out_offsets, np.int64)
    assert dist.bfs_dist_bounds(gs, nranks) == dist.bfs_partition_bounds(off, nranks)
