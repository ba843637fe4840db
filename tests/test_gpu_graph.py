"""Device graph construction vs the reference layout (graphio.from_coo)."""

import os

import numpy as np
import pytest

import oracle
from oracle import gen
from tests.util import arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gg():
    import paper_2012_07990_b200 as gg
    return gg


def test_csr_views_equal_stable_counting_sort(gg, golden_small):
    for name, rec in golden_small["graphs"].items():
        V, s, d, w = arrays(rec)
        g = gg.Graph.from_coo(V, s, d, w)
        off, nbr, ww = oracle.csr(V, s, d, w)
        assert g.out_offsets.tolist() == off.tolist(), name
        assert g.out_neighbors.tolist() == nbr.tolist(), name
        ioff, inbr, iww = oracle.csr(V, d, s, w)
        assert g.in_offsets.tolist() == ioff.tolist(), name
        assert g.in_neighbors.tolist() == inbr.tolist(), name
        if w is not None:
            assert g.out_weights.tolist() == ww.tolist()
            assert g.in_weights.tolist() == iww.tolist()


def test_out_of_range_ids_rejected(gg):
    with pytest.raises(ValueError, match="out of range"):
        gg.Graph.from_coo(3, [0, 5], [1, 2])


def test_device_generators_match_host_replicas(gg):
    g = gg.generate_rmat(12, 16, seed=2)
    V, s, d = gen.rmat(12, 16, seed=2)
    assert np.array_equal(g.coo_src, s) and np.array_equal(g.coo_dst, d)
    gw = gg.generate_rmat(10, 4, seed=9, weights=True)
    assert np.array_equal(gw.coo_weights, gen.weights(gw.num_edges, 9))
    gs = gg.generate_rmat(12, 16, seed=2, symmetrize=True)
    from paper_2012_07990_b200.graphio import symmetrize_coo
    ss, dd, _, _ = symmetrize_coo(s, d)
    assert np.array_equal(gs.coo_src, ss) and np.array_equal(gs.coo_dst, dd)
    gr = gg.generate_grid(33)
    Vg, sg, dg = gen.grid(33)
    assert gr.num_vertices == Vg and np.array_equal(gr.coo_src, sg)
    assert np.array_equal(gr.coo_dst, dg)
    assert gr.num_edges == 4 * 33 * 32


def test_sort_by_source_keeps_stable_order(gg):
    g = gg.generate_rmat(10, 8, seed=3, sort_by_source=True)
    V, s, d = gen.rmat(10, 8, seed=3)
    s2, d2, _ = gen.sort_by_source(s, d)
    assert np.array_equal(g.coo_src, s2) and np.array_equal(g.coo_dst, d2)


def test_block_edges_matches_reference(gg, golden_small):
    for case in golden_small["cases"]:
        if case["algo"] != "block_edges":
            continue
        V, s, d, w = arrays(golden_small["graphs"][case["graph"]])
        g = gg.Graph.from_coo(V, s, d, w)
        bg = gg.block_edges(g, case["n"])
        assert bg.segment_start == case["segment_start"]
        assert bg.edges_src == case["src"] and bg.edges_dst == case["dst"]


def test_sidecar_straight_to_device(tmp_path):
    """convert -> sidecar -> install on the device (no Alg. 1 rerun); the
    installed layout equals block_edges' and drives an EDGE_ONLY+BLOCKED run;
    a tampered sidecar is rejected."""
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.blocking import block_edges, load_blocked_to_device, save_blocked
    from paper_2012_07990_b200.engine import binding_pod  # noqa: F401
    g = gg.generate_rmat(10, 8, seed=9, weights=True)
    bg = block_edges(g, 100)
    path = str(tmp_path / "g.blk")
    save_blocked(bg, path)
    g2 = gg.Graph.from_coo(g.num_vertices, g.coo_src, g.coo_dst, g.coo_weights)
    load_blocked_to_device(path, g2)
    bg2 = block_edges(g2, 100)  # cached: the installed layout
    assert bg2.segment_start == bg.segment_start and bg2.edges_src == bg.edges_src
    assert bg2.edges_dst == bg.edges_dst and bg2.edges_weight == bg.edges_weight
    g3 = load_blocked_to_device(path)  # graph from the sidecar itself
    assert g3.num_edges == g.num_edges
    prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(load_balance="EDGE_ONLY", blocking=True,
                                                    blocking_size=100)})
    want = gg.bfs_levels(gg.bfs(g, 0, prog).values)
    assert gg.bfs_levels(gg.bfs(g3, 0, prog).values) == want
    # tamper: move one edge into the wrong segment
    import numpy as np
    bad = np.fromfile(path, dtype=np.uint8).copy()
    off = 8 + 48 + 8 * len(bg.segment_start) + 8 * g.num_edges  # start of dst array
    bad[off:off + 8] = np.frombuffer(np.int64(g.num_vertices - 1).tobytes(), np.uint8)
    bad.tofile(str(tmp_path / "bad.blk"))
    g4 = gg.Graph.from_coo(g.num_vertices, g.coo_src, g.coo_dst, g.coo_weights)
    with pytest.raises(ValueError):
        load_blocked_to_device(str(tmp_path / "bad.blk"), g4)


@pytest.mark.gpu
def test_reference_written_sidecar_to_device():
    """A sidecar written by the reference's save_blocked (tests/golden) is
    installed on the device as the graph's Alg. 1 layout; the device's own
    Alg. 1 on the same COO writes a byte-identical sidecar, and EdgeBlocking
    PageRank on the installed layout matches the oracle."""
    import glob
    import tempfile
    import oracle
    from oracle import gen
    from tests.conftest import GOLDEN
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.blocking import block_edges, load_blocked_to_device, save_blocked
    V, s, d = gen.rmat(8, 4, seed=11)
    w = gen.weights(len(s), 11)
    want_pr, _ = oracle.pagerank(V, s, d, 15, 0.0)
    paths = sorted(glob.glob(os.path.join(GOLDEN, "ref_sidecar_*.blk")))
    assert len(paths) == 3
    for path in paths:
        weighted = "unweighted" not in path
        g = load_blocked_to_device(path)            # graph built from the sidecar's edges
        fresh = gg.Graph.from_coo(V, s, d, w if weighted else None)
        n = int(path.rsplit("_n", 1)[1].split(".")[0])
        with tempfile.TemporaryDirectory() as tmp:
            out = os.path.join(tmp, "dev.blk")
            save_blocked(block_edges(fresh, n), out)
            assert open(out, "rb").read() == open(path, "rb").read()
        g2 = gg.Graph.from_coo(V, s, d, w if weighted else None)
        load_blocked_to_device(path, g2)            # installed into an existing graph
        import torch
        for graph in (g, g2):  # Alg. 2 over the installed layout (no Alg. 1 rerun)
            counts = torch.zeros(V, dtype=torch.int64, device="cuda")
            assert gg.apply_blocked((graph, n), gg.udfs.CountInDegree(counts)) == len(s)
            assert np.array_equal(counts.cpu().numpy(), np.bincount(d, minlength=V))
            prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(load_balance="EDGE_ONLY",
                                                            blocking=True, blocking_size=n)})
            r = gg.pagerank(graph, prog, max_iters=15, tolerance=0.0).array
            assert np.max(np.abs(r - want_pr) / want_pr) < 1e-12


def test_uint32_weights_uploaded_as_is(gg):
    """uint32 weights skip the host range passes (graphio.from_coo fast path):
    same device graph and SSSP distances as the checked int64 path; a length
    mismatch is still rejected."""
    import numpy as np
    from paper_2012_07990_b200.graphio import GraphLoadError
    rng = np.random.default_rng(3)
    V = 500
    s = rng.integers(0, V, 4000).astype(np.int32)
    d = rng.integers(0, V, 4000).astype(np.int32)
    w = rng.integers(0, 2**20, 4000).astype(np.uint32)
    g1 = gg.Graph.from_coo(V, s, d, w)
    g2 = gg.Graph.from_coo(V, s, d, w.astype(np.int64))
    assert np.array_equal(np.asarray(g1.out_weights), np.asarray(g2.out_weights))
    r1 = gg.sssp_delta(g1, 0)
    r2 = gg.sssp_delta(g2, 0)
    assert np.array_equal(r1.array, r2.array)
    with pytest.raises(GraphLoadError):
        gg.Graph.from_coo(V, s, d, w[:-1])
