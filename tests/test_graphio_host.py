"""Loader error paths (reference test_graphio.py:32-56, 121-141, 154): raised
on the host before any device call, so they run without a GPU; the
successful loads are GPU tests."""

import os

import pytest

from paper_2012_07990_b200.graphio import (GraphLoadError, load_edge_list, load_graph,
                                           load_matrix_market)


def write(tmp_path, text, name="g.txt"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_empty_file_is_error(tmp_path):
    with pytest.raises(GraphLoadError, match="no edges"):
        load_edge_list(write(tmp_path, "# only a comment\n"))


def test_malformed_line_reports_line_number(tmp_path):
    with pytest.raises(GraphLoadError, match=":2:"):
        load_edge_list(write(tmp_path, "0 1\n7\n"))


def test_weight_token_rules(tmp_path):
    with pytest.raises(GraphLoadError, match="missing weight"):
        load_edge_list(write(tmp_path, "0 1\n"), weighted=True)
    with pytest.raises(GraphLoadError, match="negative weight"):
        load_edge_list(write(tmp_path, "0 1 -3\n"), weighted=True)
    with pytest.raises(GraphLoadError, match="non-integer weight"):
        load_edge_list(write(tmp_path, "0 1 x\n"), weighted=True)


def test_matrix_market_errors(tmp_path):
    with pytest.raises(GraphLoadError, match="not a MatrixMarket"):
        load_matrix_market(write(tmp_path, "%%MatrixMarket matrix array real general\n", "a.mtx"))
    with pytest.raises(GraphLoadError, match="square"):
        load_graph(write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n2 3 1\n1 2\n",
                         "b.mtx"))
    with pytest.raises(GraphLoadError, match="1-based"):
        load_graph(write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 2\n",
                         "c.mtx"))
    with pytest.raises(GraphLoadError, match="no weights"):
        load_matrix_market(write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n"
                                           "3 3 1\n1 2\n", "d.mtx"), weighted=True)
    with pytest.raises(GraphLoadError, match="outside declared"):
        load_graph(write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 3\n",
                         "e.mtx"))
    with pytest.raises(GraphLoadError, match="non-negative integers"):
        load_matrix_market(write(tmp_path, "%%MatrixMarket matrix coordinate real general\n"
                                           "3 3 1\n1 2 2.5\n", "f.mtx"), weighted=True)


@pytest.mark.gpu
def test_matrix_market_general_and_symmetric(tmp_path):
    g = load_matrix_market(write(tmp_path, "%%MatrixMarket matrix coordinate integer general\n"
                                           "% comment\n3 3 2\n1 2 5\n3 1 7\n", "g.mtx"),
                           weighted=True)
    assert g.num_vertices == 3
    assert sorted(zip(g.coo_src.tolist(), g.coo_dst.tolist(), g.coo_weights.tolist())) == \
        [(0, 1, 5), (2, 0, 7)]
    g = load_graph(write(tmp_path, "%%MatrixMarket matrix coordinate pattern symmetric\n"
                                   "3 3 2\n2 1\n3 2\n", "s.mtx"))
    assert set(zip(g.coo_src.tolist(), g.coo_dst.tolist())) == {(1, 0), (0, 1), (2, 1), (1, 2)}
    assert g.symmetric
    g = load_graph(write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n"
                                   "3 3 1\n1 2\n", "t.mtx"), symmetrize=True)
    assert g.symmetric and g.num_edges == 2


# ---------------------------------------------------------------------------
# sidecars written by the reference's own save_blocked (oracle/make_golden.py
# sidecars(), blocking.py:189-217): read them, and write byte-identical files
# ---------------------------------------------------------------------------
def _ref_sidecars():
    import glob
    from tests.conftest import GOLDEN
    return sorted(glob.glob(os.path.join(GOLDEN, "ref_sidecar_*.blk")))


def test_reference_sidecars_round_trip_byte_identical(tmp_path):
    import numpy as np
    import oracle
    from oracle import gen
    from paper_2012_07990_b200.blocking import BlockedGraph, load_blocked, save_blocked
    paths = _ref_sidecars()
    assert len(paths) == 3
    V, s, d = gen.rmat(8, 4, seed=11)
    w = gen.weights(len(s), 11)
    for path in paths:
        bg = load_blocked(path)
        n = bg.vertices_per_segment
        weighted = "unweighted" not in path
        # the same layout from the oracle's Alg. 1 on the same COO
        perm, seg = oracle.block_edges(V, d, n)
        assert bg.segment_start == seg.tolist()
        assert bg.edges_src == s[perm].tolist() and bg.edges_dst == d[perm].tolist()
        assert bg.edges_weight == (w[perm].astype(int).tolist() if weighted else None)
        mine = BlockedGraph(V, n, seg.tolist(), s[perm].tolist(), d[perm].tolist(),
                            w[perm].astype(int).tolist() if weighted else None)
        out = tmp_path / "mine.blk"
        save_blocked(mine, str(out))
        assert out.read_bytes() == open(path, "rb").read()
