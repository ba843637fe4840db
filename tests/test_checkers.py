"""The host checkers behind ``verify`` / ``tune --check`` (the reference's
oracle.py restated in the package) against the reference's own outputs."""

import math

import numpy as np

import oracle
from paper_2012_07990_b200 import checkers
from tests.util import arrays, max_rel_err


class HostGraph:
    def __init__(self, V, s, d, w=None):
        self.num_vertices = V
        self.num_edges = len(s)
        self.coo_src, self.coo_dst = s, d
        self.out_offsets, self.out_neighbors, self.out_weights = oracle.csr(V, s, d, w)
        self.weighted = w is not None


def test_checkers_match_reference_outputs(golden_small):
    seen = set()
    for case in golden_small["cases"]:
        algo = case["algo"]
        if algo not in ("bfs", "sssp", "cc", "bc", "pagerank"):
            continue
        V, s, d, w = arrays(golden_small["graphs"][case["graph"]])
        g = HostGraph(V, s, d, w)
        if algo == "bfs":
            assert checkers.bfs_levels(g, case["source"]) == case["levels"]
        elif algo == "sssp":
            want = [math.inf if x is None else x for x in case["dist"]]
            assert checkers.dijkstra(g, case["source"]) == want
        elif algo == "cc":
            assert checkers.cc_labels(g) == case["labels"]
        elif algo == "bc":
            got = checkers.brandes(g, case["sources"])
            assert np.max(np.abs(np.asarray(got) - case["scores"]), initial=0) < 1e-9
        else:
            got = checkers.pagerank(g, case["max_iters"], case["tolerance"])
            assert max_rel_err(got, case["ranks"]) < 1e-9
        seen.add(algo)
    assert seen == {"bfs", "sssp", "cc", "bc", "pagerank"}


def test_compare_rules():
    assert checkers.compare("bfs", [0, 0, 1], [0, 1, 2])[0]
    assert not checkers.compare("bfs", [0, 0, 0], [0, 1, 2])[0]
    assert checkers.compare("sssp", np.array([0, 2**64 - 1], np.uint64), [0, math.inf])[0]
    assert not checkers.compare("cc", [0, 1], [0, 0])[0]
    assert checkers.compare("pagerank", [0.5, 0.5], [0.5, 0.5 + 1e-9])[0]
    assert not checkers.compare("bc", [1.0], [1.1])[0]


def test_size_guard():
    import pytest
    V = checkers.ORACLE_MAX_VERTICES + 1
    g = HostGraph(V, np.array([0], np.int32), np.array([1], np.int32))
    with pytest.raises(ValueError, match="size guard"):
        checkers.cc_labels(g)
