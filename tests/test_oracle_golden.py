"""Pin the CPU oracle (oracle.c) to outputs of the reference itself.

Fixtures in tests/golden/ were produced by oracle/make_golden.py, which runs
the reference package (schedge) in the dev container.
"""

import os

import numpy as np
import pytest

import oracle
from oracle import gen
from tests.util import arrays, max_rel_err

from tests.conftest import GOLDEN


def _csr(V, s, d, w=None):
    return oracle.csr(V, s, d, w)


def test_oracle_bfs_levels_match_reference(golden_small):
    n = 0
    for case in golden_small["cases"]:
        if case["algo"] != "bfs":
            continue
        V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
        off, nbr, _ = _csr(V, s, d)
        assert oracle.bfs_levels(V, off, nbr, case["source"]).tolist() == case["levels"]
        assert oracle.bfs_levels(V, off, nbr, case["source"], parallel=True).tolist() == case["levels"]
        n += 1
    assert n > 100


def test_oracle_pagerank_matches_reference(golden_small):
    for case in golden_small["cases"]:
        if case["algo"] != "pagerank":
            continue
        V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
        ranks, it = oracle.pagerank(V, s, d, case["max_iters"], case["tolerance"])
        assert it == case["stats"]["rounds"]
        assert max_rel_err(ranks, case["ranks"]) < 1e-12
        in_off, in_nbr, _ = _csr(V, d, s)
        out_off, _, _ = _csr(V, s, d)
        pr, it2 = oracle.pagerank_par(V, in_off, in_nbr, out_off, case["max_iters"],
                                      case["tolerance"])
        assert it2 == it and max_rel_err(pr, case["ranks"]) < 1e-12


def test_oracle_sssp_matches_reference(golden_small):
    n = 0
    for case in golden_small["cases"]:
        if case["algo"] != "sssp":
            continue
        V, s, d, w = arrays(golden_small["graphs"][case["graph"]])
        off, nbr, ww = _csr(V, s, d, w)
        dist, rounds = oracle.sssp_delta(V, off, nbr, ww, case["source"], case["schedule"]["delta"])
        want = [oracle.UNREACHED if x is None else x for x in case["dist"]]
        assert dist.tolist() == want
        assert rounds == case["stats"]["rounds"]
        n += 1
    assert n >= 20


def test_oracle_cc_matches_reference(golden_small):
    for case in golden_small["cases"]:
        if case["algo"] != "cc":
            continue
        V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
        labels, _ = oracle.cc(V, s, d)
        assert labels.tolist() == case["labels"]


def test_oracle_bc_matches_reference(golden_small):
    for case in golden_small["cases"]:
        if case["algo"] != "bc":
            continue
        V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
        off, nbr, _ = _csr(V, s, d)
        got = oracle.bc(V, off, nbr, case["sources"])
        assert np.max(np.abs(got - np.asarray(case["scores"]))) < 1e-9


def test_oracle_block_edges_matches_reference(golden_small):
    for case in golden_small["cases"]:
        if case["algo"] != "block_edges":
            continue
        V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
        perm, seg = oracle.block_edges(V, d, case["n"])
        assert seg.tolist() == case["segment_start"]
        assert s[perm].tolist() == case["src"] and d[perm].tolist() == case["dst"]


def test_oracle_rmat12(golden_rmat12):
    g = golden_rmat12
    V, s, d = gen.rmat(12, 16, seed=2)
    ss, dd, _, _ = __import__("paper_2012_07990_b200.graphio", fromlist=["x"]).symmetrize_coo(s, d)
    assert len(ss) == g["sym_arcs"]
    off, nbr, _ = _csr(V, ss, dd)
    assert oracle.bfs_levels(V, off, nbr, g["bfs_source"]).tolist() == g["bfs_levels"]
    labels, _ = oracle.cc(V, ss, dd)
    assert labels.tolist() == g["cc_labels"]
    bcv = oracle.bc(V, off, nbr, g["bc_sources"])
    assert max_rel_err(bcv[np.asarray(g["bc_scores"]) > 0],
                       np.asarray(g["bc_scores"])[np.asarray(g["bc_scores"]) > 0]) < 1e-9
    w = gen.weights(len(s), 4)
    offw, nbrw, ww = _csr(V, s, d, w)
    dist, _ = oracle.sssp_delta(V, offw, nbrw, ww, 0, g["sssp_delta"])
    assert dist.tolist() == [oracle.UNREACHED if x is None else x for x in g["sssp_dist"]]


def test_oracle_c1_pagerank_against_reference():
    z = np.load(os.path.join(GOLDEN, "c1_pagerank_rmat16.npz"))
    V, s, d = gen.rmat(16, 16, seed=1)
    import hashlib
    assert hashlib.sha256(s.tobytes() + d.tobytes()).hexdigest() == str(z["edge_sha256"])
    ranks, it = oracle.pagerank(V, s, d, 20, 0.0)
    assert it == 20
    assert max_rel_err(ranks, z["ranks"]) < 1e-12


# ---------------------------------------------------------------------------
# scale-16 pins (tests/golden/scale16.npz, oracle/make_golden.py scale16_cases)
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def s16():
    return np.load(os.path.join(GOLDEN, "scale16.npz"))


def _sym(V, s, d):
    from paper_2012_07990_b200.graphio import symmetrize_coo
    ss, dd, _, _ = symmetrize_coo(s, d)
    return ss.astype(np.int32), dd.astype(np.int32)


def test_oracle_scale16_bfs_cc(s16):
    V, s, d = gen.rmat(16, 16, seed=2)
    ss, dd = _sym(V, s, d)
    assert len(ss) == int(s16["sym_arcs"])
    off, nbr, _ = _csr(V, ss, dd)
    src = int(s16["bfs_source"])
    assert np.array_equal(oracle.bfs_levels(V, off, nbr, src, parallel=True), s16["bfs_levels"])
    labels, _ = oracle.cc(V, ss, dd)
    assert np.array_equal(labels, s16["cc_labels"])


def test_oracle_scale16_sssp_grid(s16):
    V, s, d = gen.grid(128)
    w = gen.weights(len(s), 4)
    off, nbr, ww = _csr(V, s, d, w)
    for delta in (64, 1024):
        got, _ = oracle.sssp_delta(V, off, nbr, ww, 0, delta)
        want = s16["sssp_d%d" % delta]
        got = np.where(got == np.uint64(2**64 - 1), -1, got.astype(np.int64))
        assert np.array_equal(got, want)


def test_oracle_scale16_bc(s16):
    V, s, d = gen.rmat(13, 8, seed=6)
    ss, dd = _sym(V, s, d)
    assert len(ss) == int(s16["bc_arcs"])
    off, nbr, _ = _csr(V, ss, dd)
    got = oracle.bc(V, off, nbr, [int(x) for x in s16["bc_sources"]])
    assert max_rel_err(got[s16["bc_scores"] > 1e-6], s16["bc_scores"][s16["bc_scores"] > 1e-6]) < 1e-9
