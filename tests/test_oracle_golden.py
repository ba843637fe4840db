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


# ---------------------------------------------------------------------------
# the OpenMP full-scale helpers (bench.py parity legs) against the same pins
# ---------------------------------------------------------------------------
def test_oracle_par_helpers_match_reference(golden_small):
    seen = {"bfs": 0, "cc": 0, "bc": 0}
    for case in golden_small["cases"]:
        algo = case["algo"]
        if algo not in seen:
            continue
        V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
        off, nbr, _ = oracle.csr_par(V, s, d)
        ref_off, ref_nbr, _ = _csr(V, s, d)
        assert np.array_equal(off, ref_off)
        for v in range(V):  # same multiset of neighbours per vertex
            assert sorted(nbr[off[v]:off[v + 1]]) == sorted(ref_nbr[off[v]:off[v + 1]])
        if algo == "bfs":
            in_off, in_nbr, _ = oracle.csr_par(V, d, s)
            lv = oracle.bfs_levels_do(V, off, nbr, case["source"], in_off, in_nbr)
            assert lv.tolist() == case["levels"]
            # a legal tree built from the levels passes; a corrupted one fails
            par = np.full(V, -1, np.int32)
            par[case["source"]] = case["source"]
            for u in range(V):
                for e in range(off[u], off[u + 1]):
                    v = nbr[e]
                    if lv[v] == lv[u] + 1 and par[v] == -1:
                        par[v] = u
            assert oracle.bfs_check_tree(V, in_off, in_nbr, case["source"], par, lv) == 0
            reached = np.flatnonzero((lv > 0))
            if len(reached):
                bad = par.copy()
                bad[reached[0]] = reached[0]
                assert oracle.bfs_check_tree(V, in_off, in_nbr, case["source"], bad, lv) >= 1
        elif algo == "cc":
            labels, _ = oracle.cc_par(V, s, d)
            assert labels.tolist() == case["labels"]
        else:
            in_off, in_nbr, _ = oracle.csr_par(V, d, s)
            got = oracle.bc_par(V, off, nbr, case["sources"], in_off, in_nbr)
            assert np.max(np.abs(got - np.asarray(case["scores"]))) < 1e-9
        seen[algo] += 1
    assert min(seen.values()) > 5


def test_oracle_par_helpers_scale16(s16):
    V, s, d = gen.rmat(16, 16, seed=2)
    ss, dd = _sym(V, s, d)
    off, nbr, _ = oracle.csr_par(V, ss, dd)
    src = int(s16["bfs_source"])
    assert np.array_equal(oracle.bfs_levels_do(V, off, nbr, src), s16["bfs_levels"])
    labels, _ = oracle.cc_par(V, ss, dd)
    assert np.array_equal(labels, s16["cc_labels"])
    V, s, d = gen.rmat(13, 8, seed=6)
    ss, dd = _sym(V, s, d)
    off, nbr, _ = oracle.csr_par(V, ss, dd)
    got = oracle.bc_par(V, off, nbr, [int(x) for x in s16["bc_sources"]])
    m = s16["bc_scores"] > 1e-6
    assert max_rel_err(got[m], s16["bc_scores"][m]) < 1e-9
    # PageRank over the unordered CSR-in equals the COO-order restatement
    V, s, d = gen.rmat(14, 8, seed=1)
    in_off, in_nbr, _ = oracle.csr_par(V, d, s)
    pr, _ = oracle.pagerank_par(V, in_off, in_nbr, oracle.offsets_par(V, s), 20, 0.0)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    assert max_rel_err(pr, want) < 1e-12
