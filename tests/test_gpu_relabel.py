"""Locality relabelling (csrc/relabel.cu): CC, BC and BFS queried on the
degree-ordered copy of the graph must return the reference's results in the
ORIGINAL ids -- canonical CC labels (each component's minimum original id,
algos.py:304-307), BC scores within 1e-5, BFS levels bit-exact with a legal
parent tree (algos.py:101-156) -- and the run statistics the reference pins
(rounds, edges traversed, direction log) must not change."""

import numpy as np
import pytest

import oracle
from oracle import gen
from tests.util import max_rel_err, program_with

pytestmark = pytest.mark.gpu

LBS = ["VERTEX_BASED", "CM", "WM", "STRICT", "EDGE_ONLY", "ETWC", "TWC"]


@pytest.fixture(scope="module")
def gg():
    import paper_2012_07990_b200 as gg
    return gg


@pytest.fixture(scope="module")
def sym(gg):
    """Symmetric RMAT-12 with a permuted id space (hubs scattered, like the
    Graph500 Kronecker inputs) plus isolated vertices."""
    V, s, d = gen.rmat(12, 8, seed=21)
    perm = np.random.default_rng(3).permutation(V).astype(np.int32)
    s, d = perm[s], perm[d]
    keep = s != d
    s, d = np.concatenate([s[keep], d[keep]]), np.concatenate([d[keep], s[keep]])
    return V, s.astype(np.int32), d.astype(np.int32), gg.Graph.from_coo(V, s, d, symmetric=True)


def _forced(monkeypatch, on):
    monkeypatch.setenv("GG_RELABEL", "1" if on else "0")


@pytest.mark.parametrize("lb", LBS)
def test_cc_relabelled_labels_are_canonical(gg, sym, lb, monkeypatch):
    V, s, d, g = sym
    want, _ = oracle.cc(V, s, d)
    prog = program_with(gg.Schedule(load_balance=lb))
    _forced(monkeypatch, True)
    got = gg.cc_soman(g, prog).array
    assert np.array_equal(got, want)


def test_cc_relabelled_fused_and_blocked(gg, sym, monkeypatch):
    V, s, d, g = sym
    want, _ = oracle.cc(V, s, d)
    _forced(monkeypatch, True)
    for sch, fusion in ((gg.Schedule(load_balance="ETWC"), True),
                        (gg.Schedule(load_balance="EDGE_ONLY", blocking=True), False)):
        assert np.array_equal(gg.cc_soman(g, program_with(sch, fusion)).array, want)


@pytest.mark.parametrize("lb", ["ETWC", "TWC", "VERTEX_BASED"])
def test_bc_relabelled_matches_oracle(gg, sym, lb, monkeypatch):
    V, s, d, g = sym
    off, nbr, _ = oracle.csr(V, s, d)
    deg = np.diff(off)
    sources = [int(np.argmax(deg)), int(np.nonzero(deg)[0][7]), int(np.nonzero(deg)[0][-1])]
    want = oracle.bc(V, off, nbr, sources)
    prog = program_with(gg.Schedule(direction="PUSH", load_balance=lb))
    _forced(monkeypatch, False)
    plain = gg.bc(g, sources, prog)
    _forced(monkeypatch, True)
    got = gg.bc(g, sources, prog)
    big = np.abs(want) > 1e-6
    assert max_rel_err(got.array[big], want[big]) < 1e-5
    assert np.all(np.abs(got.array[~big]) < 1e-9)
    assert got.stats.rounds == plain.stats.rounds  # levels are id-independent


def test_bfs_relabelled_levels_tree_and_stats(gg, sym, monkeypatch):
    V, s, d, g = sym
    off, nbr, _ = oracle.csr(V, s, d)
    src = int(np.argmax(np.diff(off)))
    hy = gg.HybridSchedule(threshold=0.05,
                           s1=gg.Schedule(direction="PUSH", load_balance="ETWC"),
                           s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                          frontier_creation="UNFUSED_BITMAP"))
    prog = gg.ScheduleProgram({"s0:s1": hy})
    _forced(monkeypatch, False)
    plain = gg.bfs(g, src, prog)
    _forced(monkeypatch, True)
    r = gg.bfs(g, src, prog)
    assert gg.bfs_levels(r.values) == oracle.bfs_levels(V, off, nbr, src).tolist()
    arcs = set(zip(s.tolist(), d.tolist()))
    for v, p in enumerate(r.values):
        if v == src:
            assert p == src
        elif p != -1:
            assert (p, v) in arcs
    # arc order inside each adjacency list is kept: the pull early-exit scans
    # and every frontier size are the same, so the statistics are too
    assert r.stats.rounds == plain.stats.rounds
    assert r.stats.edges_traversed == plain.stats.edges_traversed
    assert r.stats.direction_log == plain.stats.direction_log


def test_relabel_prepare_is_cached(gg, sym):
    g = sym[3]
    first = g.prepare_relabel()
    assert first >= 0.0
    assert g.prepare_relabel() == first  # cached on the graph


def test_relabel_invalid_source_still_raises(gg, sym, monkeypatch):
    g = sym[3]
    _forced(monkeypatch, True)
    with pytest.raises(ValueError):
        gg.bfs(g, g.num_vertices, program_with(gg.Schedule(load_balance="ETWC")))
    with pytest.raises(ValueError):
        gg.bc(g, [-1], program_with(gg.Schedule(load_balance="ETWC")))
