"""PageRank on the device vs the reference (golden) and the oracle.

Tolerance (north star): <= 1e-6 max relative error per vertex.
"""

import hashlib
import os

import numpy as np
import pytest

import oracle
from oracle import gen
from tests.conftest import GOLDEN
from tests.util import arrays, max_rel_err, program_with, sched_from

pytestmark = pytest.mark.gpu
PR_TOL = 1e-6

LBS = ["VERTEX_BASED", "CM", "WM", "STRICT", "EDGE_ONLY", "ETWC", "TWC"]


@pytest.fixture(scope="module")
def gg():
    import paper_2012_07990_b200 as gg
    return gg


def _graph(gg, rec):
    V, s, d, w = arrays(rec)
    return gg.Graph.from_coo(V, s, d, w, symmetric=rec["symmetric"])


def test_pagerank_golden_cases(gg, golden_small):
    n = 0
    for case in golden_small["cases"]:
        if case["algo"] != "pagerank":
            continue
        g = _graph(gg, golden_small["graphs"][case["graph"]])
        s = sched_from(case["schedule"])
        r = gg.pagerank(g, program_with(s), max_iters=case["max_iters"],
                        tolerance=case["tolerance"])
        assert max_rel_err(r.values, case["ranks"]) < PR_TOL, (case["graph"], case["schedule"])
        st = case["stats"]
        assert r.stats.rounds == st["rounds"]
        assert r.stats.dispatch_count == st["dispatch_count"]
        assert r.stats.edges_traversed == st["edges_traversed"]
        assert r.stats.direction_log == st["direction_log"]
        n += 1
    assert n >= 20


@pytest.mark.parametrize("lb", LBS)
@pytest.mark.parametrize("direction", ["PUSH", "PULL"])
@pytest.mark.parametrize("fusion", [False, True])
def test_pagerank_every_schedule_matches_oracle(gg, lb, direction, fusion):
    V, s, d = gen.rmat(10, 8, seed=11)
    g = gg.Graph.from_coo(V, s, d)
    want, _ = oracle.pagerank(V, s, d, 25, 0.0)
    sch = gg.Schedule(direction=direction, load_balance=lb)
    r = gg.pagerank(g, program_with(sch, fusion), max_iters=25, tolerance=0.0)
    assert max_rel_err(r.values, want) < PR_TOL
    assert r.stats.rounds == 25
    assert r.stats.dispatch_count == (1 if fusion else 25)


@pytest.mark.parametrize("n", [1, 7, 64, 1000, None])
@pytest.mark.parametrize("fusion", [False, True])
def test_pagerank_edge_blocking_matches_oracle(gg, n, fusion):
    V, s, d = gen.rmat(11, 8, seed=12)
    g = gg.Graph.from_coo(V, s, d)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True, blocking_size=n)
    r = gg.pagerank(g, program_with(sch, fusion), max_iters=20, tolerance=0.0)
    assert max_rel_err(r.values, want) < PR_TOL


@pytest.mark.parametrize("cold_one", ["0", "1"])
@pytest.mark.parametrize("n", [1, 64, 200, 1000])
def test_pagerank_edge_blocking_cold_segments_one_launch(gg, n, cold_one, monkeypatch):
    """GG_PR_COLD_ONE=1 runs every cold segment in one launch (steps dealt in
    segment order); more segments than the launch parameter holds (n=1)
    falls back to one launch per segment."""
    monkeypatch.setenv("GG_PR_COLD_ONE", cold_one)
    V, s, d = gen.rmat(12, 8, seed=13)
    g = gg.Graph.from_coo(V, s, d)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    for fp32 in (False, True):
        sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True, blocking_size=n)
        r = gg.pagerank(g, program_with(sch), max_iters=20, tolerance=0.0, contrib_fp32=fp32)
        assert max_rel_err(r.array, want) < PR_TOL


def test_c1_rmat16_device_generator_and_ranks(gg):
    """C1 (BASELINE configs[0]): the device RMAT generator is bit-identical to
    the fixture's edge list and 20 iterations match the reference's ranks."""
    z = np.load(os.path.join(GOLDEN, "c1_pagerank_rmat16.npz"))
    g = gg.generate_rmat(16, 16, seed=1)
    s, d = g.coo_src, g.coo_dst
    assert hashlib.sha256(s.tobytes() + d.tobytes()).hexdigest() == str(z["edge_sha256"])
    for sch in (None, gg.Schedule(direction="PULL", load_balance="STRICT"),
                gg.Schedule(load_balance="EDGE_ONLY", blocking=True)):
        r = gg.pagerank(g, program_with(sch), max_iters=20, tolerance=0.0)
        assert max_rel_err(r.values, z["ranks"]) < PR_TOL
    r32 = gg.pagerank(g, None, max_iters=20, tolerance=0.0, contrib_fp32=True)
    assert max_rel_err(r32.values, z["ranks"]) < PR_TOL


def test_pagerank_tolerance_stops_early(gg, golden_small):
    rec = golden_small["graphs"]["rs70"]
    g = _graph(gg, rec)
    V, s, d, _ = arrays(rec)
    want, it = oracle.pagerank(V, s, d, 100, 1e-9)
    r = gg.pagerank(g)  # reference defaults: max_iters=100, tolerance=1e-9
    assert r.stats.rounds == it
    assert max_rel_err(r.values, want) < PR_TOL


def test_pagerank_mass_conserved_each_iteration(gg):
    from paper_2012_07990_b200.graphio import Graph
    rng = np.random.default_rng(3)
    s = rng.integers(0, 40, 120)
    d = rng.integers(0, 40, 120)
    g = Graph.from_coo(40, s, d)
    sums = []
    gg.pagerank(g, max_iters=25, tolerance=0.0, on_iteration=lambda r: sums.append(sum(r)))
    assert len(sums) == 25
    assert all(abs(x - 1.0) <= 1e-12 for x in sums)


@pytest.mark.parametrize("blocked", [False, True])
def test_pagerank_observed_equals_plain_run(gg, blocked):
    """pagerank(on_iteration=...) resumes one device iteration per call
    (gg_pagerank_resume): the callback sees every iterate, the stop test runs
    before each body with L1 = inf at first (algos.py:178, :204-205), and the
    result equals the unobserved run -- at linear, not quadratic, cost."""
    V, s, d = gen.rmat(10, 8, seed=9)
    g = gg.Graph.from_coo(V, s, d)
    prog = program_with(gg.Schedule(load_balance="EDGE_ONLY", blocking=blocked))
    plain = gg.pagerank(g, prog, max_iters=60, tolerance=1e-7)
    seen = []
    obs = gg.pagerank(g, prog, max_iters=60, tolerance=1e-7, on_iteration=lambda r: seen.append(list(r)))
    assert len(seen) == plain.stats.rounds == obs.stats.rounds
    assert max_rel_err(obs.values, plain.values) < 1e-12
    assert seen[-1] == obs.values
    want, iters = oracle.pagerank(V, s, d, 60, 1e-7)
    assert iters == len(seen)
    assert max_rel_err(seen[-1], want) < PR_TOL
    # every iterate conserves the mass
    assert all(abs(sum(r) - 1.0) < 1e-9 for r in seen)


def test_pagerank_deterministic_is_bitwise_the_reference(gg, golden_small, monkeypatch):
    """ExecConfig(deterministic=True): per-destination sums in COO order, the
    dangling mass and L1 in vertex order, every operation rounded on its own
    (no FMA) -- the reference's own order for EDGE_ONLY (+ BLOCKED) and PULL
    schedules, so the ranks are the reference's bit for bit
    (runtime.py:26-50, :167; algos.py:163-208)."""
    det = gg.ExecConfig(deterministic=True)
    n = 0
    for case in golden_small["cases"]:
        if case["algo"] != "pagerank":
            continue
        rec = golden_small["graphs"][case["graph"]]
        g = _graph(gg, rec)
        sch = case["schedule"]
        prog = None if sch is None else program_with(sched_from(sch))
        r = gg.pagerank(g, prog, det, max_iters=case["max_iters"], tolerance=case["tolerance"])
        if sch is None or sch["load_balance"] == "EDGE_ONLY" or sch["direction"] == "PULL":
            assert r.values == case["ranks"], (case["graph"], sch)  # bitwise
            n += 1
        else:  # PUSH: the reference sums in its balancer's source order
            assert max_rel_err(r.values, case["ranks"]) < 1e-12
        assert r.stats.rounds == case["stats"]["rounds"]
    assert n >= 16


def test_pagerank_deterministic_c1_bitwise(gg):
    z = np.load(os.path.join(GOLDEN, "c1_pagerank_rmat16.npz"))
    g = gg.generate_rmat(16, 16, seed=1)
    det = gg.ExecConfig(deterministic=True)
    for sch in (None, gg.Schedule(load_balance="EDGE_ONLY", blocking=True),
                gg.Schedule(direction="PULL", load_balance="STRICT")):
        r = gg.pagerank(g, program_with(sch), det, max_iters=20, tolerance=0.0)
        assert np.array_equal(r.array, z["ranks"])  # the reference's ranks, bit for bit


def test_pagerank_errors(gg):
    g = gg.Graph.from_coo(2, [0], [1])
    with pytest.raises(gg.ScheduleError, match="hybrid"):
        gg.pagerank(g, gg.ScheduleProgram({"s0:s1": gg.HybridSchedule()}))
    with pytest.raises(gg.ScheduleError, match="not exposed"):
        gg.pagerank(g, gg.ScheduleProgram({"nope": gg.Schedule()}))


@pytest.mark.parametrize("fp32", [False, True])
def test_pagerank_edge_blocking_dominant_kernel_stats(gg, fp32):
    """The EB run times its hot-segment kernel (RunStats.top_*), which the
    bench's roofline uses: one launch per iteration, hot edges <= E."""
    V, s, d = gen.rmat(14, 16, seed=3)
    g = gg.Graph.from_coo(V, s, d)
    sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True)
    r = gg.pagerank(g, program_with(sch), max_iters=10, tolerance=0.0, contrib_fp32=fp32)
    want, _ = oracle.pagerank(V, s, d, 10, 0.0)
    assert max_rel_err(r.values, want) < PR_TOL
    st = r.stats
    assert st.top_launches == 10 and st.top_ms > 0.0
    assert 0 < st.top_edges <= len(s)
    assert st.edge_launches == 10 and st.edge_ms >= st.top_ms


def test_pagerank_edge_blocking_hub_source_beyond_smem_cache(gg):
    """Sources ranked past the shared-memory hot cache (a star whose centre
    is the only source, plus thousands of low-degree sources) gather from
    global memory inside the hot kernel."""
    rng = np.random.default_rng(5)
    V = 200000
    s = np.concatenate([np.zeros(50000, np.int64), rng.integers(1, V, 400000)])
    d = rng.integers(0, V, len(s))
    g = gg.Graph.from_coo(V, s, d)
    want, _ = oracle.pagerank(V, s, d, 15, 0.0)
    for fp32 in (False, True):
        sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True)
        r = gg.pagerank(g, program_with(sch), max_iters=15, tolerance=0.0, contrib_fp32=fp32)
        assert max_rel_err(r.array, want) < PR_TOL


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("case", ["single", "no_edges", "self_loops", "one_source", "ragged"])
def test_pagerank_edge_blocking_edge_cases(gg, case, fp32):
    """Empty and ragged inputs under EdgeBlocking (single vertex, edgeless,
    self-loops only, one source, V not a multiple of the vector width) vs
    the oracle, also with virtual ranks."""
    from paper_2012_07990_b200.dist import pagerank_virtual
    rng = np.random.default_rng(7)
    if case == "single":
        V, s, d = 1, np.array([0]), np.array([0])
    elif case == "no_edges":
        V, s, d = 7, np.zeros(0, np.int64), np.zeros(0, np.int64)
    elif case == "self_loops":
        V = 9
        s = d = np.arange(V)
    elif case == "one_source":
        V = 1000
        s, d = np.zeros(500, np.int64), rng.integers(0, V, 500)
    else:
        V = 4099
        s, d = rng.integers(0, V, 20000), rng.integers(0, V, 20000)
    g = gg.Graph.from_coo(V, s, d)
    want, _ = oracle.pagerank(V, s, d, 15, 0.0)
    for bs in (None, 3):
        sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True, blocking_size=bs)
        r = gg.pagerank(g, program_with(sch), max_iters=15, tolerance=0.0, contrib_fp32=fp32)
        assert max_rel_err(r.array, want) < PR_TOL, (case, bs)
        if V >= 2:
            ranks, _ = pagerank_virtual(g, 3, program_with(sch), max_iters=15, tolerance=0.0,
                                        contrib_fp32=fp32, fused_allgather=True)
            assert max_rel_err(ranks, want) < PR_TOL, (case, bs, "virtual")


def test_integration_md_reference_side_stub():
    """The ctypes stub INTEGRATION.md tells a schedge maintainer to add runs
    as written (library path substituted) and matches the oracle."""
    import re
    import types
    from tests.conftest import ROOT
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"## 2\. Binding.*?```python\n(.*?)```", text, re.S).group(1)
    code = code.replace("/path/to/paper_2012_07990_b200/libgg.so",
                        os.path.join(ROOT, "paper_2012_07990_b200", "libgg.so"))
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    V, s, d = gen.rmat(10, 8, seed=13)
    g = types.SimpleNamespace(num_vertices=V, coo_src=s.tolist(), coo_dst=d.tolist(), symmetric=False)
    got = ns["pagerank"](g, 20, 0.0, 0.85)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    assert max_rel_err(got, want) < PR_TOL
