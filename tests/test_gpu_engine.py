"""edgeset.apply semantics on the device (mirrors the reference's
test_engine.py cases with named device UDFs instead of Python callables)."""

import numpy as np
import pytest

from tests.util import arrays

pytestmark = pytest.mark.gpu

LBS = ["VERTEX_BASED", "CM", "WM", "STRICT", "EDGE_ONLY", "ETWC", "TWC"]


@pytest.fixture(scope="module")
def gg():
    import paper_2012_07990_b200 as gg
    return gg


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def graph(gg, golden_small, name):
    V, s, d, w = arrays(golden_small["graphs"][name])
    return gg.Graph.from_coo(V, s, d, w, symmetric=golden_small["graphs"][name]["symmetric"])


def bfs_round(gg, torch, g, start, schedule=None, runtime=None):
    rt = runtime or gg.Runtime(gg.ExecConfig(), g)
    parent = torch.full((g.num_vertices,), -1, dtype=torch.int32, device="cuda")
    for v in start:
        parent[v] = v
    fr = rt.frontiers.new_frontier(g.num_vertices, start)
    udf = gg.udfs.BfsParent(parent)
    out = gg.edgeset_apply(g, fr, udf, to_filter=udf.filter, schedule=schedule, runtime=rt)
    return out, rt, parent


def test_single_round_on_path(gg, torch, golden_small):
    g = graph(gg, golden_small, "path4")
    out, _, parent = bfs_round(gg, torch, g, [0])
    assert out.members() == [1]
    assert int(parent[1]) == 0


def test_empty_input(gg, torch, golden_small):
    g = graph(gg, golden_small, "path4")
    out, rt, _ = bfs_round(gg, torch, g, [])
    assert out.size == 0


@pytest.mark.parametrize("direction", ["PUSH", "PULL"])
def test_all_strategies_same_counts(gg, torch, direction):
    from oracle import gen
    V, s, d = gen.rmat(9, 8, seed=18)
    g = gg.Graph.from_coo(V, s, d)
    active = list(range(0, V, 3))
    ref = None
    for lb in LBS:
        counts = torch.zeros(V, dtype=torch.int64, device="cuda")
        rt = gg.Runtime(gg.ExecConfig(), g)
        fr = rt.frontiers.new_frontier(V, active)
        gg.edgeset_apply(g, fr, gg.udfs.CountInDegree(counts), runtime=rt, collect_output=False,
                         schedule=gg.Schedule(direction=direction, load_balance=lb))
        c = counts.cpu().numpy()
        if ref is None:
            # expected: in-degree from the active set
            act = np.zeros(V, bool)
            act[active] = True
            ref = np.bincount(d[act[s]], minlength=V)
        assert np.array_equal(c, ref), lb


@pytest.mark.parametrize("direction", ["PUSH", "PULL"])
def test_all_strategies_agree_on_one_round(gg, torch, golden_small, direction):
    g = graph(gg, golden_small, "rs150")
    start = list(range(0, 150, 7))
    members = None
    for lb in LBS:
        out, _, _ = bfs_round(gg, torch, g, start, gg.Schedule(direction=direction, load_balance=lb))
        m = sorted(out.members())
        if members is None:
            members = m
        assert m == members, lb


@pytest.mark.parametrize("repr_", ["BOOLMAP", "BITMAP"])
def test_pull_membership_reprs(gg, torch, golden_small, repr_):
    g = graph(gg, golden_small, "rs70")
    push, _, _ = bfs_round(gg, torch, g, [0])
    pull, rt, _ = bfs_round(gg, torch, g, [0], gg.Schedule(direction="PULL", pull_frontier_repr=repr_))
    assert sorted(pull.members()) == sorted(push.members())
    assert rt.stats.frontier_conversions >= 1


@pytest.mark.parametrize("creation", ["FUSED", "UNFUSED_BOOLMAP", "UNFUSED_BITMAP"])
@pytest.mark.parametrize("dedup,strategy", [(True, "MONOTONIC_COUNTERS"), (True, "BITMAP"),
                                            (True, "BOOLMAP"), (False, "MONOTONIC_COUNTERS")])
def test_creation_and_dedup_modes(gg, torch, golden_small, creation, dedup, strategy):
    g = graph(gg, golden_small, "rs70")
    s = gg.Schedule(frontier_creation=creation, dedup=dedup, dedup_strategy=strategy)
    out, rt, _ = bfs_round(gg, torch, g, [0], s)
    off = g.out_offsets
    expect = sorted(set(g.out_neighbors[off[0]:off[1]].tolist()))
    assert sorted(set(out.members())) == expect
    if creation == "FUSED":
        assert out.repr == "SPARSE" and rt.stats.creation_passes == 0
    else:
        assert out.repr == ("BOOLMAP" if creation == "UNFUSED_BOOLMAP" else "BITMAP")
        assert rt.stats.creation_passes == 1


def test_dedup_disabled_can_duplicate(gg):
    g = gg.Graph.from_coo(3, [0, 1], [2, 2])
    rt = gg.Runtime(gg.ExecConfig(), g)
    fr = rt.frontiers.new_frontier(3, [0, 1])
    out = gg.edgeset_apply(g, fr, gg.udfs.EnqueueDst(), schedule=gg.Schedule(dedup=False), runtime=rt)
    assert sorted(out.members()) == [2, 2] and out.size == 2
    rt2 = gg.Runtime(gg.ExecConfig(), g)
    fr2 = rt2.frontiers.new_frontier(3, [0, 1])
    out2 = gg.edgeset_apply(g, fr2, gg.udfs.EnqueueDst(), schedule=gg.Schedule(dedup=True), runtime=rt2)
    assert out2.members() == [2]


def test_reuse_keeps_allocations_at_two(gg, torch, golden_small):
    g = graph(gg, golden_small, "path12")
    rt = gg.Runtime(gg.ExecConfig(), g)
    parent = torch.full((12,), -1, dtype=torch.int32, device="cuda")
    parent[0] = 0
    fr = rt.frontiers.new_frontier(12, [0])
    udf = gg.udfs.BfsParent(parent)
    applies = 0
    while fr.size:
        fr = gg.edgeset_apply(g, fr, udf, to_filter=udf.filter, runtime=rt, reuse=True)
        applies += 1
    assert rt.stats.frontier_allocations == 2
    assert rt.stats.reused_frontiers == applies


def test_hybrid_threshold_strictly_greater(gg, torch, golden_small):
    g = graph(gg, golden_small, "rs150")
    hyb = gg.HybridSchedule(threshold=0.1, s1=gg.Schedule(direction="PUSH"),
                            s2=gg.Schedule(direction="PULL", frontier_creation="UNFUSED_BITMAP"))
    for n, want in ((16, ["PULL"]), (15, ["PUSH"])):
        rt = gg.Runtime(gg.ExecConfig(), g)
        parent = torch.full((150,), -1, dtype=torch.int32, device="cuda")
        fr = rt.frontiers.new_frontier(150, list(range(n)))
        udf = gg.udfs.BfsParent(parent)
        gg.hybrid_apply(g, fr, udf, udf, hyb, runtime=rt)
        assert rt.stats.direction_log == want


def test_errors(gg, golden_small):
    g = graph(gg, golden_small, "path4")
    rt = gg.Runtime(gg.ExecConfig(), g)
    fr = rt.frontiers.new_frontier(5, [0])
    with pytest.raises(gg.EngineError, match="universe"):
        gg.edgeset_apply(g, fr, gg.udfs.EnqueueDst(), runtime=rt)
    with pytest.raises(gg.ScheduleError, match="EDGE_ONLY"):
        gg.edgeset_apply(g, None, gg.udfs.EnqueueDst(),
                         schedule=gg.Schedule(blocking=True, load_balance="CM"), collect_output=False)
    with pytest.raises(gg.ScheduleError, match="device UDF"):
        gg.edgeset_apply(g, None, lambda ctx: None, collect_output=False)
    with pytest.raises(gg.ScheduleError, match="unresolved"):
        gg.hybrid_apply(g, None, gg.udfs.EnqueueDst(), gg.udfs.EnqueueDst(),
                        gg.HybridSchedule(threshold="argv[3]"))


@pytest.mark.parametrize("V", [1, 31, 33, 1000, 32768, 32769, 100003])
@pytest.mark.parametrize("target", ["BITMAP", "BOOLMAP"])
def test_dense_sparse_round_trip(gg, V, target):
    """SPARSE -> dense -> SPARSE gives the members ascending and deduplicated
    (frontier.py:186-201, 242-265) at ragged universes: partial last mask,
    several 32768-vertex blocks, empty and full sets."""
    rng = np.random.default_rng(V)
    src = np.arange(V, dtype=np.int64)
    g = gg.Graph.from_coo(V, src, src)
    rt = gg.Runtime(gg.ExecConfig(), g)
    for ids in (np.array([], np.int64), rng.integers(0, V, size=max(1, V // 3)),
                np.arange(V), np.array([V - 1, 0, V - 1]),
                rng.integers(0, V, size=3 * V + 5)):  # multisets longer than max(V, E) + 1
        fr = rt.frontiers.new_frontier(V, ids)
        dense = fr.convert(target)
        want = sorted(set(int(x) for x in ids))
        assert dense.size == len(want)
        assert dense.members() == want
        back = dense.convert("SPARSE")
        assert back.members() == want
        assert back.size == len(want)


def _hub_graph(gg, deg):
    """hub 0 -> 1..deg and every leaf -> 0 (V = deg + 1, E = 2 deg)."""
    leaves = np.arange(1, deg + 1, dtype=np.int64)
    src = np.concatenate([np.zeros(deg, np.int64), leaves])
    dst = np.concatenate([leaves, np.zeros(deg, np.int64)])
    return gg.Graph.from_coo(deg + 1, src, dst)


@pytest.mark.parametrize("lb", ["ETWC", "TWC", "STRICT", "CM", "WM", "VERTEX_BASED"])
def test_push_over_multiset_with_hub(gg, torch, lb):
    """A dedup-off EnqueueDst apply turns 20000 leaves into the hub repeated
    20000 times (a multiset, frontier.py:160-161); every PUSH balancer then
    walks the hub's 20000 arcs once per occurrence (the hub is past the
    16384-arc grid-pass bound, so ETWC/TWC queue it once per occurrence)."""
    deg = 20000
    g = _hub_graph(gg, deg)
    rt = gg.Runtime(gg.ExecConfig(), g)
    leaves = rt.frontiers.new_frontier(deg + 1, list(range(1, deg + 1)))
    hubs = gg.edgeset_apply(g, leaves, gg.udfs.EnqueueDst(), runtime=rt,
                            schedule=gg.Schedule(dedup=False))
    assert hubs.size == deg
    counts = torch.zeros(deg + 1, dtype=torch.int64, device="cuda")
    gg.edgeset_apply(g, hubs, gg.udfs.CountInDegree(counts), runtime=rt, collect_output=False,
                     schedule=gg.Schedule(direction="PUSH", load_balance=lb))
    c = counts.cpu().numpy()
    assert c[0] == 0 and np.all(c[1:] == deg)
    assert rt.stats.edges_traversed == deg + deg * deg


@pytest.mark.parametrize("lb", ["ETWC", "TWC", "VERTEX_BASED"])
def test_multiset_output_larger_than_edge_count(gg, lb):
    """[hub] * 1000 with dedup off emits 1000 * deg entries, more than the
    default max(V, E) + 1 output slots: the queue is sized from the input."""
    deg = 100
    g = _hub_graph(gg, deg)
    rt = gg.Runtime(gg.ExecConfig(), g)
    fr = rt.frontiers.new_frontier(deg + 1, [0] * 1000)
    assert fr.size == 1000
    out = gg.edgeset_apply(g, fr, gg.udfs.EnqueueDst(), runtime=rt,
                           schedule=gg.Schedule(direction="PUSH", load_balance=lb, dedup=False))
    assert out.size == 1000 * deg
    m = np.bincount(np.asarray(out.members()), minlength=deg + 1)
    assert m[0] == 0 and np.all(m[1:] == 1000)
