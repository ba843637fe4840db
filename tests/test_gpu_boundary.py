"""The reference's operator-level surface on the device: BucketQueue
(priority.py:17-118, mirrors tests/test_priority.py), every algorithm UDF
through edgeset_apply (SSSP relax, CC hook, BC forward/backward), apply_blocked
(blocking.py:116-186), fused_loop dispatch accounting (engine.py:639-662) and
concurrent queries on one shared Graph (test_algos.py:362-379)."""

import heapq
import threading

import numpy as np
import pytest

import oracle
from oracle import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gg():
    import paper_2012_07990_b200 as gg
    return gg


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# BucketQueue (tests/test_priority.py of the reference, case by case)
# ---------------------------------------------------------------------------
def test_bq_update_into_current_bucket(gg):
    q = gg.BucketQueue(10, delta=10)
    assert q.update_priority_min(3, 7) is True
    assert q.priorities[3] == 7
    assert 3 in q.current.members()
    assert q.far.size == 0


def test_bq_no_improvement_no_enqueue(gg):
    q = gg.BucketQueue(10, delta=10)
    q.update_priority_min(3, 7)
    q.take_current()
    assert q.update_priority_min(3, 9) is False
    assert q.priorities[3] == 7
    assert q.current.size == 0


def test_bq_update_into_far_bucket(gg):
    q = gg.BucketQueue(10, delta=10)
    assert q.update_priority_min(4, 23) is True
    assert 4 in q.far.members()
    assert q.current.size == 0


def test_bq_advance_moves_minimum_bucket(gg):
    q = gg.BucketQueue(10, delta=10)
    for v, p in ((1, 12), (2, 23), (3, 15)):
        q.update_priority_min(v, p)
    out = q.advance()
    assert q.current_bucket_index == 1
    assert sorted(out.members()) == [1, 3]
    assert q.far.members() == [2]


def test_bq_advance_when_empty_is_done(gg):
    q = gg.BucketQueue(4, delta=5)
    assert q.advance() is None
    assert q.done()


def test_bq_advance_requires_empty_current(gg):
    q = gg.BucketQueue(4, delta=5)
    q.update_priority_min(1, 2)
    with pytest.raises(gg.EngineError, match="non-empty"):
        q.advance()


def test_bq_stale_far_entries_are_filtered(gg):
    q = gg.BucketQueue(10, delta=10)
    q.update_priority_min(5, 25)
    q.update_priority_min(5, 3)
    assert 5 in q.current.members()
    q.take_current()
    assert q.advance() is None
    assert q.done()


def test_bq_seed_and_recycle(gg):
    q = gg.BucketQueue(6, delta=4)
    q.seed(2, priority=0)
    cur = q.take_current()
    assert cur.members() == [2]
    q.recycle(cur)
    q.update_priority_min(3, 1)
    assert q.current.members() == [3]


def test_bq_within_round_dedup_but_rounds_can_repeat(gg):
    q = gg.BucketQueue(8, delta=100)
    q.update_priority_min(4, 50)
    q.update_priority_min(4, 40)
    assert q.current.members() == [4]
    q.take_current()
    q.update_priority_min(4, 30)
    assert q.current.members() == [4]


def test_bq_negative_candidate_rejected(gg):
    q = gg.BucketQueue(4, delta=2)
    with pytest.raises(ValueError, match="non-negative"):
        q.update_priority_min(1, -1)
    with pytest.raises(ValueError, match="delta"):
        gg.BucketQueue(4, delta=0)


def _dijkstra(V, s, d, w, source):
    adj = [[] for _ in range(V)]
    for a, b, c in zip(s.tolist(), d.tolist(), w.tolist()):
        adj[a].append((b, c))
    dist = [None] * V
    dist[source] = 0
    heap = [(0, source)]
    while heap:
        du, u = heapq.heappop(heap)
        if du > dist[u]:
            continue
        for v, c in adj[u]:
            if dist[v] is None or du + c < dist[v]:
                dist[v] = du + c
                heapq.heappush(heap, (dist[v], v))
    return [gg_unreached() if x is None else x for x in dist]


def gg_unreached():
    return 2**64 - 1


def _relax_loop(gg, g, source, delta, lb, fusion):
    """algos.sssp_delta's body (algos.py:236-244) written against the
    operator API: BucketQueue + edgeset_apply(SsspRelax) + fused_loop."""
    rt = gg.Runtime(gg.ExecConfig(), g)
    q = gg.BucketQueue(g.num_vertices, delta)
    q.seed(source, 0)
    relax = gg.udfs.SsspRelax(q)
    sch = gg.Schedule(direction="PUSH", load_balance=lb)

    def body():
        if q.current.size == 0:
            q.advance()
            return
        cur = q.take_current()
        gg.edgeset_apply(g, cur, relax, schedule=sch, runtime=rt, collect_output=False)
        q.recycle(cur)

    st = gg.fused_loop(body, q.done, fusion=fusion, runtime=rt)
    return q.priorities, st


@pytest.mark.parametrize("delta", [1, 3, 16, 10**9])
@pytest.mark.parametrize("lb", ["ETWC", "TWC", "WM", "EDGE_ONLY"])
def test_custom_delta_stepping_loop_matches_dijkstra_and_driver(gg, delta, lb):
    V, s, d = gen.rmat(8, 6, seed=delta % 7)
    w = gen.weights(len(s), 9) % 30
    g = gg.Graph.from_coo(V, s, d, w)
    dist, st = _relax_loop(gg, g, 0, delta, lb, fusion=False)
    assert dist.tolist() == _dijkstra(V, s, d, w, 0)
    prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(load_balance=lb, delta=delta)})
    drv = gg.sssp_delta(g, 0, prog)
    assert dist.tolist() == drv.array.tolist()
    # one dispatch per relax round, none for advance rounds (the round count
    # itself depends on the relaxation order inside a round, as the
    # reference's threaded runs do)
    assert 1 <= st.dispatch_count <= st.rounds
    assert 1 <= drv.stats.dispatch_count <= drv.stats.rounds


def test_fused_loop_counts_one_dispatch(gg):
    """engine.py:639-662: fused, the whole loop is one dispatch; unfused,
    one per traversal (test_algos.py:65-79)."""
    V, s, d = gen.rmat(8, 6, seed=2)
    w = gen.weights(len(s), 3) % 50 + 1
    g = gg.Graph.from_coo(V, s, d, w)
    d0, st0 = _relax_loop(gg, g, 0, 20, "ETWC", fusion=False)
    d1, st1 = _relax_loop(gg, g, 0, 20, "ETWC", fusion=True)
    assert np.array_equal(d0, d1)
    assert st1.dispatch_count == 1
    assert 1 < st0.dispatch_count <= st0.rounds  # one per relax round, none per advance
    # the round count itself depends on which in-bucket improvements parallel
    # relaxation meets first (delta 20 > the lightest arcs), so the fused and
    # the unfused loop need not agree on it -- only on the distances
    assert st1.rounds >= 1
    with pytest.raises(gg.ScheduleError, match="reuses frontier"):
        gg.fused_loop(lambda: None, lambda: True, fusion=True, body_reuses_frontiers=False)


def test_custom_cc_loop_with_hook_udf(gg, torch):
    """cc_soman's loop (algos.py:296-303): hook apply over all vertices +
    pointer jumping (host-side here, as in the reference), to a fixpoint."""
    V, s, d = gen.rmat(10, 4, seed=5)
    ss, dd = np.concatenate([s, d]), np.concatenate([d, s])
    g = gg.Graph.from_coo(V, ss, dd, symmetric=True)
    want, _ = oracle.cc(V, ss, dd)
    for lb in ("ETWC", "TWC", "VERTEX_BASED", "EDGE_ONLY"):
        label = torch.arange(V, dtype=torch.int32, device="cuda")
        changed = torch.zeros(1, dtype=torch.int32, device="cuda")
        rt = gg.Runtime(gg.ExecConfig(), g)
        hook = gg.udfs.CcHook(label, changed)
        while True:
            changed.zero_()
            gg.edgeset_apply(g, None, hook, schedule=gg.Schedule(load_balance=lb), runtime=rt,
                             collect_output=False)
            while True:
                nxt = label[label.long()]
                if torch.equal(nxt, label):
                    break
                label.copy_(nxt)
            if int(changed.item()) == 0:
                break
        got = label.cpu().numpy()
        # canonical min-id labels: the fixpoint root of a component is its minimum id
        assert np.array_equal(got, want), lb
        assert np.array_equal(gg.cc_soman(g, gg.ScheduleProgram(
            {"s0:s1": gg.Schedule(load_balance=lb)})).array, want)


def test_custom_bc_loop_with_forward_backward_udfs(gg, torch):
    """bc's per-source loop (algos.py:341-392) through edgeset_apply with
    the forward / backward UDFs, against the driver and the oracle."""
    V, s, d = gen.rmat(10, 4, seed=6)
    ss, dd = np.concatenate([s, d]), np.concatenate([d, s])
    g = gg.Graph.from_coo(V, ss, dd, symmetric=True)
    off, nbr, _ = oracle.csr(V, ss, dd)
    sources = [int(ss[0]), int(ss[7])]
    want = oracle.bc(V, off, nbr, sources)
    score = np.zeros(V)
    push = gg.Schedule(direction="PUSH", load_balance="ETWC")
    for src in sources:
        rt = gg.Runtime(gg.ExecConfig(), g)
        depth = torch.full((V,), -1, dtype=torch.int32, device="cuda")
        sigma = torch.zeros(V, dtype=torch.float64, device="cuda")
        delta = torch.zeros(V, dtype=torch.float64, device="cuda")
        depth[src] = 0
        sigma[src] = 1.0
        fr = rt.frontiers.new_frontier(V, [src])
        rounds, level = [], 0
        while fr.size:
            rounds.append(fr.members())
            fwd = gg.udfs.BcForward(depth, sigma, level)
            fr = gg.edgeset_apply(g, fr, fwd, to_filter=fwd.filter, schedule=push, runtime=rt,
                                  reuse=True)
            level += 1
        bwd = gg.udfs.BcBackward(depth, sigma, delta)
        for r in range(len(rounds) - 2, -1, -1):
            wave = rt.frontiers.new_frontier(V, rounds[r])
            gg.edgeset_apply(g, wave, bwd, schedule=push, runtime=rt, collect_output=False)
        dl = delta.cpu().numpy()
        dl[src] = 0.0
        score += dl
    score /= 2.0
    assert np.max(np.abs(score - want)) <= 1e-9 * max(1.0, np.max(np.abs(want)))
    drv = gg.bc(g, sources, gg.ScheduleProgram({"s0:s1": push})).array
    assert np.max(np.abs(drv - want)) <= 1e-9 * max(1.0, np.max(np.abs(want)))


# ---------------------------------------------------------------------------
# apply_blocked (blocking.py:116-186)
# ---------------------------------------------------------------------------
def test_apply_blocked_counts_every_edge_once(gg, torch):
    V, s, d = gen.rmat(9, 8, seed=4)
    g = gg.Graph.from_coo(V, s, d)
    for n in (1, 7, 64, V):
        bg = gg.block_edges(g, n)
        counts = torch.zeros(V, dtype=torch.int64, device="cuda")
        rt = gg.Runtime(gg.ExecConfig(), g)
        done = gg.apply_blocked(bg, gg.udfs.CountInDegree(counts), runtime=rt)
        assert done == len(s)
        assert np.array_equal(counts.cpu().numpy(), np.bincount(d, minlength=V))
        assert rt.stats.dispatch_count == 1   # the whole Alg. 2 is one dispatch
        assert gg.apply_blocked((g, n), gg.udfs.CountInDegree(counts)) == len(s)


def test_apply_blocked_pagerank_gather_matches_unblocked(gg, torch):
    V, s, d = gen.rmat(9, 8, seed=9)
    g = gg.Graph.from_coo(V, s, d)
    contrib = torch.rand(V, dtype=torch.float64, device="cuda")
    acc_b = torch.zeros(V, dtype=torch.float64, device="cuda")
    gg.apply_blocked(gg.block_edges(g, 37), gg.udfs.PageRankGather(acc_b, contrib))
    c = contrib.cpu().numpy()
    want = np.zeros(V)
    np.add.at(want, d, c[s])
    assert np.allclose(acc_b.cpu().numpy(), want, rtol=1e-12, atol=0)
    with pytest.raises(gg.EngineError, match="make_context"):
        gg.apply_blocked((g, 37), gg.udfs.PageRankGather(acc_b, contrib),
                         make_context=lambda w: None)


# ---------------------------------------------------------------------------
# concurrent independent queries on one Graph (test_algos.py:362-379)
# ---------------------------------------------------------------------------
def test_concurrent_queries_on_shared_graph(gg):
    V, s, d = gen.rmat(11, 8, seed=12)
    ss, dd = np.concatenate([s, d]), np.concatenate([d, s])
    w = gen.weights(len(ss), 5)
    g = gg.Graph.from_coo(V, ss, dd, w, symmetric=True)
    off, nbr, ww = oracle.csr(V, ss, dd, w)
    want_pr, _ = oracle.pagerank(V, ss, dd, 10, 0.0)
    want_lv = oracle.bfs_levels(V, off, nbr, 3)
    want_cc, _ = oracle.cc(V, ss, dd)
    want_sp, _ = oracle.sssp_delta(V, off, nbr, ww, 3, 64)
    # two PageRank layouts alternate (f64 / f32 contributions): the shared
    # graph's layout cache is replaced while another thread still runs on it
    jobs = {
        "pr64": lambda: gg.pagerank(g, gg.ScheduleProgram({"s0:s1": gg.Schedule(
            load_balance="EDGE_ONLY", blocking=True)}), max_iters=10, tolerance=0.0).array,
        "pr32": lambda: gg.pagerank(g, gg.ScheduleProgram({"s0:s1": gg.Schedule(
            load_balance="EDGE_ONLY", blocking=True)}), max_iters=10, tolerance=0.0,
            contrib_fp32=True).array,
        "bfs": lambda: np.asarray(gg.bfs_levels(gg.bfs(g, 3).values)),
        "cc": lambda: gg.cc_soman(g).array,
        "sssp": lambda: gg.sssp_delta(g, 3, gg.ScheduleProgram(
            {"s0:s1": gg.Schedule(delta=64)})).array,
    }
    results, errors = {}, []

    def worker(k):
        try:
            for rep in range(6):
                key = list(jobs)[(k + rep) % len(jobs)]
                results.setdefault(key, []).append(jobs[key]())
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == []
    for r in results["pr64"]:
        assert np.max(np.abs(r - want_pr) / want_pr) < 1e-12
    for r in results["pr32"]:
        assert np.max(np.abs(r - want_pr) / want_pr) < 1e-6
    for r in results["bfs"]:
        assert np.array_equal(r, want_lv)
    for r in results["cc"]:
        assert np.array_equal(r, want_cc)
    for r in results["sssp"]:
        assert np.array_equal(r, want_sp)
