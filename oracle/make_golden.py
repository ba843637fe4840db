"""Generate tests/golden/* by running the REFERENCE package (schedge) here.

TEST INFRASTRUCTURE: run in the dev container, where /root/reference exists:
    python oracle/make_golden.py
The fixtures pin both the CPU oracle (oracle.c) and, on the GPU box, the
device engine to the reference's own outputs and RunStats.  Graph builders
are the reference's test builders (pkg/tests/util.py) plus the counter-based
RMAT/grid generators of oracle/gen.py (bit-identical to csrc/graph.cu).
"""

import hashlib
import json
import math
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, ROOT)

import schedge  # noqa: E402
from schedge import algos, blocking, engine, oracle as ref_oracle  # noqa: E402
from schedge.graphio import Graph, _symmetrize, with_random_weights  # noqa: E402
from schedge.runtime import ExecConfig, Runtime  # noqa: E402
from schedge.sched import Schedule, ScheduleProgram, parse_schedule  # noqa: E402
import util  # noqa: E402  (reference test builders)

from oracle import gen  # noqa: E402


def graph_record(g):
    return {"V": g.num_vertices, "src": list(g.coo_src), "dst": list(g.coo_dst),
            "w": None if g.coo_weights is None else list(g.coo_weights),
            "symmetric": bool(g.symmetric)}


def stats_record(st):
    d = st.to_dict()
    return {k: d[k] for k in ("dispatch_count", "rounds", "edges_traversed", "direction_log",
                              "frontier_conversions", "frontier_allocations",
                              "reused_frontiers", "creation_passes")}


def program_with(s, fusion=False):
    p = ScheduleProgram({"s0:s1": s.copy()})
    if fusion:
        p.bindings["s0"] = Schedule(kernel_fusion=True)
    return p


def sched_dict(s):
    return {k: getattr(s, k) for k in ("direction", "pull_frontier_repr", "load_balance",
                                        "blocking", "blocking_size", "frontier_creation",
                                        "dedup", "dedup_strategy", "delta", "kernel_fusion")}


def small_cases():
    cases = []
    graphs = {
        "path4": util.path_graph(4),
        "path12": util.path_graph(12),
        "rs70": util.random_symmetric(70, 220, 0),
        "rs150": util.random_symmetric(150, 450, 1),
        "pa200": util.preferential_attachment(200, 3, 2),
        "pa800": util.preferential_attachment(800, 3, 4),
        "tri": Graph.from_coo(6, [0, 1, 2, 3, 4, 5], [1, 2, 0, 4, 5, 3], symmetric=True),
        "clique24": util.clique(24),
        "iso3": Graph.from_coo(3, [1], [2]),
        "loops": Graph.from_coo(4, [0, 0, 0, 1, 2, 2], [0, 1, 1, 2, 2, 3], [5, 1, 1, 2, 9, 4]),
    }
    weighted = {
        "rd60w": util.random_directed(60, 240, 0, weighted=True, max_weight=50),
        "rd60w1": util.random_directed(60, 240, 1, weighted=True, max_weight=50),
        "hand3": Graph.from_coo(3, [0, 0, 1], [1, 2, 2], [2, 10, 3]),
        "rd150w": util.random_directed(150, 600, 21, weighted=True, max_weight=40),
        "pathw": with_random_weights(util.path_graph(6), 1, 1000, seed=1),
        "loops": graphs["loops"],
    }
    lbs = ["VERTEX_BASED", "CM", "WM", "STRICT", "EDGE_ONLY", "ETWC", "TWC"]
    # BFS: default schedule + every LB + pull + hybrid (stats are deterministic)
    for name in ("path4", "path12", "rs70", "rs150", "pa200", "tri", "clique24", "iso3", "loops"):
        g = graphs[name]
        for lb in lbs:
            for direction in ("PUSH", "PULL"):
                s = Schedule(direction=direction, load_balance=lb)
                r = algos.bfs(g, 0, program_with(s))
                cases.append({"algo": "bfs", "graph": name, "source": 0, "schedule": sched_dict(s),
                              "levels": algos.bfs_levels(r.values), "parents": r.values,
                              "stats": stats_record(r.stats)})
    hybrid_text = """
    SimpleGPUSchedule s1;
    s1.configDirection(PUSH);
    SimpleGPUSchedule s2;
    s2.configDirection(PULL, BITMAP);
    s2.configFrontierCreation(UNFUSED_BITMAP);
    HybridGPUSchedule h1(INPUT_VERTEXSET_SIZE, 0.05, s1, s2);
    apply("s0:s1", h1);
    """
    for name in ("pa200", "pa800", "path12"):
        g = graphs[name]
        hub = max(range(g.num_vertices), key=lambda v: g.out_offsets[v + 1] - g.out_offsets[v])
        r = algos.bfs(g, hub, parse_schedule(hybrid_text))
        cases.append({"algo": "bfs", "graph": name, "source": hub, "schedule_text": hybrid_text,
                      "levels": algos.bfs_levels(r.values), "parents": r.values,
                      "stats": stats_record(r.stats)})
    # PageRank
    for name in ("rs70", "pa200", "loops", "clique24"):
        g = graphs[name]
        for s in (Schedule(load_balance="EDGE_ONLY"), Schedule(direction="PULL"),
                  Schedule(load_balance="EDGE_ONLY", blocking=True, blocking_size=16),
                  Schedule(direction="PULL", load_balance="TWC"), Schedule(load_balance="STRICT")):
            r = algos.pagerank(g, program_with(s), max_iters=30, tolerance=0.0)
            cases.append({"algo": "pagerank", "graph": name, "max_iters": 30, "tolerance": 0.0,
                          "schedule": sched_dict(s), "ranks": r.values,
                          "stats": stats_record(r.stats)})
        r = algos.pagerank(g)
        cases.append({"algo": "pagerank", "graph": name, "max_iters": 100, "tolerance": 1e-9,
                      "schedule": None, "ranks": r.values, "stats": stats_record(r.stats)})
    # SSSP
    for name, g in weighted.items():
        for delta in (1, 16, 64, 10**9):
            s = Schedule(delta=delta)
            r = algos.sssp_delta(g, 0, program_with(s))
            cases.append({"algo": "sssp", "graph": name, "source": 0, "schedule": sched_dict(s),
                          "dist": [None if math.isinf(x) else int(x) for x in r.values],
                          "stats": stats_record(r.stats)})
    # CC
    for name in ("rs70", "rs150", "pa200", "tri", "path12", "clique24"):
        g = graphs[name]
        for lb in ("VERTEX_BASED", "EDGE_ONLY", "ETWC", "CM", "TWC"):
            s = Schedule(load_balance=lb)
            r = algos.cc_soman(g, program_with(s))
            cases.append({"algo": "cc", "graph": name, "schedule": sched_dict(s),
                          "labels": r.values, "stats": stats_record(r.stats)})
    # BC
    for name, srcs in (("rs70", [0, 7, 21]), ("pa200", [0, 5, 50]), ("path4", [0, 1, 2, 3]),
                       ("tri", [0, 3]), ("clique24", [0, 1])):
        g = graphs[name]
        for s in (Schedule(), Schedule(direction="PULL"), Schedule(load_balance="ETWC")):
            r = algos.bc(g, srcs, program_with(s))
            cases.append({"algo": "bc", "graph": name, "sources": srcs, "schedule": sched_dict(s),
                          "scores": r.values, "stats": stats_record(r.stats)})
    # EdgeBlocking Alg. 1
    for name in ("rs70", "pa200", "loops"):
        g = graphs[name]
        for n in (1, 3, 7, 16, 10**6):
            bg = blocking.block_edges(g, n)
            cases.append({"algo": "block_edges", "graph": name, "n": n,
                          "segment_start": list(bg.segment_start), "src": list(bg.edges_src),
                          "dst": list(bg.edges_dst)})
    # ETWC / TWC / STRICT partitions (engine.py:51-142)
    for name in ("pa200", "rs150"):
        g = graphs[name]
        active = list(range(0, g.num_vertices, 3))
        for workers, cta, warp in ((1, 256, 32), (4, 64, 8), (3, 32, 4)):
            cfg = ExecConfig(num_workers=workers, cta_size=cta, warp_size=warp)
            cases.append({"algo": "partition", "graph": name, "active": active,
                          "cfg": [workers, cta, warp],
                          "etwc": engine.lb_partition_etwc(active, g, cfg),
                          "twc": engine.lb_partition_twc(active, g, cfg),
                          "strict": engine.lb_partition_strict(active, g, cfg)})
    all_graphs = dict(graphs)
    all_graphs.update(weighted)
    return {"graphs": {k: graph_record(v) for k, v in all_graphs.items()}, "cases": cases}


def c1_pagerank():
    """C1: PageRank 20 iterations on RMAT scale 16 (BASELINE configs[0])."""
    V, s, d = gen.rmat(16, 16, seed=1)
    t0 = time.time()
    g = Graph.from_coo(V, s, d)
    build = time.time() - t0
    t0 = time.time()
    r = algos.pagerank(g, None, ExecConfig(num_workers=1), max_iters=20, tolerance=0.0)
    run = time.time() - t0
    h = hashlib.sha256(s.tobytes() + d.tobytes()).hexdigest()
    np.savez_compressed(os.path.join(OUT, "c1_pagerank_rmat16.npz"),
                        ranks=np.asarray(r.values, np.float64), edge_sha256=h,
                        stats=json.dumps(stats_record(r.stats)))
    return {"build_s": build, "run_s": run, "sha": h}


def sidecars():
    """Blocked-graph sidecars written by the reference's own save_blocked
    (blocking.py:189-217): a weighted RMAT-8 at two widths."""
    V, s, d = gen.rmat(8, 4, seed=11)
    w = gen.weights(len(s), 11)
    g = Graph.from_coo(V, s.tolist(), d.tolist(), w.astype(np.int64).tolist())
    for n in (16, 100):
        bg = blocking.block_edges(g, n)
        blocking.save_blocked(bg, os.path.join(OUT, "ref_sidecar_rmat8_n%d.blk" % n))
    gu = Graph.from_coo(V, s.tolist(), d.tolist())
    blocking.save_blocked(blocking.block_edges(gu, 32),
                          os.path.join(OUT, "ref_sidecar_rmat8_unweighted_n32.blk"))


def rmat12_cases():
    """Scale-12 RMAT (symmetrised for BFS/CC/BC, weighted for SSSP)."""
    V, s, d = gen.rmat(12, 16, seed=2)
    ss, dd, _, _ = _symmetrize(s.tolist(), d.tolist(), None)
    gs = Graph.from_coo(V, ss, dd, symmetric=True)
    out = {"V": V, "seed": 2}
    hub = int(np.argmax(np.diff(np.asarray(gs.out_offsets))))
    out["bfs_source"] = hub
    out["bfs_levels"] = algos.bfs_levels(algos.bfs(gs, hub).values)
    out["cc_labels"] = algos.cc_soman(gs).values
    out["bc_sources"] = [hub, 1, 2]
    out["bc_scores"] = algos.bc(gs, [hub, 1, 2]).values
    w = gen.weights(len(s), 4)
    gw = Graph.from_coo(V, s, d, w.tolist())
    out["sssp_source"] = 0
    out["sssp_delta"] = 64
    r = algos.sssp_delta(gw, 0, program_with(Schedule(delta=64)))
    out["sssp_dist"] = [None if math.isinf(x) else int(x) for x in r.values]
    out["sym_arcs"] = len(ss)
    with open(os.path.join(OUT, "rmat12.json"), "w") as fh:
        json.dump(out, fh)


def scale16_cases():
    """Larger pins (reference at scale <= 18): BFS levels and CC
    labels on symmetrised RMAT-16 (seed 2), delta-stepping distances on the
    128x128 grid (weights seed 4), BC on symmetrised RMAT-13 (seed 6)."""
    V, s, d = gen.rmat(16, 16, seed=2)
    ss, dd, _, _ = _symmetrize(s.tolist(), d.tolist(), None)
    gs = Graph.from_coo(V, ss, dd, symmetric=True)
    hub = int(np.argmax(np.diff(np.asarray(gs.out_offsets))))
    levels = algos.bfs_levels(algos.bfs(gs, hub).values)
    labels = algos.cc_soman(gs).values
    Vg, gsrc, gdst = gen.grid(128)
    wg = gen.weights(len(gsrc), 4)
    gg_ = Graph.from_coo(Vg, gsrc.tolist(), gdst.tolist(), wg.tolist())
    dist = {}
    for delta in (64, 1024):
        r = algos.sssp_delta(gg_, 0, program_with(Schedule(delta=delta)))
        dist[delta] = np.asarray([-1 if math.isinf(x) else int(x) for x in r.values], np.int64)
    Vb, bs, bd = gen.rmat(13, 8, seed=6)
    bss, bdd, _, _ = _symmetrize(bs.tolist(), bd.tolist(), None)
    gb = Graph.from_coo(Vb, bss, bdd, symmetric=True)
    bsrc = [int(np.argmax(np.diff(np.asarray(gb.out_offsets)))), 5]
    scores = np.asarray(algos.bc(gb, bsrc).values, np.float64)
    np.savez_compressed(os.path.join(OUT, "scale16.npz"), bfs_source=hub,
                        bfs_levels=np.asarray(levels, np.int32), cc_labels=np.asarray(labels, np.int32),
                        sym_arcs=len(ss), sssp_d64=dist[64], sssp_d1024=dist[1024],
                        bc_sources=np.asarray(bsrc), bc_scores=scores, bc_arcs=len(bss))


def tune_candidates():
    """tests/golden/tune_candidates.json: the reference tuner's candidate
    lists (cli.candidate_schedules) per algorithm -- count, first five keys,
    and a seeded random strategy with a limit."""
    import json
    from schedge import cli, sched
    out = {}
    for algo in cli.ALGO_DIMENSIONS:
        c = cli.candidate_schedules(algo)
        r = cli.candidate_schedules(algo, seed=3, strategy="random", limit=7)
        out[algo] = {"n": len(c), "first5": [sched.schedule_key(s) for s in c[:5]],
                     "random3_7": [sched.schedule_key(s) for s in r]}
    with open(os.path.join(OUT, "tune_candidates.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    t = time.time()
    data = small_cases()
    with open(os.path.join(OUT, "reference_small.json"), "w") as fh:
        json.dump(data, fh)
    print("small cases:", len(data["cases"]), "%.1fs" % (time.time() - t))
    t = time.time()
    rmat12_cases()
    print("rmat12: %.1fs" % (time.time() - t))
    print("c1:", c1_pagerank())
    tune_candidates()
    scale16_cases()
    sidecars()
