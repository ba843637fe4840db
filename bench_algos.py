"""Per-algorithm workloads of BASELINE.json configs[1..3] (SURVEY §8d rows
C2-C4), run through the package's public API on one GPU.  bench.py calls
``run(args)`` for ``--config c2|c3|c4`` and prints the returned JSON line.

  c2  direction-optimizing BFS, RMAT-24 ef16 seed 2, symmetrised + dedup,
      64 sources (seed 3, degree > 0); hybrid s1 = PUSH+ETWC,
      s2 = PULL+BITMAP+UNFUSED_BITMAP; Graph500 TEPS (m_c = sum of degrees of
      reached vertices / 2), harmonic mean over sources.
  c3  fused delta-stepping SSSP on the 4096x4096 4-neighbour grid, uint32
      weights U[1,1000] per arc (seed 4), source 0; GTEPS = A / time.
  c4  CC (Soman hook + pointer jumping) and BC (4 sources, seed 6) on
      Graph500 Kronecker scale 25 ef16 (seed 5), symmetrised + dedup;
      ETWC vs TWC ("TWCE" baseline) vs VERTEX_BASED.
      CC GTEPS = A * hooking rounds / time; BC GTEPS = 2*m_c per source / time.

Time is the library's own device time (``RunStats.kernel_ms``: CUDA events
on the stream the kernels run on), per call, after warm-up calls.  Roofline
bytes follow SURVEY §8(d)'s fixed B_alg definitions.
"""

import json
import statistics
import time

import numpy as np


def _hmean(xs):
    xs = [x for x in xs if x > 0]
    return len(xs) / sum(1.0 / x for x in xs) if xs else 0.0


def _pick_sources(deg, n, seed):
    rng = np.random.default_rng(seed)
    cand = np.flatnonzero(deg > 0)
    return [int(x) for x in rng.choice(cand, size=min(n, len(cand)), replace=False)]


def _roof(alg_bytes, ms, peak):
    ach = alg_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": None, "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": ms}


def bfs_c2(gg, args, peak):
    scale = args.scale or 24
    t0 = time.perf_counter()
    g = gg.generate_rmat(scale, 16, seed=2, symmetrize=True)
    gen_s = time.perf_counter() - t0
    V, A = g.num_vertices, g.num_edges
    deg = np.diff(np.asarray(g.out_offsets, dtype=np.int64))
    sources = _pick_sources(deg, args.sources or 64, 3)
    theta = args.theta
    hy = gg.HybridSchedule(threshold=theta,
                           s1=gg.Schedule(direction="PUSH", load_balance="ETWC",
                                          dedup=args.dedup),
                           s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                          frontier_creation="UNFUSED_BITMAP",
                                          load_balance=args.pull_lb))
    b = {"s0:s1": hy}
    if args.fusion:
        b["s0"] = gg.Schedule(kernel_fusion=True)
    prog = gg.ScheduleProgram(b)
    import torch
    parents = torch.empty(V, dtype=torch.int32, device="cuda")
    for s in sources[:max(3, args.warmup)]:
        gg.bfs(g, s, prog, out=parents)
    teps, ms_all, rounds = [], [], []
    alg = []
    for s in sources:
        r = gg.bfs(g, s, prog, out=parents)
        reached = (parents >= 0).cpu().numpy()
        m_c = int(deg[reached].sum()) // 2
        ms = r.stats.kernel_ms
        ms_all.append(ms)
        rounds.append(r.stats.rounds)
        teps.append(m_c / (ms * 1e-3) / 1e9)
        alg.append(4.0 * int(deg[reached].sum()) + 16.0 * V)
    if args.check:
        import oracle
        off = np.asarray(g.out_offsets, dtype=np.int64)
        nbr = np.asarray(g.out_neighbors, dtype=np.int32)
        s = sources[0]
        r = gg.bfs(g, s, prog)
        assert gg.bfs_levels(r.values) == oracle.bfs_levels(V, off, nbr, s, parallel=True).tolist()
    med_ms = statistics.median(ms_all)
    i_med = ms_all.index(sorted(ms_all)[len(ms_all) // 2])
    line = {"value": _hmean(teps), "ms_per_step": med_ms, "steps": len(sources),
            "config": {"workload": "bfs_do_etwc_rmat%d_ef16_sym" % scale, "V": V, "arcs": A,
                       "sources": len(sources), "source_seed": 3,
                       "schedule": {"s1": "PUSH+ETWC" + ("" if args.dedup else "+DEDUP_DISABLED"),
                                    "s2": "PULL+BITMAP+UNFUSED_BITMAP+%s" % args.pull_lb,
                                    "threshold": theta,
                                    "kernel_fusion": bool(args.fusion)},
                       "gteps_median": statistics.median(teps), "gteps_min": min(teps),
                       "gteps_max": max(teps), "rounds_median": statistics.median(rounds),
                       "generate_s": gen_s,
                       "l2": "graph (%.1f GB) larger than L2; no flush" % (A * 4 / 1e9)},
            "roofline": dict(_roof(alg[i_med], ms_all[i_med], peak),
                             note="B_alg = 4*A_c + 16*V per source (SURVEY 8d); bottom-up "
                                  "skips arcs so frac can exceed 1 (informational)"),
            "dtype": "int32"}
    return line


def sssp_c3(gg, args, peak):
    side = args.side or 4096
    t0 = time.perf_counter()
    g = gg.generate_grid(side, seed=4, weights=True)
    gen_s = time.perf_counter() - t0
    V, A = g.num_vertices, g.num_edges
    deltas = [args.delta] if args.delta else [1024, 4096, 8192, 16384, 32768, 65536]
    import torch
    dist = torch.empty(V, dtype=torch.int64, device="cuda")
    sweep = {}
    for d in deltas:
        b = {"s0:s1": gg.Schedule(direction="PUSH", load_balance=args.lb, delta=d)}
        if not args.no_fusion:
            b["s0"] = gg.Schedule(kernel_fusion=True)
        prog = gg.ScheduleProgram(b)
        for _ in range(max(1, min(args.warmup, 2))):
            gg.sssp_delta(g, 0, prog, out=dist)
        ms = []
        st = None
        for _ in range(max(1, args.steps)):
            r = gg.sssp_delta(g, 0, prog, out=dist)
            ms.append(r.stats.kernel_ms)
            st = r.stats
        sweep[d] = {"ms": statistics.median(ms), "rounds": st.rounds,
                    "edges_traversed": st.edges_traversed,
                    "gteps": A / (statistics.median(ms) * 1e-3) / 1e9}
    best = min(sweep, key=lambda d: sweep[d]["ms"])
    if args.check:
        import oracle
        off = np.asarray(g.out_offsets, dtype=np.int64)
        nbr = np.asarray(g.out_neighbors, dtype=np.int32)
        w = np.asarray(g.out_weights, dtype=np.uint32)
        want, _ = oracle.sssp_delta(V, off, nbr, w, 0, best)
        prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(direction="PUSH", load_balance=args.lb,
                                                        delta=best),
                                   "s0": gg.Schedule(kernel_fusion=True)})
        got = gg.sssp_delta(g, 0, prog, out=np.empty(V, np.uint64)).array
        assert np.array_equal(got, want)
    ms = sweep[best]["ms"]
    return {"value": sweep[best]["gteps"], "ms_per_step": ms, "steps": max(1, args.steps),
            "config": {"workload": "sssp_delta_fused_grid%d" % side, "V": V, "arcs": A,
                       "source": 0, "weights": "uint32 U[1,1000] per arc, seed 4",
                       "best_delta": best, "lb": args.lb, "kernel_fusion": not args.no_fusion,
                       "delta_sweep": {str(k): v for k, v in sweep.items()},
                       "generate_s": gen_s},
            "roofline": dict(_roof(8.0 * A + 16.0 * V, ms, peak),
                             note="B_alg = 8*A + 16*V (SURVEY 8d); latency-bound (rounds)"),
            "dtype": "uint64"}


def cc_bc_c4(gg, args, peak):
    scale = args.scale or 25
    t0 = time.perf_counter()
    g = gg.generate_kronecker(scale, 16, seed=5, symmetrize=True, sort_by_source=True)
    gen_s = time.perf_counter() - t0
    V, A = g.num_vertices, g.num_edges
    deg = np.diff(np.asarray(g.out_offsets, dtype=np.int64))
    lbs = args.lbs.split(",")
    import torch
    labels = torch.empty(V, dtype=torch.int32, device="cuda")
    scores = torch.empty(V, dtype=torch.float64, device="cuda")
    bc_sources = _pick_sources(deg, args.sources or 4, 6)
    cc_res, bc_res = {}, {}
    for lb in lbs:
        # "EB" = EDGE_ONLY + BLOCKED (EdgeBlocking, blocking.py:78-186), "EDGE" = EDGE_ONLY,
        # "HYBRID" = BC only: PUSH+ETWC below 1% of V, PULL+BITMAP above (CC takes no hybrid)
        if lb == "HYBRID":
            hy = gg.HybridSchedule(threshold=0.01,
                                   s1=gg.Schedule(direction="PUSH", load_balance="ETWC"),
                                   s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                                  frontier_creation="UNFUSED_BITMAP"))
            progh = gg.ScheduleProgram({"s0:s1": hy})
            gg.bc(g, bc_sources[:1], progh, out=scores)
            r = gg.bc(g, bc_sources, progh, out=scores)
            bc_res[lb] = {"ms": r.stats.kernel_ms, "rounds": r.stats.rounds,
                          "edges_traversed": r.stats.edges_traversed}
            continue
        if lb == "EB":
            sch = gg.Schedule(load_balance="EDGE_ONLY", blocking=True)
        elif lb == "EDGE":
            sch = gg.Schedule(load_balance="EDGE_ONLY")
        else:
            sch = gg.Schedule(direction="PUSH", load_balance=lb)
        prog = gg.ScheduleProgram({"s0:s1": sch})
        for _ in range(max(1, min(args.warmup, 2))):
            gg.cc_soman(g, prog, out=labels)
        ms, st = [], None
        for _ in range(max(1, args.steps)):
            r = gg.cc_soman(g, prog, out=labels)
            ms.append(r.stats.kernel_ms)
            st = r.stats
        m = statistics.median(ms)
        cc_res[lb] = {"ms": m, "rounds": st.rounds, "edges_traversed": st.edges_traversed,
                      "gteps": st.edges_traversed / (m * 1e-3) / 1e9,
                      "frac": ((4.0 * A + 16.0 * V) * st.rounds / (m * 1e-3) / 1e9) / peak}
        if lb in ("EB", "EDGE"):  # frontier traversals: EDGE_ONLY would scan every arc per level
            continue
        gg.bc(g, bc_sources[:1], prog, out=scores)
        r = gg.bc(g, bc_sources, prog, out=scores)
        bm = r.stats.kernel_ms
        # reached arcs per source ~ the giant component: sum of degrees of
        # vertices with a path from the source (same component as sources[0])
        bc_res[lb] = {"ms": bm, "rounds": r.stats.rounds,
                      "edges_traversed": r.stats.edges_traversed}
    lab = labels.cpu().numpy()
    m_c = []
    for s in bc_sources:
        m_c.append(int(deg[lab == lab[s]].sum()) // 2)
    for lb in bc_res:
        bc_res[lb]["gteps"] = 2.0 * sum(m_c) / (bc_res[lb]["ms"] * 1e-3) / 1e9
    if args.check:
        import oracle
        want, _ = oracle.cc(V, np.asarray(g.coo_src), np.asarray(g.coo_dst))
        assert np.array_equal(lab, want)
    head = lbs[0]
    ms = cc_res[head]["ms"]
    return {"value": cc_res[head]["gteps"], "ms_per_step": ms, "steps": max(1, args.steps),
            "config": {"workload": "cc_bc_kron%d_ef16_sym" % scale, "V": V, "arcs": A,
                       "coo_order": "by source (edge-list order; matters for EDGE_ONLY/EB only)",
                       "headline": "CC %s (GTEPS = A x hooking rounds / time)" % head,
                       "cc": cc_res, "bc": bc_res, "bc_sources": bc_sources,
                       "bc_m_c": m_c, "generate_s": gen_s},
            "roofline": dict(_roof((4.0 * A + 16.0 * V) * cc_res[head]["rounds"], ms, peak),
                             note="B_alg = (4*A + 16*V) per hooking round (SURVEY 8d)"),
            "dtype": "int32"}


def run(args, peak, peak_kind):
    import paper_2012_07990_b200 as gg
    import torch
    torch.cuda.set_device(0)
    fn = {"c2": bfs_c2, "c3": sssp_c3, "c4": cc_bc_c4}[args.config]
    line = fn(gg, args, peak)
    line["roofline"]["peak_kind"] = peak_kind
    return line


if __name__ == "__main__":
    raise SystemExit("run through bench.py --config c2|c3|c4")
