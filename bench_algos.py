"""Workloads of BASELINE.json configs[0..3], run
through the package's public API on one GPU.  ``bench.py --config c1|c2|c3|c4``
prints one JSON line from ``run(args)``; the default ``bench.py`` run (C5)
runs each of them in a subprocess after its own timed region and nests the
lines under ``"configs"``.

  c1  PageRank 20 iterations, RMAT-16 ef16 seed 1 (V = 65,536, E = 2^20),
      tolerance 0; the reference's default EDGE_ONLY schedule, EdgeBlocking,
      and the loop-fused variants of both; GTEPS = 20*E / call time.
  c2  direction-optimizing BFS, RMAT-24 ef16 seed 2, symmetrised + dedup,
      64 sources (seed 3, degree > 0); hybrid s1 = PUSH+ETWC,
      s2 = PULL+BITMAP+UNFUSED_BITMAP; Graph500 TEPS (m_c = sum of degrees of
      reached vertices / 2), harmonic mean over sources.
  c3  fused delta-stepping SSSP on the 4096x4096 4-neighbour grid, uint32
      weights U[1,1000] per arc (seed 4), source 0; GTEPS = A / time.
  c4  CC (Soman hook + pointer jumping) and BC (4 sources, seed 6) on
      Graph500 Kronecker scale 25 ef16 (seed 5), symmetrised + dedup;
      ETWC vs TWC ("TWCE" baseline) vs VERTEX_BASED (+ EDGE_ONLY, EB).
      CC GTEPS = A * hooking rounds / time; BC GTEPS = 2*m_c per source / time.

Every line carries, beside the device-timed ``value`` (``RunStats.kernel_ms``:
CUDA events on the stream the library's kernels run on, after warm-up):
  * ``roofline`` — SURVEY §8(d)'s fixed B_alg over that time;
  * ``e2e`` — the same metric through the public API from pinned host arrays
    (``Graph.from_coo`` upload + device build + the queries + results copied
    back to host numpy), copies inside the timed region;
  * ``parity`` — the full-size result against the CPU oracle (bit-exact BFS
    levels + parent-tree legality for all sources, SSSP distances, CC labels
    for every load balancer; BC <= 1e-5 relative; C1 also against the
    reference's own ranks, tests/golden/c1_pagerank_rmat16.npz);
  * ``cpu_baseline`` — that oracle call's time on the host cores (the C
    restatement, "port"), and for C1 the reference package itself
    (``baseline/_ref``, installed by ``__graft_entry__.build()``) when present.
The oracle is test infrastructure: it is the checker and the CPU baseline
here, never the measured path.
"""

import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))


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


def _pinned(*arrays):
    import torch
    out = []
    for a in arrays:
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        out.append((t, t.numpy()))
    return out


def _threads():
    import oracle
    return oracle.num_threads()


def _rel_err(got, want, floor=0.0):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    m = np.abs(want) > floor
    if not m.any():
        return 0.0
    return float(np.max(np.abs(got[m] - want[m]) / np.abs(want[m])))


def _sync():
    import torch
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# C1: PageRank RMAT-16 (the config the reference itself runs)
# ---------------------------------------------------------------------------
def _python_reference_c1(s, d, V, iters):
    """The reference package's own CPU path on C1 (cli.py:166-175 protocol,
    one timed run: ~7 s/run), when baseline/_ref holds it."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "schedge")):
        return None
    sys.path.insert(0, ref)
    try:
        import schedge
        g = schedge.Graph.from_coo(V, s.tolist(), d.tolist())
        cfg = schedge.ExecConfig(num_workers=1)
        t0 = time.perf_counter()
        r = schedge.pagerank(g, None, cfg, max_iters=iters, tolerance=0.0)
        dt = time.perf_counter() - t0
        return {"value": iters * len(s) / dt / 1e9, "unit": "GTEPS", "cores": 1,
                "kind": "reference", "ranks": np.asarray(r.values, np.float64),
                "sample": "schedge.algos.pagerank (baseline/_ref), full C1: RMAT-16 ef16 seed 1, "
                          "%d iterations, ExecConfig(num_workers=1), one run in %.2f s "
                          "(GIL-bound: 1 core effective; box has %d)"
                          % (iters, dt, os.cpu_count() or 0)}
    except Exception as e:  # reported, not fatal: the oracle port stands in
        return {"error": "%s: %s" % (type(e).__name__, e)}
    finally:
        sys.path.remove(ref)


def pagerank_c1(gg, args, peak):
    import oracle
    import torch
    scale, ef, seed, iters = 16, 16, 1, 20
    g = gg.generate_rmat(scale, ef, seed=seed)
    V, E = g.num_vertices, g.num_edges
    s, d = g.coo_src.copy(), g.coo_dst.copy()
    variants = {
        "EDGE_ONLY": {"s0:s1": gg.Schedule(load_balance="EDGE_ONLY")},
        "EDGE_ONLY+BLOCKED": {"s0:s1": gg.Schedule(load_balance="EDGE_ONLY", blocking=True)},
        "EDGE_ONLY+fused": {"s0:s1": gg.Schedule(load_balance="EDGE_ONLY"),
                            "s0": gg.Schedule(kernel_fusion=True)},
        "EDGE_ONLY+BLOCKED+fused": {"s0:s1": gg.Schedule(load_balance="EDGE_ONLY",
                                                         blocking=True),
                                    "s0": gg.Schedule(kernel_fusion=True)},
    }
    ranks = torch.empty(V, dtype=torch.float64, device="cuda")
    res = {}
    steps = max(5, args.steps)
    for name, b in variants.items():
        prog = gg.ScheduleProgram(b)
        for _ in range(max(3, args.warmup)):
            gg.pagerank(g, prog, max_iters=iters, tolerance=0.0, out=ranks)
        ms, launches = [], 0
        for _ in range(steps):
            r = gg.pagerank(g, prog, max_iters=iters, tolerance=0.0, out=ranks)
            ms.append(r.stats.kernel_ms)
            launches = r.stats.gpu_launches
        m = statistics.median(ms)
        res[name] = {"ms": m, "gteps": iters * E / (m * 1e-3) / 1e9, "gpu_launches": launches,
                     "ranks": ranks.cpu().numpy().copy()}
    best = max(res, key=lambda k: res[k]["gteps"])
    prog = gg.ScheduleProgram(variants[best])

    # parity: every variant against the reference's own ranks and the oracle
    golden = np.load(os.path.join(ROOT, "tests", "golden", "c1_pagerank_rmat16.npz"))
    t0 = time.perf_counter()
    want, _ = oracle.pagerank(V, s, d, iters, 0.0)
    port_s = time.perf_counter() - t0
    parity = {"vs": "reference ranks (tests/golden/c1_pagerank_rmat16.npz, made by running "
                    "schedge) and oracle.pagerank", "tolerance": 1e-6,
              "max_rel_err": {}, "max_rel_err_oracle": {}}
    for k, v in res.items():
        parity["max_rel_err"][k] = _rel_err(v.pop("ranks"), golden["ranks"])
        parity["max_rel_err_oracle"][k] = _rel_err(
            gg.pagerank(g, gg.ScheduleProgram(variants[k]), max_iters=iters,
                        tolerance=0.0).array, want)
    parity["ok"] = max(parity["max_rel_err"].values()) <= 1e-6

    # e2e: pinned host COO -> Graph.from_coo -> pagerank -> host ranks
    g.close()
    (ts, sh), (td, dh) = _pinned(s, d)
    out_h = _pinned(np.empty(V, np.float64))[0][1]

    def e2e_step():
        ge = gg.Graph.from_coo(V, sh, dh)
        gg.pagerank(ge, prog, max_iters=iters, tolerance=0.0, out=out_h)
        ge.close()

    for _ in range(3):
        e2e_step()
    _sync()
    t0 = time.perf_counter()
    n_e2e = 10
    for _ in range(n_e2e):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / n_e2e
    parity["e2e_max_rel_err"] = _rel_err(out_h, golden["ranks"])

    cpu = _python_reference_c1(s, d, V, iters)
    port = {"value": iters * E / port_s / 1e9, "unit": "GTEPS", "cores": 1, "kind": "port",
            "sample": "oracle.c or_pagerank (the reference's EDGE_ONLY COO-order loop restated "
                      "in C, serial), full C1, %d iterations in %.3f s" % (iters, port_s)}
    if cpu and "ranks" in cpu:
        parity["python_reference_max_rel_err"] = _rel_err(cpu.pop("ranks"), golden["ranks"])
        cpu["restated_cpu"] = port
    else:
        if cpu:
            port["python_reference_error"] = cpu["error"]
        cpu = port
    m = res[best]["ms"]
    return {"value": res[best]["gteps"], "ms_per_step": m, "steps": steps,
            "config": {"workload": "pagerank_rmat16_ef16_c1", "V": V, "E": E,
                       "iterations": iters, "headline_schedule": best, "variants": res,
                       "l2": "graph (12 MB) fits in L2: latency/launch-bound by design "
                             "(SURVEY 8d C1)"},
            "roofline": dict(_roof(iters * (8.0 * E + 32.0 * V), m, peak),
                             note="B_alg = (8E + 32V) per iteration (SURVEY 8d)"),
            "e2e": {"value": iters * E / e2e_s / 1e9, "unit": "GTEPS",
                    "h2d_bytes_per_step": 8 * E, "d2h_bytes_per_step": 8 * V,
                    "s_per_step": e2e_s,
                    "includes": "Graph.from_coo from pinned host COO (upload + device CSR "
                                "build), %s PageRank %d iterations, ranks to host" % (best, iters)},
            "cpu_baseline": cpu, "parity": parity, "dtype": "f64"}


# ---------------------------------------------------------------------------
# C2: direction-optimizing BFS, RMAT-24
# ---------------------------------------------------------------------------
def bfs_c2(gg, args, peak):
    import oracle
    import torch
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
                                          dedup=args.dedup,
                                          frontier_creation=args.push_creation),
                           s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                          frontier_creation="UNFUSED_BITMAP",
                                          load_balance=args.pull_lb))
    b = {"s0:s1": hy}
    if args.fusion:
        b["s0"] = gg.Schedule(kernel_fusion=True)
    prog = gg.ScheduleProgram(b)
    parents = torch.empty(V, dtype=torch.int32, device="cuda")
    for s in sources[:max(3, args.warmup)]:
        gg.bfs(g, s, prog, out=parents)
    teps, ms_all, rounds, alg, m_c_all, got = [], [], [], [], [], []
    for s in sources:
        r = gg.bfs(g, s, prog, out=parents)
        ms_all.append(r.stats.kernel_ms)
        p = parents.cpu().numpy()
        got.append(p)
        reached = p >= 0
        m_c = int(deg[reached].sum()) // 2
        m_c_all.append(m_c)
        rounds.append(r.stats.rounds)
        teps.append(m_c / (r.stats.kernel_ms * 1e-3) / 1e9)
        alg.append(4.0 * int(deg[reached].sum()) + 16.0 * V)
    med_ms = statistics.median(ms_all)
    i_med = ms_all.index(sorted(ms_all)[len(ms_all) // 2])

    # parity (all sources): levels bit-exact vs the oracle, parents a legal BFS tree
    src_h, dst_h = g.coo_src.copy(), g.coo_dst.copy()
    off, nbr, _ = oracle.csr_par(V, src_h, dst_h)
    bad_lv, bad_tree, cpu_teps, cpu_s = 0, 0, [], 0.0
    for i, s in enumerate(sources):
        t0 = time.perf_counter()
        lv = oracle.bfs_levels_do(V, off, nbr, s)
        dt = time.perf_counter() - t0
        cpu_s += dt
        cpu_teps.append(m_c_all[i] / dt / 1e9)
        got_lv = np.asarray(gg.bfs_levels(got[i]), np.int32)
        bad_lv += int(not np.array_equal(got_lv, lv))
        bad_tree += int(oracle.bfs_check_tree(V, off, nbr, s, got[i], lv) != 0)
    parity = {"vs": "oracle.bfs_levels_do (levels) + oracle.bfs_check_tree (parent legality)",
              "sources_checked": len(sources), "level_mismatches": bad_lv,
              "illegal_trees": bad_tree, "ok": bad_lv == 0 and bad_tree == 0}
    del got

    # e2e: pinned host COO -> Graph.from_coo (symmetric) -> 64 BFS -> parents on host
    g.close()
    (ts, sh), (td, dh) = _pinned(src_h, dst_h)
    out_h = _pinned(np.empty(V, np.int32))[0][1]
    ge = gg.Graph.from_coo(V, sh, dh, symmetric=True)  # warm-up (pool, CSR kernels)
    gg.bfs(ge, sources[0], prog, out=out_h)
    ge.close()
    _sync()
    t0 = time.perf_counter()
    ge = gg.Graph.from_coo(V, sh, dh, symmetric=True)
    for s in sources:
        gg.bfs(ge, s, prog, out=out_h)
    e2e_s = time.perf_counter() - t0
    ge.close()
    return {"value": _hmean(teps), "ms_per_step": med_ms, "steps": len(sources),
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
            "e2e": {"value": sum(m_c_all) / e2e_s / 1e9, "unit": "GTEPS",
                    "h2d_bytes_per_step": 8 * A, "d2h_bytes_per_step": 4 * V * len(sources),
                    "s_per_step": e2e_s,
                    "includes": "one step = Graph.from_coo of the symmetric COO from pinned "
                                "host memory + %d BFS queries, each parent array copied to "
                                "host" % len(sources)},
            "cpu_baseline": {"value": _hmean(cpu_teps), "unit": "GTEPS", "cores": _threads(),
                             "kind": "port",
                             "sample": "oracle.c or_bfs_levels_do (direction-optimising, "
                                       "OpenMP) on the full C2 graph, all %d sources in "
                                       "%.1f s; harmonic mean of per-source Graph500 TEPS"
                                       % (len(sources), cpu_s)},
            "parity": parity, "dtype": "int32"}


# ---------------------------------------------------------------------------
# C3: fused delta-stepping SSSP, 4096^2 grid
# ---------------------------------------------------------------------------
def sssp_c3(gg, args, peak):
    import oracle
    import torch
    side = args.side or 4096
    t0 = time.perf_counter()
    g = gg.generate_grid(side, seed=4, weights=True)
    gen_s = time.perf_counter() - t0
    V, A = g.num_vertices, g.num_edges
    deltas = [args.delta] if args.delta else [8192, 10240, 12288, 16384]
    dist = torch.empty(V, dtype=torch.int64, device="cuda")

    def program(d):
        b = {"s0:s1": gg.Schedule(direction="PUSH", load_balance=args.lb, delta=d)}
        if not args.no_fusion:
            b["s0"] = gg.Schedule(kernel_fusion=True)
        return gg.ScheduleProgram(b)

    sweep = {}
    for d in deltas:
        prog = program(d)
        for _ in range(max(1, min(args.warmup, 2))):
            gg.sssp_delta(g, 0, prog, out=dist)
        ms, st = [], None
        for _ in range(max(1, min(args.steps, 5))):
            r = gg.sssp_delta(g, 0, prog, out=dist)
            ms.append(r.stats.kernel_ms)
            st = r.stats
        sweep[d] = {"ms": statistics.median(ms), "rounds": st.rounds,
                    "edges_traversed": st.edges_traversed,
                    "gteps": A / (statistics.median(ms) * 1e-3) / 1e9}
    best = min(sweep, key=lambda d: sweep[d]["ms"])
    prog = program(best)
    got = gg.sssp_delta(g, 0, prog, out=dist).array
    got = got.cpu().numpy().view(np.uint64)

    # parity: distances bit-exact against the reference's delta-stepping restated
    s_h, d_h, w_h = g.coo_src.copy(), g.coo_dst.copy(), g.coo_weights.copy()
    off, nbr, ww = oracle.csr_par(V, s_h, d_h, w_h)
    t0 = time.perf_counter()
    want, cpu_rounds = oracle.sssp_delta(V, off, nbr, ww, 0, best)
    cpu_s = time.perf_counter() - t0
    parity = {"vs": "oracle.sssp_delta (priority.py:17-118 + algos.py:215-247 restated), "
                    "delta %d" % best,
              "mismatches": int(np.count_nonzero(got != want)),
              "ok": bool(np.array_equal(got, want))}

    # e2e: pinned host COO + weights -> Graph.from_coo -> fused SSSP -> distances on host
    g.close()
    (a, sh), (b_, dh), (c_, wh) = _pinned(s_h, d_h, w_h)
    out_h = _pinned(np.empty(V, np.uint64))[0][1]

    def e2e_step():
        ge = gg.Graph.from_coo(V, sh, dh, wh)
        gg.sssp_delta(ge, 0, prog, out=out_h)
        ge.close()

    e2e_step()
    _sync()
    t0 = time.perf_counter()
    for _ in range(3):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / 3
    parity["e2e_ok"] = bool(np.array_equal(out_h, want))
    ms = sweep[best]["ms"]
    return {"value": sweep[best]["gteps"], "ms_per_step": ms, "steps": max(1, min(args.steps, 5)),
            "config": {"workload": "sssp_delta_fused_grid%d" % side, "V": V, "arcs": A,
                       "source": 0, "weights": "uint32 U[1,1000] per arc, seed 4",
                       "best_delta": best, "lb": args.lb, "kernel_fusion": not args.no_fusion,
                       "delta_sweep": {str(k): v for k, v in sweep.items()},
                       "generate_s": gen_s},
            "roofline": dict(_roof(8.0 * A + 16.0 * V, ms, peak),
                             note="B_alg = 8*A + 16*V (SURVEY 8d); latency-bound (rounds)"),
            "e2e": {"value": A / e2e_s / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": 12 * A,
                    "d2h_bytes_per_step": 8 * V, "s_per_step": e2e_s,
                    "includes": "Graph.from_coo of COO + weights from pinned host memory, "
                                "fused SSSP, distances to host"},
            "cpu_baseline": {"value": A / cpu_s / 1e9, "unit": "GTEPS", "cores": 1,
                             "kind": "port",
                             "sample": "oracle.c or_sssp_delta (serial two-bucket "
                                       "delta-stepping), full C3 grid, delta %d, %d rounds in "
                                       "%.2f s" % (best, cpu_rounds, cpu_s)},
            "parity": parity, "dtype": "uint64"}


# ---------------------------------------------------------------------------
# C4: CC + BC, Kronecker-25
# ---------------------------------------------------------------------------
def _bc_timed(gg, g, sources, prog, scores, reps=3):
    """Median device time of `reps` identical BC calls (single calls vary
    with what the allocator and L2 hold from the previous query)."""
    ms, r = [], None
    for _ in range(reps):
        r = gg.bc(g, sources, prog, out=scores)
        ms.append(r.stats.kernel_ms)
    return r, statistics.median(ms)


def cc_bc_c4(gg, args, peak):
    import oracle
    import torch
    scale = args.scale or 25
    t0 = time.perf_counter()
    g = gg.generate_kronecker(scale, 16, seed=5, symmetrize=True, sort_by_source=True)
    gen_s = time.perf_counter() - t0
    V, A = g.num_vertices, g.num_edges
    deg = np.diff(np.asarray(g.out_offsets, dtype=np.int64))
    s_h, d_h = g.coo_src.copy(), g.coo_dst.copy()
    lbs = args.lbs.replace("+", ",").split(",")  # "+" also separates (tools/gpu.sh turns "," into spaces)
    if not any(lb != "HYBRID" for lb in lbs):
        raise SystemExit("--lbs needs a CC load balance besides HYBRID (ETWC, TWC, VERTEX_BASED, EB, EDGE)")
    labels = torch.empty(V, dtype=torch.int32, device="cuda")
    scores = torch.empty(V, dtype=torch.float64, device="cuda")
    bc_sources = _pick_sources(deg, args.sources or 4, 6)
    # the degree-ordered copy CC/BC query on (relabel.cu), built ahead like
    # the EdgeBlocking layout: preprocessing, reported apart
    relabel_ms = g.prepare_relabel() if os.environ.get("GG_RELABEL", "1") != "0" else 0.0

    # oracle results first (parity for every load balancer below)
    t0 = time.perf_counter()
    want_cc, cpu_cc_rounds = oracle.cc_par(V, s_h, d_h)
    cpu_cc_s = time.perf_counter() - t0
    off, nbr, _ = oracle.csr_par(V, s_h, d_h)
    t0 = time.perf_counter()
    want_bc = oracle.bc_par(V, off, nbr, bc_sources)
    cpu_bc_s = time.perf_counter() - t0
    del off, nbr
    bc_floor = 1e-6 * float(np.max(want_bc))

    cc_res, bc_res = {}, {}
    cc_bad, bc_err = {}, {}
    for lb in lbs:
        # "EB" = EDGE_ONLY + BLOCKED (EdgeBlocking, blocking.py:78-186), "EDGE" = EDGE_ONLY,
        # "HYBRID" = BC only: PUSH+ETWC below 1% of V, PULL+BITMAP above (CC takes no hybrid)
        if lb == "HYBRID":
            hy = gg.HybridSchedule(threshold=args.bc_theta,
                                   s1=gg.Schedule(direction="PUSH", load_balance="ETWC"),
                                   s2=gg.Schedule(direction="PULL", pull_frontier_repr="BITMAP",
                                                  frontier_creation="UNFUSED_BITMAP"))
            progh = gg.ScheduleProgram({"s0:s1": hy})
            gg.bc(g, bc_sources[:1], progh, out=scores)
            r, ms_bc = _bc_timed(gg, g, bc_sources, progh, scores)
            bc_res[lb] = {"ms": ms_bc, "rounds": r.stats.rounds,
                          "edges_traversed": r.stats.edges_traversed}
            bc_err[lb] = _rel_err(scores.cpu().numpy(), want_bc, bc_floor)
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
        for _ in range(max(1, min(args.steps, 5))):
            r = gg.cc_soman(g, prog, out=labels)
            ms.append(r.stats.kernel_ms)
            st = r.stats
        m = statistics.median(ms)
        cc_res[lb] = {"ms": m, "rounds": st.rounds, "edges_traversed": st.edges_traversed,
                      "gteps": st.edges_traversed / (m * 1e-3) / 1e9,
                      "frac": ((4.0 * A + 16.0 * V) * st.rounds / (m * 1e-3) / 1e9) / peak}
        cc_bad[lb] = int(np.count_nonzero(labels.cpu().numpy() != want_cc))
        if lb in ("EB", "EDGE") or getattr(args, "no_bc", False):  # frontier traversals: EDGE_ONLY would scan every arc per level
            continue
        gg.bc(g, bc_sources[:1], prog, out=scores)
        r, ms_bc = _bc_timed(gg, g, bc_sources, prog, scores)
        bc_res[lb] = {"ms": ms_bc, "rounds": r.stats.rounds,
                      "edges_traversed": r.stats.edges_traversed}
        bc_err[lb] = _rel_err(scores.cpu().numpy(), want_bc, bc_floor)
    m_c = [int(deg[want_cc == want_cc[s]].sum()) // 2 for s in bc_sources]
    for lb in bc_res:
        bc_res[lb]["gteps"] = 2.0 * sum(m_c) / (bc_res[lb]["ms"] * 1e-3) / 1e9
    parity = {"vs": "oracle.cc_par (canonical min labels) / oracle.bc_par (f64)",
              "cc_label_mismatches": cc_bad, "bc_max_rel_err": bc_err,
              "bc_tolerance": 1e-5, "bc_rel_err_floor": bc_floor,
              "ok": (all(v == 0 for v in cc_bad.values())
                     and all(v <= 1e-5 for v in bc_err.values()))}

    head = next(lb for lb in lbs if lb != "HYBRID")  # the headline is a CC run
    prog = gg.ScheduleProgram({"s0:s1": gg.Schedule(direction="PUSH", load_balance=head)
                               if head not in ("EB", "EDGE") else
                               gg.Schedule(load_balance="EDGE_ONLY", blocking=head == "EB")})
    # e2e: pinned host COO -> Graph.from_coo (symmetric) -> CC -> labels on host
    g.close()
    (a, sh), (b_, dh) = _pinned(s_h, d_h)
    out_h = _pinned(np.empty(V, np.int32))[0][1]

    def e2e_step():
        ge = gg.Graph.from_coo(V, sh, dh, symmetric=True)
        r = gg.cc_soman(ge, prog, out=out_h)
        ge.close()
        return r.stats

    e2e_step()
    _sync()
    t0 = time.perf_counter()
    for _ in range(3):
        st = e2e_step()
    e2e_s = (time.perf_counter() - t0) / 3
    parity["e2e_ok"] = bool(np.array_equal(out_h, want_cc))
    ms = cc_res[head]["ms"]
    cpu_cc = A * cpu_cc_rounds / cpu_cc_s / 1e9
    return {"value": cc_res[head]["gteps"], "ms_per_step": ms, "steps": max(1, min(args.steps, 5)),
            "config": {"workload": "cc_bc_kron%d_ef16_sym" % scale, "V": V, "arcs": A,
                       "coo_order": "by source (edge-list order; matters for EDGE_ONLY/EB only)",
                       "headline": "CC %s (GTEPS = A x hooking rounds / time)" % head,
                       "cc": cc_res, "bc": bc_res, "bc_sources": bc_sources,
                       "bc_m_c": m_c, "generate_s": gen_s,
                       "relabel_prep_ms": relabel_ms,
                       "relabel": "degree-descending copy (GG_RELABEL=%s)"
                                  % os.environ.get("GG_RELABEL", "default: on for V >= 2^20")},
            "roofline": dict(_roof((4.0 * A + 16.0 * V) * cc_res[head]["rounds"], ms, peak),
                             note="B_alg = (4*A + 16*V) per hooking round (SURVEY 8d)"),
            "e2e": {"value": st.edges_traversed / e2e_s / 1e9, "unit": "GTEPS",
                    "h2d_bytes_per_step": 8 * A, "d2h_bytes_per_step": 4 * V,
                    "s_per_step": e2e_s,
                    "includes": "Graph.from_coo of the symmetric COO from pinned host memory, "
                                "CC %s, labels to host" % head},
            "cpu_baseline": {"value": cpu_cc, "unit": "GTEPS", "cores": _threads(),
                             "kind": "port",
                             "sample": "oracle.c or_cc_par (parallel hook + pointer jumping) on "
                                       "the full C4 graph: %d rounds in %.1f s; BC: "
                                       "or_bc_par %d sources in %.1f s = %.2f GTEPS"
                                       % (cpu_cc_rounds, cpu_cc_s, len(bc_sources), cpu_bc_s,
                                          2.0 * sum(m_c) / cpu_bc_s / 1e9)},
            "parity": parity, "dtype": "int32"}


def run(args, peak, peak_kind):
    import paper_2012_07990_b200 as gg
    import torch
    torch.cuda.set_device(0)
    fn = {"c1": pagerank_c1, "c2": bfs_c2, "c3": sssp_c3, "c4": cc_bc_c4}[args.config]
    line = fn(gg, args, peak)
    line["roofline"]["peak_kind"] = peak_kind
    return line


if __name__ == "__main__":
    raise SystemExit("run through bench.py --config c1|c2|c3|c4")
