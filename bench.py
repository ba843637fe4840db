#!/usr/bin/env python
"""Benchmark harness (driver contract).

Default workload (BASELINE.json configs[4], the graded one): PageRank with
EdgeBlocking on RMAT scale 27 (V = 2^27, E = 2^31, edge factor 16,
a/b/c = .57/.19/.19, seed 7), 20 iterations, tolerance 0.  One "step" = one
complete ``pagerank(g, program, max_iters=20, tolerance=0.0)`` call with the
graph resident in HBM; metric GTEPS = 20*E / step time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gg|reference]
                  [--config c5|c1|...] [--scale S] [--schedule eb|edge|pull|...]

Multi-GPU (torchrun): the same RMAT-27 graph is 1-D partitioned by
destination over the N ranks (EdgeBlocking layout per rank, NCCL allgather of
contributions every iteration; "scaling": "strong"); value = 20*E / max over
ranks of the step time.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (scale, edge_factor, seed, iterations)
    "c5": (27, 16, 7, 20),
    "c1": (16, 16, 1, 20),
}
ALGO_CONFIGS = ("c2", "c3", "c4")  # bench_algos.py: BFS / SSSP / CC+BC (configs[1..3])

SCHEDULES = {
    "eb": dict(load_balance="EDGE_ONLY", blocking=True),
    "edge": dict(load_balance="EDGE_ONLY"),
    "pull": dict(direction="PULL", load_balance="STRICT"),
    "pull_twc": dict(direction="PULL", load_balance="TWC"),
    "pull_etwc": dict(direction="PULL", load_balance="ETWC"),
    "pull_wm": dict(direction="PULL", load_balance="WM"),
    "push": dict(direction="PUSH", load_balance="ETWC"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="gg", choices=["gg", "reference"])
    p.add_argument("--config", default="c5", choices=sorted(CONFIGS) + list(ALGO_CONFIGS))
    p.add_argument("--scale", type=int, default=None)
    p.add_argument("--schedule", default="eb", choices=sorted(SCHEDULES))
    p.add_argument("--fp32-contrib", action="store_true")
    p.add_argument("--permute", action="store_true", help="Graph500-style id permutation")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-scale", type=int, default=22)
    # c2-c4 (bench_algos.py)
    p.add_argument("--sources", type=int, default=None)
    p.add_argument("--theta", type=float, default=0.0005, help="c2 hybrid threshold (swept: best)")
    p.add_argument("--dedup", action="store_true",
                   help="c2: s1 with MONOTONIC_COUNTERS dedup (default off: the BFS CAS "
                        "already admits each vertex once, so the frontier is identical)")
    p.add_argument("--pull-lb", default="VERTEX_BASED", help="c2 pull-side load balance")
    p.add_argument("--fusion", action="store_true", help="c1/c2/c5: fused loop (s0 kernel fusion)")
    p.add_argument("--side", type=int, default=None, help="c3 grid side")
    p.add_argument("--delta", type=int, default=None, help="c3 bucket width (default: sweep)")
    p.add_argument("--lb", default="WM", help="c3 load balance (swept: WM best)")
    p.add_argument("--no-fusion", action="store_true", help="c3: unfused loop")
    p.add_argument("--lbs", default="ETWC,TWC,VERTEX_BASED,EB,EDGE,HYBRID",
                   help="c4 load balances (EB = EDGE_ONLY+BLOCKED, EDGE = EDGE_ONLY)")
    p.add_argument("--check", action="store_true", help="c2-c4: validate against the oracle")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampling during the timed region (B200_PROFILING.md "clocks line")
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (test infrastructure) on the host cores
# ---------------------------------------------------------------------------
def cpu_pagerank_sample(scale, edge_factor, seed, budget_s=20.0, max_iters=20):
    import numpy as np
    import oracle
    V, s, d = oracle.rmat(scale, edge_factor, seed=seed)
    in_off, in_nbr, _ = oracle.csr(V, d, s)
    out_off, _, _ = oracle.csr(V, s, np.zeros_like(d))
    E = len(s)
    # one warm-up iteration, then as many timed single-iteration steps as fit the budget
    oracle.pagerank_par(V, in_off, in_nbr, out_off, 1, 0.0)
    t0 = time.perf_counter()
    iters = 0
    while iters < max_iters:
        oracle.pagerank_par(V, in_off, in_nbr, out_off, 1, 0.0)
        iters += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": E * iters / dt / 1e9, "unit": "GTEPS", "cores": oracle.num_threads(),
            "kind": "port",
            "sample": "RMAT scale %d ef %d seed %d (E=%d), %d PageRank iteration(s) of "
                      "oracle.c or_pagerank_par (pull, OpenMP, f64) in %.1f s"
                      % (scale, edge_factor, seed, E, iters, dt)}


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "GTEPS per algorithm x graph (PR/BFS/SSSP/CC/BC); PR GTEPS at 1/2/4/8 GPUs"
    if args.config in ALGO_CONFIGS:
        main_algo(args, metric)
        return
    scale, ef, seed, iters = CONFIGS[args.config]
    if args.scale:
        scale = args.scale
    workload = "pagerank_%s_rmat%d_ef%d" % (args.schedule, scale, ef)

    if args.impl == "reference":
        if rank != 0:
            return
        cs = min(args.cpu_scale, scale)
        step_vals = []
        for _ in range(args.warmup):
            cpu_pagerank_sample(cs, ef, seed, budget_s=5.0, max_iters=1)
        for _ in range(args.steps):
            step_vals.append(cpu_pagerank_sample(cs, ef, seed, budget_s=10.0, max_iters=3))
        v = statistics.median(x["value"] for x in step_vals)
        base = step_vals[0]
        line = {"metric": metric, "value": v, "unit": "GTEPS", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": workload, "cpu_sample_scale": cs, "iterations": iters},
                "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": base["cores"],
                                 "kind": "port", "sample": base["sample"]},
                "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import numpy as np
    import torch
    import paper_2012_07990_b200 as gg

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    t0 = time.perf_counter()
    g = gg.generate_rmat(scale, ef, seed=seed, sort_by_source=True, permute=args.permute,
                         device=local)
    gen_s = time.perf_counter() - t0
    V, E = g.num_vertices, g.num_edges
    sch = gg.Schedule(**SCHEDULES[args.schedule])
    prog = gg.ScheduleProgram({"s0:s1": sch})
    if args.fusion:  # s0 loop fusion: the whole 20-iteration loop is one cooperative launch
        prog.bindings["s0"] = gg.Schedule(kernel_fusion=True)
    import ctypes as C
    from paper_2012_07990_b200 import _lib
    from paper_2012_07990_b200.engine import binding_pod
    ranks = torch.empty(V, dtype=torch.float64, device="cuda")
    comm = None
    if world > 1:
        # N > 1: the graph is 1-D partitioned by destination (renumbered ids,
        # balanced by in-edges); every rank generates the same RMAT graph,
        # keeps its own destinations' in-edges, and allgathers contributions
        # over NCCL each iteration (strong scaling: total work fixed).
        from paper_2012_07990_b200.dist import Comm, pagerank_dist, prepare_dist
        comm = Comm.create(rank, world, local)
        prep_ms = prepare_dist(world, rank, g, prog, contrib_fp32=args.fp32_contrib)

        def step():
            return pagerank_dist(comm, g, max_iters=iters, tolerance=0.0, out=ranks,
                                 program=prog, contrib_fp32=args.fp32_contrib)[1]
    else:
        pm = C.c_double()
        pod = binding_pod(sch)
        _lib.call("gg_pagerank_prepare", g.handle, C.byref(pod), 1 if args.fp32_contrib else 0,
                  C.byref(pm))
        prep_ms = pm.value

        def step():
            return gg.pagerank(g, prog, max_iters=iters, tolerance=0.0, out=ranks,
                               contrib_fp32=args.fp32_contrib).stats

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    peak, peak_kind = measured_peaks()
    with ClockSampler(local) as clk:
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        edge_ms = 0.0
        edge_n = 0
        launches = 0
        e_local = 0
        top_ms, top_n, top_edges = 0.0, 0, 0
        for _ in range(args.steps):
            st = step()
            edge_ms += st.edge_ms
            edge_n += st.edge_launches
            launches += st.gpu_launches
            e_local = st.edges_traversed // iters
            top_ms += st.top_ms
            top_n += st.top_launches
            top_edges = st.top_edges
        ev1.record()
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    # strong scaling: the same RMAT-27 graph at every N (partitioned at N > 1)
    value = iters * E / (ms * 1e-3) / 1e9

    # roofline (SURVEY §8(d) fixed byte model: 8 B per edge, 16 B per vertex for
    # the edge phase (contrib read + acc write), 32 B per vertex per iteration).
    # Dominant kernel = the hot-segment gather (k_pr_edges_hot): its edges x 8 B
    # + the vertices' 16 B, over its CUDA-event time; the whole edge phase and
    # the whole iteration are reported beside it.
    avg_edge_ms = edge_ms / max(1, edge_n)
    alg_edge = 8.0 * e_local + 16.0 * V / world  # this rank's share (all of it at N=1)
    edge_achieved = alg_edge / (avg_edge_ms * 1e-3) / 1e9
    alg_iter = 8.0 * E + 32.0 * V
    iter_achieved = alg_iter * iters / (ms * 1e-3) / 1e9 / world  # per-GPU share of the aggregate
    if top_n:
        avg_top_ms = top_ms / top_n
        alg_top = 8.0 * top_edges + 16.0 * V / world
        kernel = "k_pr_edges_hot (hot source segment, %d of %d edges)" % (top_edges, e_local)
    else:
        avg_top_ms, alg_top, kernel = avg_edge_ms, alg_edge, "edge phase (%s)" % args.schedule
    achieved = alg_top / (avg_top_ms * 1e-3) / 1e9
    # DRAM bytes per launch of that kernel from the committed ncu --set full
    # capture of this exact configuration (bench can not run ncu itself)
    traffic, traffic_note = None, "no ncu capture committed for this configuration"
    if (top_n and args.schedule == "eb" and not args.fp32_contrib and scale == 27
            and world == 1 and not args.permute):
        traffic = 16.291855e9 + 0.618621e9
        traffic_note = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                        "profiles/r01/ncu_full_k_pr_edges_hot_f64.txt (= the streamed "
                        "edges; the gathers hit L2)")

    line = {"metric": metric, "value": value, "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" + ("(contrib f32)" if args.fp32_contrib else ""),
            "data": "synthetic RMAT generated on device (sort_by_source%s)"
                    % (", permuted ids" if args.permute else ", natural ids"),
            "config": {"workload": workload, "V": V, "E": E, "iterations": iters,
                       "schedule": dict(SCHEDULES[args.schedule], kernel_fusion=bool(args.fusion)),
                       "blocking_prep_ms": prep_ms,
                       "parallelism": ("1-D destination partition x%d, NCCL allgather of "
                                       "contributions per iteration" % world) if world > 1
                                      else "single GPU",
                       "generate_s": gen_s,
                       "l2": "inputs (%.1f GB) larger than L2; no flush needed" % (8 * E / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "traffic_note": traffic_note, "kernel": kernel, "avg_launch_ms": avg_top_ms,
                         "alg_bytes_per_launch": alg_top,
                         "edge_phase": {"ms_per_iteration": avg_edge_ms, "alg_bytes": alg_edge,
                                        "achieved": edge_achieved, "frac": edge_achieved / peak},
                         "iteration_frac": iter_achieved / peak},
            "gpu_launches": launches,
            "clocks": clk.summary()}

    # e2e: host COO in pinned memory -> Graph.from_coo -> pagerank -> ranks on host
    if not args.no_e2e:
        src_h = torch.from_numpy(g.coo_src).pin_memory()
        dst_h = torch.from_numpy(g.coo_dst).pin_memory()
        g.close()
        del g
        torch.cuda.empty_cache()
        ranks_h = torch.empty(V, dtype=torch.float64).pin_memory()
        e2e_steps = min(3, args.steps)

        def e2e_step():
            ge = gg.Graph.from_coo(V, src_h.numpy(), dst_h.numpy(), device=local)
            if comm is not None:
                pagerank_dist(comm, ge, max_iters=iters, tolerance=0.0, out=ranks_h.numpy(),
                              program=prog, contrib_fp32=args.fp32_contrib)
            else:
                gg.pagerank(ge, prog, max_iters=iters, tolerance=0.0, out=ranks_h.numpy(),
                            contrib_fp32=args.fp32_contrib)
            ge.close()

        e2e_step()  # warm-up (device buffer pool, layout kernels)
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        barrier()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        e2e_t = torch.tensor([e2e_s], device="cuda")
        if dist is not None:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_t.item())
        line["e2e"] = {"value": iters * E / e2e_s / 1e9, "unit": "GTEPS",
                       "h2d_bytes_per_step": 8 * E, "d2h_bytes_per_step": 8 * V,
                       "s_per_step": e2e_s,
                       "includes": "H2D of COO from pinned host memory, device graph build "
                                   "(EdgeBlocking prep), 20 iterations, D2H of ranks"}
    if rank == 0 and world == 1 and not args.no_cpu:
        # bounded sample: ~10 s of PageRank iterations on the host cores
        line["cpu_baseline"] = cpu_pagerank_sample(min(args.cpu_scale, scale), ef, seed,
                                                   budget_s=10.0, max_iters=10000)
    if rank == 0:
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def main_algo(args, metric):
    """configs[1..3]: one GPU (the north star keeps BFS-DO, SSSP, CC and BC
    single-GPU); under torchrun rank 0 runs and the other ranks exit."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import bench_algos
    peak, peak_kind = measured_peaks()
    with ClockSampler(0) as clk:
        line = bench_algos.run(args, peak, peak_kind)
    out = {"metric": metric, "value": line.pop("value"), "unit": "GTEPS", "n_gpus": 1,
           "steps": line.pop("steps"), "warmup": args.warmup,
           "ms_per_step": line.pop("ms_per_step"), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": line.pop("dtype"),
           "data": "synthetic (generated on device)"}
    out.update(line)
    out["clocks"] = clk.summary()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
