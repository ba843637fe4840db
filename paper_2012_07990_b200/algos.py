"""The five algorithms on the device (reference algos.py).

Same signatures, label bindings ("s0" loop / "s0:s1" apply), defaults and
errors as the reference; every traversal runs in libgg.so.  Each call is one
C-ABI call: the round loop, hybrid switch, bucket queue and loop fusion run
natively (fused loops as one cooperative launch).
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import binding_pod
from .graphio import Graph, symmetrize_coo
from .priority import UNREACHED
from .runtime import ExecConfig, RunStats
from .sched import (PUSH, HybridSchedule, Schedule, ScheduleError, ScheduleProgram,
                    validate, validate_hybrid)

ALGO_NAMES = ("bfs", "pagerank", "sssp", "cc", "bc")

ALGO_LABELS = {
    "bfs": {"s0": "iteration loop (kernel fusion)", "s0:s1": "edge apply"},
    "pagerank": {"s0": "iteration loop (kernel fusion)", "s0:s1": "edge apply"},
    "sssp": {"s0": "iteration loop (kernel fusion)", "s0:s1": "relax apply (delta)"},
    "cc": {"s0": "iteration loop (kernel fusion)", "s0:s1": "hook apply"},
    "bc": {"s0": "per-source loop (fusion rejected)", "s0:s1": "forward apply"},
}

HYBRID_CAPABLE = ("bfs", "bc")


class AlgoResult:
    """``(values, stats)`` as the reference's AlgoResult (algos.py:35-38).

    ``array`` is the result buffer (numpy or a CUDA tensor); ``values`` -- the
    reference's Python list -- is built from it on first access, so callers
    that only use the array (the bench's 134M-vertex runs) never pay for a
    list conversion.  ``values`` is None for device-resident results.
    """

    __slots__ = ("_values", "_make", "stats", "array")

    def __init__(self, values, stats, array=None):
        self._values, self._make = (None, values) if callable(values) else (values, None)
        self.stats = stats
        self.array = array

    @property
    def values(self):
        if self._make is not None:
            self._values, self._make = self._make(), None
        return self._values

    def __repr__(self):
        return "AlgoResult(values=%s, stats=%r)" % (
            "<%d values>" % len(self.array) if self.array is not None else self.values, self.stats)


@dataclass
class _Plan:
    apply_schedule: object
    fusion: bool


def default_schedule(algo):
    """PageRank defaults to EDGE_ONLY, everything else to Schedule() (algos.py:47-50)."""
    if algo == "pagerank":
        return Schedule(load_balance="EDGE_ONLY")
    return Schedule()


def _plan(program, algo):
    """Label validation and binding resolution (algos.py:53-76)."""
    program = program or ScheduleProgram()
    program.validate_bound_labels(set(ALGO_LABELS[algo]))
    loop = program.binding("s0")
    if isinstance(loop, HybridSchedule):
        raise ScheduleError("loop label 's0' takes a SimpleGPUSchedule")
    bound = program.binding("s0:s1")
    if bound is None:
        bound = default_schedule(algo)
    if isinstance(bound, HybridSchedule):
        if algo not in HYBRID_CAPABLE:
            raise ScheduleError("label 's0:s1' of %s takes a SimpleGPUSchedule (hybrid "
                                "direction switching applies to %s)"
                                % (algo, "/".join(HYBRID_CAPABLE)))
        if not bound.resolved():
            raise ScheduleError("unresolved threshold %r; supply --sched-arg" % bound.threshold)
        problems = validate_hybrid(bound)
    else:
        problems = validate(bound)
    if problems:
        raise ScheduleError("invalid schedule for %s: %s" % (algo, "; ".join(problems)))
    fusion = bool(loop.kernel_fusion) if loop is not None else False
    return _Plan(bound, fusion)


def _check_source(g, source):
    if not 0 <= source < g.num_vertices:
        raise ValueError("invalid source %d for graph with %d vertices"
                         % (source, g.num_vertices))


def _exec(exec_cfg):
    cfg = exec_cfg or ExecConfig()
    return cfg.to_pod()


def _out(n, dtype, out):
    """Result buffer: caller-provided (host numpy or CUDA tensor) or fresh numpy."""
    if out is not None:
        return out
    return np.empty(n, dtype=dtype)


def _values(arr):
    """Deferred list of a host result (None for device buffers)."""
    return (lambda: arr.tolist()) if isinstance(arr, np.ndarray) else None


# ---------------------------------------------------------------------------
# BFS
# ---------------------------------------------------------------------------
def bfs(g, source, program=None, exec_cfg=None, out=None):
    """Parent array of a BFS; -1 unreached (algos.py:101-135)."""
    _check_source(g, source)
    plan = _plan(program, "bfs")
    pod, cfg = binding_pod(plan.apply_schedule), _exec(exec_cfg)
    parents = _out(g.num_vertices, np.int32, out)
    st = _lib.new_stats()
    _lib.call("gg_bfs", g.handle, int(source), C.byref(pod), 1 if plan.fusion else 0,
              C.byref(cfg), _lib.ptr(parents), C.byref(st))
    return AlgoResult(_values(parents), RunStats.from_pod(st), parents)


def bfs_levels(parents):
    """Hop distance implied by a BFS parent forest (-1 unreached), vectorised
    pointer doubling (same result as algos.py:138-156)."""
    p = np.asarray(parents, dtype=np.int64)
    n = len(p)
    level = np.full(n, -1, dtype=np.int64)
    if n == 0:
        return []
    reached = p >= 0
    anc = np.where(reached, p, np.arange(n))
    dist = np.where(reached & (p != np.arange(n)), 1, 0).astype(np.int64)
    # doubling: dist to root along parent pointers
    for _ in range(64):
        nxt = anc[anc]
        if np.array_equal(nxt, anc):
            break
        dist = dist + dist[anc]
        anc = nxt
    level[reached] = dist[reached]
    return level.tolist()


# ---------------------------------------------------------------------------
# PageRank
# ---------------------------------------------------------------------------
def pagerank(g, program=None, exec_cfg=None, max_iters=100, tolerance=1e-9, damping=0.85,
             on_iteration=None, out=None, contrib_fp32=False):
    """Power iteration, uniform teleport and dangling redistribution
    (algos.py:163-208).  ``on_iteration`` is honoured by running one
    iteration per device call and re-seeding is not needed: it receives the
    rank vector after each iteration (host copy; slow path for tests)."""
    if g.num_vertices == 0:
        raise ValueError("empty graph")
    plan = _plan(program, "pagerank")
    pod, cfg = binding_pod(plan.apply_schedule), _exec(exec_cfg)
    if on_iteration is not None:
        return _pagerank_observed(g, plan, pod, cfg, max_iters, tolerance, damping,
                                  on_iteration)
    ranks = _out(g.num_vertices, np.float64, out)
    st = _lib.new_stats()
    _lib.call("gg_pagerank_ex", g.handle, C.byref(pod), 1 if plan.fusion else 0, C.byref(cfg),
              int(max_iters), float(tolerance), float(damping), 1 if contrib_fp32 else 0,
              _lib.ptr(ranks), C.byref(st))
    return AlgoResult(_values(ranks), RunStats.from_pod(st), ranks)


def _pagerank_observed(g, plan, pod, cfg, max_iters, tolerance, damping, on_iteration):
    # Observing every iteration: one device iteration per call, each resumed
    # from the previous ranks (gg_pagerank_resume; the rank vector is the
    # whole state between iterations), so n iterations cost n, not n(n+1)/2.
    # Stop test before each body with L1 = inf initially (algos.py:178,
    # :204-205; engine.py:659-661).
    V = g.num_vertices
    prev = np.full(V, 1.0 / V, np.float64)
    ranks = np.empty(V, np.float64)
    total = RunStats()
    it, l1 = 0, math.inf
    while not (it >= max_iters or l1 < tolerance):
        st = _lib.new_stats()
        _lib.call("gg_pagerank_resume", g.handle, C.byref(pod), 1 if plan.fusion else 0,
                  C.byref(cfg), 1, 0.0, float(damping), _lib.ptr(prev), _lib.ptr(ranks), C.byref(st))
        one = RunStats.from_pod(st)
        for f in ("dispatch_count", "rounds", "edges_traversed", "frontier_conversions",
                  "frontier_allocations", "reused_frontiers", "creation_passes", "kernel_ms",
                  "wall_ms", "gpu_launches", "edge_ms", "edge_launches", "top_ms", "top_launches"):
            setattr(total, f, getattr(total, f) + getattr(one, f))
        total.direction_log += one.direction_log
        it += 1
        l1 = float(np.abs(ranks - prev).sum())
        on_iteration(ranks.tolist())
        prev, ranks = ranks, prev
    if plan.fusion:
        total.dispatch_count = 1  # the whole loop is one fused dispatch (runtime.py:194-209)
    return AlgoResult(prev.tolist(), total, prev)


# ---------------------------------------------------------------------------
# SSSP (delta-stepping)
# ---------------------------------------------------------------------------
def sssp_delta(g, source, program=None, exec_cfg=None, out=None):
    """Exact distances by delta-stepping; inf for unreachable (algos.py:215-247).
    PUSH is forced; the bucket width is the apply schedule's delta."""
    _check_source(g, source)
    if not g.weighted:
        raise ValueError("sssp needs edge weights (load weighted or inject random weights)")
    plan = _plan(program, "sssp")
    s = plan.apply_schedule.copy()
    s.direction = PUSH
    pod, cfg = binding_pod(s), _exec(exec_cfg)
    dist = _out(g.num_vertices, np.uint64, out)
    st = _lib.new_stats()
    _lib.call("gg_sssp_delta", g.handle, int(source), C.byref(pod), 1 if plan.fusion else 0,
              C.byref(cfg), _lib.ptr(dist), C.byref(st))
    values = None
    if isinstance(dist, np.ndarray):
        values = lambda: [math.inf if d == UNREACHED else int(d) for d in dist.tolist()]  # noqa: E731
    return AlgoResult(values, RunStats.from_pod(st), dist)


# ---------------------------------------------------------------------------
# Connected components
# ---------------------------------------------------------------------------
def cc_soman(g, program=None, exec_cfg=None, out=None):
    """Hook + pointer-jump to fixpoint; labels canonicalised to the component's
    minimum vertex id (algos.py:267-307)."""
    if not g.symmetric:
        warnings.warn("cc expects a symmetric graph; symmetrizing a copy")
        s, d, w, _ = symmetrize_coo(g.coo_src, g.coo_dst, g.coo_weights)
        g = Graph.from_coo(g.num_vertices, s, d, w, symmetric=True, device=g.device)
    plan = _plan(program, "cc")
    pod, cfg = binding_pod(plan.apply_schedule), _exec(exec_cfg)
    labels = _out(g.num_vertices, np.int32, out)
    st = _lib.new_stats()
    _lib.call("gg_cc", g.handle, C.byref(pod), 1 if plan.fusion else 0, C.byref(cfg),
              _lib.ptr(labels), C.byref(st))
    return AlgoResult(_values(labels), RunStats.from_pod(st), labels)


# ---------------------------------------------------------------------------
# Betweenness centrality
# ---------------------------------------------------------------------------
def bc(g, sources, program=None, exec_cfg=None, out=None):
    """Brandes restricted to ``sources``, halved (algos.py:314-395)."""
    if not len(sources):
        raise ValueError("sources must be a non-empty list")
    for s0 in sources:
        _check_source(g, s0)
    if not g.symmetric:
        raise ValueError("bc assumes a symmetric graph; load with symmetrize")
    plan = _plan(program, "bc")
    if plan.fusion:
        raise ScheduleError("kernel fusion rejected for bc: the loop body retains per-round "
                            "frontiers (not reusable)")
    pod, cfg = binding_pod(plan.apply_schedule), _exec(exec_cfg)
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64))
    scores = _out(g.num_vertices, np.float64, out)
    st = _lib.new_stats()
    _lib.call("gg_bc", g.handle, _lib.ptr(src), len(src), C.byref(pod), C.byref(cfg),
              _lib.ptr(scores), C.byref(st))
    return AlgoResult(_values(scores), RunStats.from_pod(st), scores)
