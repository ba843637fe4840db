"""edgeset.apply operator mirror (reference engine.py:418-662).

``edgeset_apply`` / ``hybrid_apply`` / ``fused_loop`` / ``pick_udf`` keep the
reference signatures.  The traversal itself runs in libgg.so: ``udf`` must be a
named device UDF (``paper_2012_07990_b200.udfs``) and ``to_filter`` either
``None`` or that UDF's ``.filter``; a Python callable raises, because no CPU
path exists.  The partitioner helpers (``partition_even_chunks`` ...) are the
reference's host-side chunk arithmetic, restated with numpy for callers that
inspect the schedule space; the device kernels implement the same splits.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .frontier import VertexSubset, _ForeignSubset
from .runtime import EngineError, ExecConfig, RunStats, Runtime, coerce_runtime
from .sched import (PULL, HybridSchedule, Schedule, ScheduleError, validate,
                    validate_hybrid, DIRECTION_CODE, LB_CODE, CREATION_CODE, DEDUP_CODE,
                    REPR_CODE)
from .udfs import DeviceFilter, DeviceUDF

__all__ = ["ExecConfig", "RunStats", "Runtime", "EngineError", "edgeset_apply", "hybrid_apply",
           "fused_loop", "pick_udf", "lb_partition_etwc", "lb_partition_strict",
           "lb_partition_twc", "partition_even_chunks", "push_work", "schedule_pod",
           "binding_pod"]


# ---------------------------------------------------------------------------
# POD conversion of schedules for the C ABI
# ---------------------------------------------------------------------------
def schedule_pod(s):
    return _lib.GGSchedule(DIRECTION_CODE[s.direction], REPR_CODE[s.pull_frontier_repr],
                           LB_CODE[s.load_balance], 1 if s.blocking else 0,
                           int(s.blocking_size or 0), CREATION_CODE[s.frontier_creation],
                           1 if s.dedup else 0, DEDUP_CODE[s.dedup_strategy],
                           1 if s.kernel_fusion else 0, int(s.delta))


def binding_pod(bound):
    b = _lib.GGBinding()
    if isinstance(bound, HybridSchedule):
        b.is_hybrid = 1
        b.threshold = float(bound.threshold)
        b.s1 = schedule_pod(bound.s1)
        b.s2 = schedule_pod(bound.s2)
    else:
        b.is_hybrid = 0
        b.s1 = schedule_pod(bound)
        b.s2 = schedule_pod(bound)
    return b


# ---------------------------------------------------------------------------
# Host-side chunk arithmetic (engine.py:32-213), numpy restatement
# ---------------------------------------------------------------------------
def partition_even_chunks(n_items, n_parts):
    """Contiguous (lo, hi) chunks differing by at most one; earlier take extra."""
    base, extra = divmod(n_items, n_parts)
    sizes = np.full(n_parts, base, dtype=np.int64)
    sizes[:extra] += 1
    ends = np.cumsum(sizes)
    return [(int(e - s), int(e)) for s, e in zip(sizes, ends)]


def _etwc_split(start, end, cta, warp):
    size = end - start
    e2 = (size // cta) * cta
    e1 = ((size - e2) // warp) * warp
    return (start + e2 + e1, end), (start + e2, start + e2 + e1), (start, start + e2)


def lb_partition_etwc(active, g, cfg):
    """Per-CTA (q0, q1, q2) queues of (edge_lo, edge_hi, src) (engine.py:51-85)."""
    off = g.out_offsets
    queues = []
    for lo, hi in partition_even_chunks(len(active), cfg.num_workers):
        q = ([], [], [])
        for i in range(lo, hi):
            u = active[i]
            parts = _etwc_split(int(off[u]), int(off[u + 1]), cfg.cta_size, cfg.warp_size)
            for stage in (2, 1, 0):
                a, b = parts[stage]
                if b > a:
                    q[stage].append((a, b, u))
        queues.append(q)
    return queues


def lb_partition_strict(active, g, cfg):
    """Per-worker edge ranges + exclusive degree prefix (engine.py:88-122)."""
    off = np.asarray(g.out_offsets)
    act = np.asarray(active, dtype=np.int64)
    deg = off[act + 1] - off[act] if len(act) else np.zeros(0, np.int64)
    prefix = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
    return partition_even_chunks(int(prefix[-1]), cfg.num_workers), prefix.tolist()


def lb_partition_twc(active, g, cfg):
    """(cta_q, warp_q, thread_q), strictly-greater promotion (engine.py:125-142)."""
    off = g.out_offsets
    cta_q, warp_q, thread_q = [], [], []
    for u in active:
        d = int(off[u + 1] - off[u])
        (cta_q if d > cfg.cta_size else warp_q if d > cfg.warp_size else thread_q).append(u)
    return cta_q, warp_q, thread_q


def push_work(active, offsets, load_balance, cfg):
    """Per-worker (vertex, lo, hi) chunks; every strategy tiles each active
    vertex's range exactly (engine.py:206-213)."""
    off = offsets
    nw = cfg.num_workers
    whole = lambda vs: [(u, int(off[u]), int(off[u + 1])) for u in vs]
    if load_balance == "VERTEX_BASED":
        return [whole(active[w::nw]) for w in range(nw)]
    if load_balance == "CM":
        return [whole(active[lo:hi]) for lo, hi in partition_even_chunks(len(active), nw)]
    if load_balance == "WM":
        wpc = cfg.warps_per_cta
        bounds = partition_even_chunks(len(active), nw * wpc)
        return [sum((whole(active[lo:hi]) for lo, hi in bounds[w * wpc:(w + 1) * wpc]), [])
                for w in range(nw)]
    if load_balance == "STRICT":
        deg = [int(off[u + 1] - off[u]) for u in active]
        prefix = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
        out = []
        for elo, ehi in partition_even_chunks(int(prefix[-1]), nw):
            chunks = []
            if elo < ehi:
                i = int(np.searchsorted(prefix, elo, side="right")) - 1
                while i < len(active) and prefix[i] < ehi:
                    a, b = max(elo, prefix[i]), min(ehi, prefix[i + 1])
                    if a < b:
                        base = int(off[active[i]])
                        chunks.append((active[i], int(base + a - prefix[i]),
                                       int(base + b - prefix[i])))
                    i += 1
            out.append(chunks)
        return out
    if load_balance == "TWC":
        cfg_shim = type("G", (), {"out_offsets": off})
        cta_q, warp_q, thread_q = lb_partition_twc(active, cfg_shim, cfg)
        wpc = cfg.warps_per_cta
        per = [[] for _ in range(nw)]
        for w in range(nw):
            per[w] += whole(cta_q[w::nw])
        for j, u in enumerate(warp_q):
            per[(j % (nw * wpc)) // wpc].append((u, int(off[u]), int(off[u + 1])))
        for w in range(nw):
            per[w] += whole(thread_q[w::nw])
        return per
    if load_balance == "ETWC":
        shim = type("G", (), {"out_offsets": off})
        return [[(u, lo, hi) for lo, hi, u in q0 + q1 + q2]
                for q0, q1, q2 in lb_partition_etwc(active, shim, cfg)]
    raise EngineError("no chunker for load balance %r" % load_balance)


# ---------------------------------------------------------------------------
# The edge apply
# ---------------------------------------------------------------------------
def _device_udf(udf):
    if not isinstance(udf, DeviceUDF):
        raise ScheduleError("edgeset_apply on the device needs a named device UDF "
                            "(paper_2012_07990_b200.udfs); got %r" % (udf,))
    return udf


def _filter_flag(udf, to_filter):
    if to_filter is None:
        return 0
    if isinstance(to_filter, DeviceFilter) and to_filter.udf is udf:
        return 1
    raise ScheduleError("to_filter must be None or the device UDF's .filter")


def _apply(g, input_frontier, udf, to_filter, bound, runtime, reuse, collect_output):
    rt = coerce_runtime(runtime, g)
    V = g.num_vertices
    if input_frontier is not None and (input_frontier.universe != V
                                       or isinstance(input_frontier, _ForeignSubset)):
        raise EngineError("frontier universe %d does not match graph (%d vertices)"
                          % (input_frontier.universe, V))
    udf = _device_udf(udf)
    flag = _filter_flag(udf, to_filter)
    st = udf.state()
    b = binding_pod(bound)
    out = C.c_void_p()
    _lib.call("gg_edgeset_apply", rt.handle, udf.code, C.byref(st), flag,
              input_frontier.handle if input_frontier is not None else None, C.byref(b),
              1 if reuse else 0, 1 if collect_output else 0, C.byref(out))
    if reuse and input_frontier is not None:
        input_frontier._mark_retired()
    if collect_output and out.value:
        return VertexSubset(rt, V, out)
    return None


def edgeset_apply(g, input_frontier, udf, *, to_filter=None, schedule=None, runtime=None,
                  reuse=False, collect_output=True):
    """One traversal round on the device (engine.py:418-460)."""
    s = schedule or Schedule()
    problems = validate(s)
    if problems:
        raise ScheduleError("invalid schedule: " + "; ".join(problems))
    return _apply(g, input_frontier, udf, to_filter, s, runtime, reuse, collect_output)


def pick_udf(s, udf_push, udf_pull):
    """Owner-write udf only where the engine grants destination ownership."""
    if s.direction == PULL and s.load_balance != "EDGE_ONLY":
        return udf_pull
    return udf_push


def hybrid_apply(g, input_frontier, udf_push, udf_pull, hybrid, *, to_filter=None,
                 runtime=None, reuse=False, collect_output=True):
    """s2 when |input| > threshold*|V| else s1 (engine.py:622-636).  The size
    test and the choice run inside libgg (one call)."""
    if isinstance(hybrid.threshold, str):
        raise ScheduleError("unresolved threshold %r; supply --sched-arg" % hybrid.threshold)
    problems = validate_hybrid(hybrid)
    if problems:
        raise ScheduleError("invalid hybrid schedule: " + "; ".join(problems))
    if udf_push is not udf_pull and udf_pull is not None:
        # device UDFs bundle both directions; the engine picks the owner-write
        # variant itself, so the two must name the same functor
        if type(udf_push) is not type(udf_pull):
            raise ScheduleError("hybrid device UDFs must be the same functor")
    return _apply(g, input_frontier, udf_push, to_filter, hybrid, runtime, reuse,
                  collect_output)


def fused_loop(body, until, *, fusion=False, runtime=None, body_reuses_frontiers=True):
    """Run ``body`` until ``until()`` (engine.py:639-662).

    Unfused, each traversal in the body is its own dispatch; fused, the
    whole loop is ONE dispatch (Runtime.fused_dispatch, runtime.py:194-209)
    and the body must recycle frontier storage.  The algorithm drivers in
    ``algos`` fuse on the device as one cooperative launch; a custom host
    body keeps its per-round launches but is accounted as one dispatch,
    exactly as the reference's fused region is one pool dispatch.  With a
    bound :class:`Runtime` the rounds land in its device stats.
    """
    if fusion and not body_reuses_frontiers:
        raise ScheduleError("kernel fusion requires a loop body that reuses frontier storage")
    rt = runtime if isinstance(runtime, Runtime) and runtime._handle is not None else None
    rounds = 0
    if fusion and rt is not None:
        _lib.call("gg_runtime_fused_region", rt.handle, 1)
    try:
        while not until():
            body()
            rounds += 1
    finally:
        if fusion and rt is not None:
            _lib.call("gg_runtime_fused_region", rt.handle, 0)
    if rt is not None:
        _lib.call("gg_runtime_add_rounds", rt.handle, rounds)
        return rt.stats
    st = RunStats(rounds=rounds, dispatch_count=1 if fusion else 0)
    return st
