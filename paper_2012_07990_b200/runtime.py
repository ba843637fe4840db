"""Execution substrate mirror (reference runtime.py).

``ExecConfig``/``RunStats``/``EngineError`` keep the reference's fields,
defaults and validation messages (runtime.py:26-67).  ``Runtime`` owns one
device-side ``gg_runtime`` (stats, frontier pool, dedup state) per query, the
way the reference's Runtime is per algorithm call (algos.py:109).
``EdgeContext`` exists for API parity only: a Python callable cannot run per
edge on the device, so named device UDFs (``udfs``) replace it.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import asdict, dataclass, field

from . import _lib

DIRECTION_NAMES = {0: "PUSH", 1: "PULL"}


class EngineError(RuntimeError):
    pass


@dataclass
class ExecConfig:
    """CTA hierarchy shape (runtime.py:26-50).

    On the device ``cta_size`` is the CTA granularity of the ETWC/TWC
    balancers and ``warp_size`` must be 32 (hardware).  ``num_workers`` is
    the reference's host-simulation knob: validated and accepted, the grid is
    always sized to the GPU.  ``deterministic`` makes ``pagerank`` sum in the
    reference's fixed order (runtime.py:167): its ranks are then bitwise the
    reference's for EDGE_ONLY (+ BLOCKED) and PULL schedules (slow: the
    sequential sums run on one thread each).
    """

    num_workers: int = 1
    cta_size: int = 256
    warp_size: int = 32
    deterministic: bool = False

    def validate(self):
        if self.num_workers < 1:
            raise EngineError("num_workers must be >= 1")
        if self.warp_size < 1 or self.cta_size < 1:
            raise EngineError("warp_size and cta_size must be >= 1")
        if self.cta_size % self.warp_size:
            raise EngineError("warp_size must divide cta_size")

    @property
    def warps_per_cta(self):
        return self.cta_size // self.warp_size

    def to_pod(self):
        self.validate()
        return _lib.GGExec(self.num_workers, self.cta_size, self.warp_size,
                           1 if self.deterministic else 0)


@dataclass
class RunStats:
    """Counters of one algorithm run (runtime.py:53-67) + device timings."""

    dispatch_count: int = 0
    rounds: int = 0
    edges_traversed: int = 0
    direction_log: list = field(default_factory=list)
    frontier_conversions: int = 0
    frontier_allocations: int = 0
    reused_frontiers: int = 0
    creation_passes: int = 0
    kernel_ms: float = 0.0
    wall_ms: float = 0.0
    gpu_launches: int = 0
    edge_ms: float = 0.0
    edge_launches: int = 0
    top_ms: float = 0.0       # dominant kernel (PageRank EB: hot-segment gather)
    top_launches: int = 0
    top_edges: int = 0        # edges per launch of it

    def to_dict(self):
        return asdict(self)

    @classmethod
    def from_pod(cls, st):
        n = min(st.direction_log_len, st.direction_log_cap)
        log = [DIRECTION_NAMES[st.direction_log[i]] for i in range(n)]
        return cls(st.dispatch_count, st.rounds, st.edges_traversed, log,
                   st.frontier_conversions, st.frontier_allocations, st.reused_frontiers,
                   st.creation_passes, st.kernel_ms, st.wall_ms, st.gpu_launches,
                   st.edge_ms, st.edge_launches, st.top_ms, st.top_launches, st.top_edges)


class Runtime:
    """Per-query device state bound to one graph (runtime.py:199-248)."""

    def __init__(self, cfg=None, graph=None):
        self.cfg = cfg or ExecConfig()
        self.cfg.validate()
        self._handle = None
        self.graph = None
        self.frontiers = FrontierPool(self)
        if graph is not None:
            self.bind(graph)

    def bind(self, graph):
        if self._handle is not None:
            if graph is not self.graph:
                raise EngineError("runtime already bound to another graph")
            return self
        h = C.c_void_p()
        pod = self.cfg.to_pod()
        _lib.call("gg_runtime_create", graph.handle, C.byref(pod), C.byref(h))
        self._handle = h
        self.graph = graph
        return self

    @property
    def handle(self):
        if self._handle is None:
            raise EngineError("runtime is not bound to a graph yet")
        return self._handle

    @property
    def stats(self):
        if self._handle is None:
            return RunStats()
        st = _lib.new_stats()
        _lib.call("gg_runtime_stats", self._handle, C.byref(st))
        return RunStats.from_pod(st)

    def close(self):
        if self._handle is not None:
            _lib.load().gg_runtime_destroy(self._handle)
            self._handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FrontierPool:
    """FrontierPool facade (runtime.py:124-157); storage lives on the device."""

    def __init__(self, rt):
        self._rt = rt

    def new_frontier(self, universe, ids, graph=None):
        from .frontier import VertexSubset
        rt = self._rt
        if graph is not None:
            rt.bind(graph)
        return VertexSubset.from_ids(rt, universe, ids)

    def release(self, vs):
        vs._release(self._rt)


def coerce_runtime(runtime, graph):
    if runtime is None:
        return Runtime(ExecConfig(), graph)
    if isinstance(runtime, ExecConfig):
        return Runtime(runtime, graph)
    return runtime.bind(graph)


class EdgeContext:
    """The reference's per-edge UDF API (runtime.py:299-362).

    Present for API parity; device traversals cannot call back into Python,
    so constructing one for an edge apply raises.
    """

    def __init__(self, *a, **k):
        raise EngineError("EdgeContext callbacks cannot run on the device; use a named "
                          "device UDF from paper_2012_07990_b200.udfs")


def pool_stats():
    """Device caching-pool counters: {"mallocs", "frees", "cached_bytes"}
    (driver allocations and frees since the library loaded)."""
    m, f, c = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.call("gg_pool_stats", C.byref(m), C.byref(f), C.byref(c))
    return {"mallocs": m.value, "frees": f.value, "cached_bytes": c.value}


def release_cached_memory():
    """Return every cached device block to the driver."""
    _lib.call("gg_release_cached_memory")
