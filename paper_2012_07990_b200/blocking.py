"""EdgeBlocking mirror (reference blocking.py).

``block_edges`` runs Alg. 1 on the device (stable partition of the COO by
``dst // n``) and caches the layout on the graph (blocking.py:69-75);
``BlockedGraph`` exposes it with the reference's fields (``segment_start`` =
inclusive ends).  ``default_blocking_size`` sizes the segment from the L2 of
the graph's GPU (queried), where the reference uses a fixed 2 MiB budget
(``reference_blocking_size`` keeps that rule).  The sidecar format
(blocking.py:189-217) is byte-compatible.
"""

from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _lib
from .runtime import EngineError

DEFAULT_CACHE_BUDGET = 2 * 1024 * 1024
BYTES_PER_VERTEX_DATUM = 8
_SIDECAR_MAGIC = b"SCHEDGEB"
_SIDECAR_VERSION = 1


def reference_blocking_size(num_vertices, cache_budget=DEFAULT_CACHE_BUDGET):
    """The reference's rule (blocking.py:63-66)."""
    n = max(1, cache_budget // BYTES_PER_VERTEX_DATUM)
    return min(n, max(1, num_vertices))


def default_blocking_size(num_vertices_or_graph, cache_budget=None):
    """Vertices per segment.  Given a device Graph: half of that GPU's L2 as
    f64 destination data; given a vertex count: the reference rule."""
    if hasattr(num_vertices_or_graph, "handle"):
        if cache_budget is not None:
            return reference_blocking_size(num_vertices_or_graph.num_vertices, cache_budget)
        return int(_lib.load().gg_default_blocking_size(num_vertices_or_graph.handle))
    return reference_blocking_size(num_vertices_or_graph,
                                   cache_budget if cache_budget is not None else DEFAULT_CACHE_BUDGET)


class BlockedGraph:
    """COO grouped into destination segments (blocking.py:24-60)."""

    def __init__(self, num_vertices, vertices_per_segment, segment_start, edges_src,
                 edges_dst, edges_weight=None, prep_ms=0.0):
        self.num_vertices = num_vertices
        self.num_edges = len(edges_src)
        self.vertices_per_segment = vertices_per_segment
        self.num_segments = len(segment_start)
        self.segment_start = segment_start
        self.edges_src = edges_src
        self.edges_dst = edges_dst
        self.edges_weight = edges_weight
        self.prep_ms = prep_ms
        self.graph = None  # the device Graph whose cached layout this is

    def segment_range(self, s):
        lo = self.segment_start[s - 1] if s else 0
        return lo, self.segment_start[s]

    def edge_multiset(self):
        w = self.edges_weight if self.edges_weight is not None else [0] * self.num_edges
        return sorted(zip(list(self.edges_src), list(self.edges_dst), list(w)))


def block_edges(g, n):
    """Alg. 1 on the device; returns the host view of the blocked layout."""
    if n < 1:
        raise ValueError("vertices per segment must be >= 1")
    if g.num_vertices == 0:
        raise ValueError("empty graph")
    h = C.c_void_p()
    prep = C.c_double()
    _lib.call("gg_block_edges", g.handle, int(n), C.byref(h), C.byref(prep))
    nseg = C.c_int64()
    _lib.call("gg_blocked_info", h, C.byref(nseg), None)
    E = g.num_edges
    seg = np.empty(max(nseg.value, 1), np.int64)
    src = np.empty(max(E, 1), np.int32)
    dst = np.empty(max(E, 1), np.int32)
    _lib.call("gg_blocked_copy_array", h, 0, _lib.ptr(seg))
    _lib.call("gg_blocked_copy_array", h, 1, _lib.ptr(src))
    _lib.call("gg_blocked_copy_array", h, 2, _lib.ptr(dst))
    w = None
    if g.weighted:
        w = np.empty(max(E, 1), np.uint32)
        _lib.call("gg_blocked_copy_array", h, 3, _lib.ptr(w))
        w = w[:E].astype(np.int64).tolist()
    bg = BlockedGraph(g.num_vertices, n, seg[:nseg.value].tolist(), src[:E].tolist(),
                      dst[:E].tolist(), w, prep.value)
    bg.graph = g
    return bg


blocked_for = block_edges


def apply_blocked(bg, process_edge, runtime=None, make_context=None):
    """Alg. 2 (blocking.py:116-186): ``process_edge`` once per edge of the
    blocked layout, segments in order with a grid barrier between them, one
    dispatch; returns the number of edges processed.

    ``bg`` is the graph's blocked layout: a :class:`BlockedGraph` from
    :func:`block_edges` (with ``bg.graph`` set) or a ``(graph, n)`` pair;
    ``process_edge`` is a named device UDF (its atomic form runs per edge,
    as the reference's EDGE_ONLY apply does).  ``make_context`` has no device
    counterpart (per-worker Python contexts) and must be None.
    """
    from .engine import _device_udf
    from .runtime import coerce_runtime
    if make_context is not None:
        raise EngineError("make_context callbacks cannot run on the device")
    if isinstance(bg, tuple):
        g, n = bg
    else:
        g, n = getattr(bg, "graph", None), bg.vertices_per_segment
        if g is None:
            raise EngineError("apply_blocked needs the device graph the layout was built "
                              "from (block_edges(g, n) or (g, n))")
    udf = _device_udf(process_edge)
    rt = coerce_runtime(runtime, g)
    st = udf.state()
    edges = C.c_int64()
    _lib.call("gg_apply_blocked", rt.handle, int(n), udf.code, C.byref(st), C.byref(edges))
    return edges.value


def save_blocked(bg, path):
    """Little-endian 64-bit sidecar (blocking.py:189-197)."""
    with open(path, "wb") as fh:
        fh.write(_SIDECAR_MAGIC)
        has_w = 1 if bg.edges_weight is not None else 0
        fh.write(struct.pack("<qqqqqq", _SIDECAR_VERSION, bg.num_vertices, bg.num_edges,
                             bg.vertices_per_segment, bg.num_segments, has_w))
        for arr in (bg.segment_start, bg.edges_src, bg.edges_dst):
            np.asarray(arr, dtype="<i8").tofile(fh)
        if has_w:
            np.asarray(bg.edges_weight, dtype="<i8").tofile(fh)


def load_blocked(path):
    with open(path, "rb") as fh:
        if fh.read(len(_SIDECAR_MAGIC)) != _SIDECAR_MAGIC:
            raise EngineError("%s: not a blocked-graph sidecar" % path)
        version, nv, ne, n, ns, has_w = struct.unpack("<qqqqqq", fh.read(48))
        if version != _SIDECAR_VERSION:
            raise EngineError("%s: unsupported sidecar version %d" % (path, version))
        seg = np.fromfile(fh, dtype="<i8", count=ns).tolist()
        src = np.fromfile(fh, dtype="<i8", count=ne).tolist()
        dst = np.fromfile(fh, dtype="<i8", count=ne).tolist()
        w = np.fromfile(fh, dtype="<i8", count=ne).tolist() if has_w else None
    return BlockedGraph(nv, n, seg, src, dst, w)


def load_blocked_to_device(path, g=None, device=0, symmetric=False):
    """A sidecar straight to the device: the layout is
    installed as the graph's cached Alg. 1 result for its width, validated
    against the graph (segment bounds, edge multiset), without re-blocking.
    With ``g`` None the graph itself is built from the sidecar's edges (the
    blocked order is a valid COO order, and Alg. 1 is stable, so blocking it
    again would reproduce the same layout).  Returns the device Graph."""
    from .graphio import Graph, GraphLoadError
    with open(path, "rb") as fh:
        if fh.read(len(_SIDECAR_MAGIC)) != _SIDECAR_MAGIC:
            raise EngineError("%s: not a blocked-graph sidecar" % path)
        version, nv, ne, n, ns, has_w = struct.unpack("<qqqqqq", fh.read(48))
        if version != _SIDECAR_VERSION:
            raise EngineError("%s: unsupported sidecar version %d" % (path, version))
        seg = np.fromfile(fh, dtype="<i8", count=ns)
        src = np.fromfile(fh, dtype="<i8", count=ne)
        dst = np.fromfile(fh, dtype="<i8", count=ne)
        w = np.fromfile(fh, dtype="<i8", count=ne) if has_w else None
    if len(seg) != ns or len(src) != ne or len(dst) != ne or (has_w and len(w) != ne):
        raise EngineError("%s: truncated sidecar" % path)
    if ne and (max(src.max(), dst.max()) >= min(nv, 2 ** 31) or min(src.min(), dst.min()) < 0):
        raise GraphLoadError("%s: vertex id out of range" % path)
    s32 = np.ascontiguousarray(src.astype(np.int32))
    d32 = np.ascontiguousarray(dst.astype(np.int32))
    w32 = None if w is None else np.ascontiguousarray(w.astype(np.uint32))
    if g is None:
        g = Graph.from_coo(nv, s32, d32, w32, symmetric=symmetric, device=device)
    elif g.num_vertices != nv or g.num_edges != ne:
        raise EngineError("%s: sidecar does not match the graph (%d/%d vertices, %d/%d edges)"
                          % (path, nv, g.num_vertices, ne, g.num_edges))
    seg = np.ascontiguousarray(seg.astype(np.int64))
    _lib.call("gg_blocked_install", g.handle, int(n), int(ns), _lib.ptr(seg), _lib.ptr(s32),
              _lib.ptr(d32), _lib.ptr(w32), None)
    return g
