"""VertexSubset on the device (reference frontier.py:129-269).

SPARSE = int32 queue + device count, BITMAP = 1 bit/vertex (same byte/bit
order as the reference's bytearray), BOOLMAP = 1 byte/vertex.  Storage is
owned by the query's device runtime and recycled through its frontier pool.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

SPARSE = "SPARSE"
BITMAP = "BITMAP"
BOOLMAP = "BOOLMAP"
MONOTONIC_COUNTERS = "MONOTONIC_COUNTERS"
REPR_CODE = {SPARSE: 0, BITMAP: 1, BOOLMAP: 2}
REPR_NAME = {v: k for k, v in REPR_CODE.items()}


class FrontierError(ValueError):
    pass


class VertexSubset:
    """A set (or, with dedup off, multiset) of active vertices on the GPU."""

    def __init__(self, runtime, universe, handle):
        self._rt = runtime
        self.universe = universe
        self._h = handle
        self._retired = False

    @classmethod
    def from_ids(cls, runtime, universe, ids):
        ids = np.ascontiguousarray(np.asarray(list(ids) if not isinstance(ids, np.ndarray)
                                              else ids, dtype=np.int64))
        if len(ids) and (ids.min() < 0 or ids.max() >= universe):
            bad = int(ids[(ids < 0) | (ids >= universe)][0])
            raise FrontierError("vertex id %d out of range [0, %d)" % (bad, universe))
        if runtime.graph is not None and runtime.graph.num_vertices != universe:
            # the device pool is sized by the bound graph; keep the universe for
            # the mismatch check in edgeset_apply
            return _ForeignSubset(runtime, universe, ids)
        ids32 = ids.astype(np.int32)
        h = C.c_void_p()
        _lib.call("gg_frontier_new", runtime.handle, _lib.ptr(ids32), len(ids32), C.byref(h))
        return cls(runtime, universe, h)

    @property
    def handle(self):
        if self._retired or self._h is None:
            raise FrontierError("frontier was retired")
        return self._h

    @property
    def repr(self):
        r = C.c_int32()
        _lib.call("gg_frontier_repr", self.handle, C.byref(r))
        return REPR_NAME[r.value]

    @property
    def size(self):
        n = C.c_int64()
        _lib.call("gg_frontier_size", self.handle, C.byref(n))
        return n.value

    def members(self):
        """Member ids: insertion order for SPARSE, ascending for dense."""
        n = self.size
        out = np.empty(max(n, 1), dtype=np.int32)
        got = C.c_int64()
        _lib.call("gg_frontier_members", self.handle, _lib.ptr(out), len(out), C.byref(got))
        return out[:got.value].tolist()

    def contains(self, v):
        return v in set(self.members())

    def convert(self, target):
        if target not in REPR_CODE:
            raise FrontierError("unknown representation %r" % target)
        h = C.c_void_p()
        _lib.call("gg_frontier_convert", self._rt.handle, self.handle, REPR_CODE[target],
                  C.byref(h))
        return VertexSubset(self._rt, self.universe, h)

    def _release(self, rt):
        if self._retired:
            return
        _lib.call("gg_frontier_release", rt.handle, self.handle)
        self._mark_retired()

    def _mark_retired(self):
        self._retired = True

    def retire(self):
        self._mark_retired()

    def __del__(self):
        try:
            if self._h is not None:
                _lib.load().gg_frontier_free(self._h)
                self._h = None
        except Exception:
            pass

    def __repr__(self):
        return "VertexSubset(universe=%d, repr=%s, size=%d)" % (self.universe, self.repr,
                                                                 self.size)


class _ForeignSubset(VertexSubset):
    """A subset whose universe differs from the runtime's graph (kept host-side
    only so that edgeset_apply can raise the reference's universe error)."""

    def __init__(self, runtime, universe, ids):
        super().__init__(runtime, universe, None)
        self._ids = ids

    @property
    def size(self):
        return len(self._ids)

    def members(self):
        return self._ids.tolist()
