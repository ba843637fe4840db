"""Two-bucket priority queue for ordered traversals (reference priority.py).

:class:`BucketQueue` keeps the reference's contract (priority.py:17-118) with
its state on a GPU: priorities ``u64[universe]`` (``UNREACHED`` = 2^64-1),
``current`` = vertices whose priority lies in ``[index*delta,
(index+1)*delta)``, ``far`` = everything farther out, re-bucketed lazily by
:meth:`advance` (stale entries dropped).  ``update_priority_min`` for a whole
frontier runs as the device UDF :class:`~paper_2012_07990_b200.udfs.SsspRelax`
inside ``edgeset_apply``; the single-vertex method here is the same device
update for one vertex.  ``sssp_delta``'s fused loop keeps the queue inside one
cooperative launch (csrc/sssp.cu).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

UNREACHED = 2**64 - 1  # reserved infinity sentinel for 64-bit priorities (priority.py:14)


class _BucketView:
    """``current`` / ``far`` of a queue: ``size`` and ``members()`` like a
    SPARSE VertexSubset (insertion order)."""

    def __init__(self, queue, which):
        self._q = queue
        self._which = which

    @property
    def size(self):
        return self._q._info()[1 + self._which]

    def members(self):
        n = self.size
        out = np.empty(max(n, 1), np.int32)
        got = C.c_int64()
        _lib.call("gg_bucket_queue_members", self._q.handle, self._which, _lib.ptr(out), len(out),
                  C.byref(got))
        return out[:got.value].tolist()

    def __contains__(self, v):
        return v in self.members()


class BucketQueue:
    """Delta-bucketed work queue over per-vertex priorities (priority.py:17)."""

    def __init__(self, universe, delta, locks=None, device=0):
        if delta < 1:
            raise ValueError("delta must be >= 1")
        self.universe = universe
        self.delta = delta
        h = C.c_void_p()
        _lib.call("gg_bucket_queue_create", int(device), int(universe), int(delta), C.byref(h))
        self._h = h

    @property
    def handle(self):
        if self._h is None:
            from .runtime import EngineError
            raise EngineError("bucket queue was closed")
        return self._h

    def _info(self):
        idx, nc, nf = C.c_uint64(), C.c_int64(), C.c_int64()
        _lib.call("gg_bucket_queue_info", self.handle, C.byref(idx), C.byref(nc), C.byref(nf))
        return idx.value, nc.value, nf.value

    @property
    def current_bucket_index(self):
        return self._info()[0]

    @property
    def current(self):
        return _BucketView(self, 0)

    @property
    def far(self):
        return _BucketView(self, 1)

    @property
    def priorities(self):
        """Host copy of the priorities (numpy uint64; UNREACHED for unseen)."""
        out = np.empty(self.universe, np.uint64)
        _lib.call("gg_bucket_queue_priorities", self.handle, _lib.ptr(out))
        return out

    def seed(self, v, priority=0):
        """Place a starting vertex; the bucket index snaps to its bucket."""
        _lib.call("gg_bucket_queue_seed", self.handle, int(v), int(priority))

    def take_current(self):
        """Hand the pending current bucket to the caller (a SPARSE
        VertexSubset on the device) and start a fresh one."""
        from .frontier import VertexSubset
        h = C.c_void_p()
        _lib.call("gg_bucket_queue_take_current", self.handle, C.byref(h))
        return VertexSubset(None, self.universe, h)

    def recycle(self, taken):
        """Return a drained bucket's storage for the next round."""
        _lib.call("gg_bucket_queue_recycle", self.handle, taken.handle)
        taken._mark_retired()

    def update_priority_min(self, v, candidate):
        """Lower ``priorities[v]`` to ``candidate`` if smaller; on improvement
        enqueue into current (same bucket as the index) or far."""
        if candidate < 0:
            raise ValueError("priorities are non-negative")
        imp = C.c_int32()
        _lib.call("gg_bucket_queue_update_min", self.handle, int(v), int(candidate),
                  C.byref(imp))
        return bool(imp.value)

    def advance(self):
        """Move the nearest far bucket into current; None when drained."""
        ne = C.c_int32()
        _lib.call("gg_bucket_queue_advance", self.handle, C.byref(ne))
        return self.current if ne.value else None

    def done(self):
        _, nc, nf = self._info()
        return nc == 0 and nf == 0

    def close(self):
        if self._h is not None:
            _lib.load().gg_bucket_queue_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
