"""Named device UDFs: the device stand-ins for the reference's per-edge
Python callables (EdgeContext, runtime.py:299-362; algos.py UDFs).

Each object carries the device arrays it reads/writes (torch CUDA tensors are
used purely as device allocations) and the udf id of include/gg.h.
``udf.filter`` is the matching ``to_filter`` (e.g. ``parent[v] == -1``).
"""

from __future__ import annotations

from . import _lib


class DeviceFilter:
    def __init__(self, udf):
        self.udf = udf


class DeviceUDF:
    code = None

    def __init__(self, *arrays):
        self.arrays = arrays

    @property
    def filter(self):
        return DeviceFilter(self)

    def state(self):
        st = _lib.GGUdfState()
        if len(self.arrays) > 0:
            st.arr0 = self.arrays[0].data_ptr()
        if len(self.arrays) > 1:
            st.arr1 = self.arrays[1].data_ptr()
        return st


class BfsParent(DeviceUDF):
    """push: CAS(parent[dst], -1 -> src) + enqueue; pull: owner store + enqueue;
    filter parent[v] == -1 (algos.py:114-125).  parent: int32 CUDA tensor."""
    code = _lib.UDF_BFS


class CountInDegree(DeviceUDF):
    """atomic_add(counts[dst], 1) (test_engine.py:246-264). counts: int64 CUDA tensor."""
    code = _lib.UDF_COUNT


class EnqueueDst(DeviceUDF):
    """ctx.enqueue(ctx.dst) with no guard (test_engine.py:384-399)."""
    code = _lib.UDF_ENQUEUE


class PageRankGather(DeviceUDF):
    """atomic_add(acc[dst], contrib[src]) (algos.py:180-181); f64 tensors."""
    code = _lib.UDF_PR
