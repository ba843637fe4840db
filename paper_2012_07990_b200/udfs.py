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
        for k, a in enumerate(self.arrays[:3]):
            setattr(st, "arr%d" % k, a.data_ptr())
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


class CcHook(DeviceUDF):
    """cc_soman's hook (algos.py:283-293): la, lb = label[src], label[dst];
    atomic_min(label, max(la, lb), min(la, lb)); a lowering sets changed[0].
    label: int32 CUDA tensor (V); changed: int32 CUDA tensor (1)."""
    code = _lib.UDF_CC_HOOK

    def __init__(self, label, changed):
        super().__init__(label, changed)


class BcForward(DeviceUDF):
    """bc's forward round at ``level`` (algos.py:353-365): CAS depth[dst]
    -1 -> level+1 with enqueue, sigma[dst] += sigma[src] when depth[dst] ==
    level+1; filter depth == -1 or level+1 (push) / owner store (pull).
    depth: int32, sigma: float64 CUDA tensors (V)."""
    code = _lib.UDF_BC_FORWARD

    def __init__(self, depth, sigma, level=0):
        super().__init__(depth, sigma)
        self.level = level

    def state(self):
        st = super().state()
        st.i0 = int(self.level)
        return st


class BcBackward(DeviceUDF):
    """bc's backward round (algos.py:378-382), push only: delta[src] +=
    sigma[src]/sigma[dst]*(1+delta[dst]) when depth[dst] == depth[src]+1.
    depth: int32, sigma / delta: float64 CUDA tensors (V)."""
    code = _lib.UDF_BC_BACKWARD

    def __init__(self, depth, sigma, delta):
        super().__init__(depth, sigma, delta)


class SsspRelax(DeviceUDF):
    """sssp_delta's relaxation (algos.py:233-234):
    queue.update_priority_min(dst, priorities[src] + weight) on a device
    :class:`~paper_2012_07990_b200.priority.BucketQueue`."""
    code = _lib.UDF_SSSP_RELAX

    def __init__(self, queue):
        super().__init__()
        self.queue = queue

    def state(self):
        st = _lib.GGUdfState()
        st.arr0 = self.queue.handle
        return st
