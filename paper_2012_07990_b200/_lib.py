"""ctypes binding of libgg.so (include/gg.h).

The product path has no fallback: if the shared library is missing or the
device is absent, calls raise.  ``load()`` only needs the .so (it is safe on a
CPU-only host, where it is used to check the exported symbols); the compute
entry points need a CUDA device.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GG_LIB_PATH") or os.path.join(_HERE, "libgg.so")  # override: A/B builds

# status codes (gg.h)
GG_OK = 0
GG_ERR_SCHEDULE = -1
GG_ERR_ENGINE = -2
GG_ERR_VALUE = -3
GG_ERR_CUDA = -4
GG_ERR_NCCL = -5
GG_ERR_FRONTIER = -6
GG_ERR_OOM = -7

UDF_BFS, UDF_COUNT, UDF_ENQUEUE, UDF_PR = 0, 1, 2, 3
UDF_CC_HOOK, UDF_BC_FORWARD, UDF_BC_BACKWARD, UDF_SSSP_RELAX = 4, 5, 6, 7


class GGSchedule(C.Structure):
    _fields_ = [("direction", C.c_int32), ("pull_repr", C.c_int32),
                ("load_balance", C.c_int32), ("blocking", C.c_int32),
                ("blocking_size", C.c_int64), ("frontier_creation", C.c_int32),
                ("dedup", C.c_int32), ("dedup_strategy", C.c_int32),
                ("kernel_fusion", C.c_int32), ("delta", C.c_int64)]


class GGBinding(C.Structure):
    _fields_ = [("is_hybrid", C.c_int32), ("threshold", C.c_double),
                ("s1", GGSchedule), ("s2", GGSchedule)]


class GGExec(C.Structure):
    _fields_ = [("num_workers", C.c_int32), ("cta_size", C.c_int32),
                ("warp_size", C.c_int32), ("deterministic", C.c_int32)]


class GGStats(C.Structure):
    _fields_ = [("dispatch_count", C.c_int64), ("rounds", C.c_int64),
                ("edges_traversed", C.c_int64), ("frontier_conversions", C.c_int64),
                ("frontier_allocations", C.c_int64), ("reused_frontiers", C.c_int64),
                ("creation_passes", C.c_int64), ("direction_log", C.POINTER(C.c_int32)),
                ("direction_log_cap", C.c_int64), ("direction_log_len", C.c_int64),
                ("kernel_ms", C.c_double), ("wall_ms", C.c_double),
                ("gpu_launches", C.c_int64), ("edge_ms", C.c_double),
                ("edge_launches", C.c_int64), ("top_ms", C.c_double),
                ("top_launches", C.c_int64), ("top_edges", C.c_int64)]


class GGDeviceInfo(C.Structure):
    _fields_ = [("device", C.c_int32), ("sm_count", C.c_int32), ("l2_bytes", C.c_int64),
                ("hbm_bytes", C.c_int64), ("cc_major", C.c_int32), ("cc_minor", C.c_int32),
                ("max_smem_per_block", C.c_int32), ("name", C.c_char * 128)]


class GGUdfState(C.Structure):
    _fields_ = [("arr0", C.c_void_p), ("arr1", C.c_void_p), ("i0", C.c_int64),
                ("arr2", C.c_void_p)]


VP = C.c_void_p
PP = C.POINTER(C.c_void_p)
I32, I64, F64, U64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64

# name -> (restype, argtypes); the list is the symbol contract checked by the
# CPU test-suite against include/gg.h.
SIGNATURES = {
    "gg_last_error": (C.c_char_p, []),
    "gg_version": (C.c_char_p, []),
    "gg_device_count": (I32, [C.POINTER(I32)]),
    "gg_device_info_get": (I32, [I32, C.POINTER(GGDeviceInfo)]),
    "gg_graph_create": (I32, [I32, I64, I64, VP, VP, VP, I32, PP]),
    "gg_graph_create_device": (I32, [I32, I64, I64, VP, VP, VP, I32, PP]),
    "gg_graph_destroy": (I32, [VP]),
    "gg_graph_info": (I32, [VP, C.POINTER(I64), C.POINTER(I64), C.POINTER(I32),
                            C.POINTER(I32), C.POINTER(I32)]),
    "gg_graph_copy_array": (I32, [VP, I32, VP]),
    "gg_graph_drop_coo": (I32, [VP]),
    "gg_generate": (I32, [I32, I32, I32, I32, F64, F64, F64, U64, I32, PP]),
    "gg_default_blocking_size": (I64, [VP]),
    "gg_block_edges": (I32, [VP, I64, PP, C.POINTER(F64)]),
    "gg_blocked_info": (I32, [VP, C.POINTER(I64), C.POINTER(I64)]),
    "gg_blocked_copy_array": (I32, [VP, I32, VP]),
    "gg_blocked_install": (I32, [VP, I64, I64, VP, VP, VP, VP, PP]),
    "gg_runtime_create": (I32, [VP, C.POINTER(GGExec), PP]),
    "gg_runtime_destroy": (I32, [VP]),
    "gg_runtime_stats": (I32, [VP, C.POINTER(GGStats)]),
    "gg_frontier_new": (I32, [VP, VP, I64, PP]),
    "gg_frontier_release": (I32, [VP, VP]),
    "gg_frontier_free": (I32, [VP]),
    "gg_frontier_size": (I32, [VP, C.POINTER(I64)]),
    "gg_frontier_repr": (I32, [VP, C.POINTER(I32)]),
    "gg_frontier_members": (I32, [VP, VP, I64, C.POINTER(I64)]),
    "gg_frontier_convert": (I32, [VP, VP, I32, PP]),
    "gg_edgeset_apply": (I32, [VP, I32, C.POINTER(GGUdfState), I32, VP,
                               C.POINTER(GGBinding), I32, I32, PP]),
    "gg_partition_dump": (I32, [VP, VP, I32, VP, I64, C.POINTER(I64)]),
    "gg_runtime_fused_region": (I32, [VP, I32]),
    "gg_runtime_add_rounds": (I32, [VP, I64]),
    "gg_bucket_queue_create": (I32, [I32, I64, U64, PP]),
    "gg_bucket_queue_destroy": (I32, [VP]),
    "gg_bucket_queue_seed": (I32, [VP, I64, U64]),
    "gg_bucket_queue_update_min": (I32, [VP, I64, U64, C.POINTER(I32)]),
    "gg_bucket_queue_take_current": (I32, [VP, PP]),
    "gg_bucket_queue_recycle": (I32, [VP, VP]),
    "gg_bucket_queue_advance": (I32, [VP, C.POINTER(I32)]),
    "gg_bucket_queue_info": (I32, [VP, C.POINTER(U64), C.POINTER(I64), C.POINTER(I64)]),
    "gg_bucket_queue_members": (I32, [VP, I32, VP, I64, C.POINTER(I64)]),
    "gg_bucket_queue_priorities": (I32, [VP, VP]),
    "gg_apply_blocked": (I32, [VP, I64, I32, C.POINTER(GGUdfState), C.POINTER(I64)]),
    "gg_bfs": (I32, [VP, I64, C.POINTER(GGBinding), I32, C.POINTER(GGExec), VP,
                     C.POINTER(GGStats)]),
    "gg_pagerank": (I32, [VP, C.POINTER(GGBinding), I32, C.POINTER(GGExec), I64, F64, F64,
                          VP, C.POINTER(GGStats)]),
    "gg_pagerank_prepare": (I32, [VP, C.POINTER(GGBinding), I32, C.POINTER(F64)]),
    "gg_relabel_prepare": (I32, [VP, C.POINTER(F64)]),
    "gg_last_exchange_bytes": (I32, [C.POINTER(C.c_uint64)]),
    "gg_pagerank_ex": (I32, [VP, C.POINTER(GGBinding), I32, C.POINTER(GGExec), I64, F64,
                             F64, I32, VP, C.POINTER(GGStats)]),
    "gg_pagerank_resume": (I32, [VP, C.POINTER(GGBinding), I32, C.POINTER(GGExec), I64, F64,
                                 F64, VP, VP, C.POINTER(GGStats)]),
    "gg_sssp_delta": (I32, [VP, I64, C.POINTER(GGBinding), I32, C.POINTER(GGExec), VP,
                            C.POINTER(GGStats)]),
    "gg_cc": (I32, [VP, C.POINTER(GGBinding), I32, C.POINTER(GGExec), VP,
                    C.POINTER(GGStats)]),
    "gg_bc": (I32, [VP, VP, I64, C.POINTER(GGBinding), C.POINTER(GGExec), VP,
                    C.POINTER(GGStats)]),
    "gg_nccl_unique_id": (I32, [VP]),
    "gg_release_cached_memory": (I32, []),
    "gg_pool_stats": (I32, [C.POINTER(I64)] * 3),
    "gg_comm_init": (I32, [I32, I32, I32, VP, PP]),
    "gg_comm_destroy": (I32, [VP]),
    "gg_pagerank_dist": (I32, [VP, VP, I64, F64, F64, VP, C.POINTER(GGStats)]),
    "gg_pagerank_dist_ex": (I32, [VP, VP, C.POINTER(GGBinding), I32, I64, F64, F64, VP,
                                  C.POINTER(GGStats)]),
    "gg_pagerank_dist_prepare": (I32, [I32, I32, VP, C.POINTER(GGBinding), I32,
                                       C.POINTER(F64), VP, VP]),
    "gg_bfs_dist_bounds": (I32, [VP, I32, VP]),
    "gg_bfs_dist": (I32, [VP, VP, I64, F64, VP, C.POINTER(GGStats)]),
    "gg_bfs_virtual": (I32, [VP, I32, I64, F64, VP, C.POINTER(GGStats)]),
    "gg_pagerank_virtual": (I32, [VP, I32, C.POINTER(GGBinding), I32, I32, I64, F64, F64, VP,
                                  C.POINTER(GGStats)]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libgg.so (raises ImportError when it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError("libgg.so not built at %s; run __graft_entry__.build() or "
                              "`make -C paper_2012_07990_b200/csrc`" % LIB_PATH)
        lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue  # reported by missing_symbols()
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def missing_symbols():
    lib = load()
    return [n for n in SIGNATURES if getattr(lib, n, None) is None]


def error_class(code):
    from .sched import ScheduleError
    from .runtime import EngineError
    from .frontier import FrontierError
    return {GG_ERR_SCHEDULE: ScheduleError, GG_ERR_ENGINE: EngineError,
            GG_ERR_VALUE: ValueError, GG_ERR_FRONTIER: FrontierError,
            GG_ERR_OOM: MemoryError}.get(code, RuntimeError)


def check(code):
    """Raise the reference's exception class for a gg_status."""
    if code == GG_OK:
        return
    msg = load().gg_last_error().decode(errors="replace")
    raise error_class(code)(msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def device_count():
    n = I32(0)
    call("gg_device_count", C.byref(n))
    return n.value


def device_info(dev=0):
    info = GGDeviceInfo()
    call("gg_device_info_get", dev, C.byref(info))
    return info


def ptr(a):
    """Data pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())


def new_stats(log_cap=1 << 16):
    st = GGStats()
    buf = (C.c_int32 * log_cap)()
    st.direction_log = C.cast(buf, C.POINTER(C.c_int32))
    st.direction_log_cap = log_cap
    st._buf = buf  # keep alive
    return st
