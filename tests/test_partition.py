"""Load-balancer splits pinned to the reference's own partitions
(tests/golden/reference_small.json "partition" cases, made by running
schedge's engine.lb_partition_etwc / _twc / _strict, engine.py:51-142):
the host restatements in engine.py on every case, and the device kernels'
per-vertex split (gg_partition_dump, the same __device__ split functions
k_push_etwc / k_twc_bin use) where the device's fixed warp of 32 applies."""

import numpy as np
import pytest

import oracle
from tests.util import arrays


class _G:
    def __init__(self, off):
        self.out_offsets = off


class _Cfg:
    def __init__(self, nw, cta, warp):
        self.num_workers, self.cta_size, self.warp_size = nw, cta, warp


def _cases(golden_small):
    for case in golden_small["cases"]:
        if case["algo"] == "partition":
            V, s, d, _ = arrays(golden_small["graphs"][case["graph"]])
            off, _, _ = oracle.csr(V, s, d)
            yield case, V, s, d, off


def _tup(x):
    return [tuple(_tup(y) if isinstance(y, list) else y for y in q) for q in x]


def test_host_partitions_match_reference(golden_small):
    from paper_2012_07990_b200 import engine
    n = 0
    for case, V, s, d, off in _cases(golden_small):
        cfg = _Cfg(*case["cfg"])
        g = _G(off)
        got = engine.lb_partition_etwc(case["active"], g, cfg)
        want = [tuple([tuple(map(tuple, q)) for q in w]) for w in case["etwc"]]
        assert [tuple(tuple(q) for q in w) for w in got] == want
        assert [list(q) for q in engine.lb_partition_twc(case["active"], g, cfg)] == case["twc"]
        ranges, prefix = engine.lb_partition_strict(case["active"], g, cfg)
        assert [list(r) for r in ranges] == case["strict"][0] and prefix == case["strict"][1]
        n += 1
    assert n == 6


def _per_vertex_etwc(case):
    """(e0, e1, e2) per active entry, from the reference's queues."""
    sizes = {}
    for q0, q1, q2 in case["etwc"]:
        for stage, q in ((0, q0), (1, q1), (2, q2)):
            for lo, hi, u in q:
                sizes.setdefault(u, [0, 0, 0])[stage] += hi - lo
    return [sizes.get(u, [0, 0, 0]) for u in case["active"]]


@pytest.mark.gpu
def test_device_split_matches_reference(golden_small):
    import ctypes as C
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200 import _lib
    n_checked = 0
    for case, V, s, d, off in _cases(golden_small):
        nw, cta, warp = case["cfg"]
        if warp != 32:  # the device warp is the hardware's 32 lanes
            continue
        g = gg.Graph.from_coo(V, s, d)
        rt = gg.Runtime(gg.ExecConfig(cta_size=cta), g)
        fr = rt.frontiers.new_frontier(V, case["active"])
        n = len(case["active"])
        out = np.empty(3 * n + 1, np.int64)
        got = C.c_int64()
        lb = {"ETWC": 5, "TWC": 6, "STRICT": 3}
        _lib.call("gg_partition_dump", rt.handle, fr.handle, lb["ETWC"], _lib.ptr(out), len(out),
                  C.byref(got))
        assert out[:got.value].reshape(-1, 3).tolist() == _per_vertex_etwc(case)
        _lib.call("gg_partition_dump", rt.handle, fr.handle, lb["TWC"], _lib.ptr(out), len(out),
                  C.byref(got))
        cta_q, warp_q, thread_q = case["twc"]
        want = [2 if u in cta_q else 1 if u in warp_q else 0 for u in case["active"]]
        assert out[:got.value].tolist() == want
        _lib.call("gg_partition_dump", rt.handle, fr.handle, lb["STRICT"], _lib.ptr(out), len(out),
                  C.byref(got))
        assert out[:got.value].tolist() == case["strict"][1]
        n_checked += 1
    assert n_checked == 2


@pytest.mark.gpu
@pytest.mark.parametrize("cta", [32, 64, 256, 1024])
def test_device_split_matches_host_restatement(cta):
    """Random multiset active lists with hubs, every CTA size the engine
    accepts: the device split equals engine.py's restatement entry by entry."""
    import ctypes as C
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200 import _lib, engine
    from oracle import gen
    V, s, d = gen.rmat(11, 16, seed=cta)
    g = gg.Graph.from_coo(V, s, d)
    off, _, _ = oracle.csr(V, s, d)
    rng = np.random.default_rng(cta)
    active = rng.integers(0, V, size=3 * V).tolist()  # duplicates included
    rt = gg.Runtime(gg.ExecConfig(cta_size=cta), g)
    fr = rt.frontiers.new_frontier(V, active)
    out = np.empty(3 * len(active) + 1, np.int64)
    got = C.c_int64()
    _lib.call("gg_partition_dump", rt.handle, fr.handle, 5, _lib.ptr(out), len(out), C.byref(got))
    cfg = _Cfg(1, cta, 32)
    q0, q1, q2 = engine.lb_partition_etwc(active, _G(off), cfg)[0]
    want = np.zeros((len(active), 3), np.int64)
    # queue entries appear in active order per stage; map them back by position
    pos = {0: 0, 1: 0, 2: 0}
    for i, u in enumerate(active):
        for stage, q in ((0, q0), (1, q1), (2, q2)):
            if pos[stage] < len(q) and q[pos[stage]][2] == u:
                a, b, _ = q[pos[stage]]
                want[i, stage] = b - a
                pos[stage] += 1
    assert np.array_equal(out[:got.value].reshape(-1, 3), want)
    _lib.call("gg_partition_dump", rt.handle, fr.handle, 6, _lib.ptr(out), len(out), C.byref(got))
    cq, wq, tq = engine.lb_partition_twc(active, _G(off), cfg)
    assert (out[:got.value] == 2).sum() == len(cq) and (out[:got.value] == 1).sum() == len(wq)
    deg = off[np.asarray(active) + 1] - off[np.asarray(active)]
    assert np.array_equal(out[:got.value], np.where(deg > cta, 2, np.where(deg > 32, 1, 0)))
    _lib.call("gg_partition_dump", rt.handle, fr.handle, 3, _lib.ptr(out), len(out), C.byref(got))
    assert out[:got.value].tolist() == engine.lb_partition_strict(active, _G(off), cfg)[1]
