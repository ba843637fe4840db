"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A restatement of the reference package `schedge`'s algorithms (oracle.c,
each function cites the reference file:line it follows), pinned against
fixtures produced by running the reference itself (tests/golden/, made by
oracle/make_golden.py).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package, and only as the
checker or the CPU baseline; the product library never calls it.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

UNREACHED = 2**64 - 1


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        I64, F64 = C.c_int64, C.c_double
        L.or_pagerank.restype = I64
        L.or_pagerank.argtypes = [I64, I64, P, P, I64, F64, F64, P]
        L.or_pagerank_par.restype = I64
        L.or_pagerank_par.argtypes = [I64, P, P, P, I64, F64, F64, P]
        L.or_bfs_levels.argtypes = [I64, P, P, I64, P]
        L.or_bfs_levels_par.argtypes = [I64, P, P, I64, P]
        L.or_sssp_delta.restype = I64
        L.or_sssp_delta.argtypes = [I64, P, P, P, I64, I64, P]
        L.or_cc.restype = I64
        L.or_cc.argtypes = [I64, I64, P, P, P]
        L.or_bc.argtypes = [I64, P, P, P, I64, P]
        L.or_block_edges.argtypes = [I64, I64, P, I64, P, P]
        L.or_build_csr.argtypes = [I64, I64, P, P, P, P, P, P]
        L.or_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=dt))


def num_threads():
    return lib().or_num_threads()


def csr(V, keys, vals, w=None):
    """Stable CSR of keys -> vals (graphio.py:95-102)."""
    keys, vals = _c(keys, np.int32), _c(vals, np.int32)
    E = len(keys)
    off = np.zeros(V + 1, np.int64)
    nbr = np.zeros(max(E, 1), np.int32)
    wout = None
    wi = None
    if w is not None:
        wi = _c(w, np.uint32)
        wout = np.zeros(max(E, 1), np.uint32)
    lib().or_build_csr(V, E, _p(keys), _p(vals), _p(wi), _p(off), _p(nbr), _p(wout))
    return off, nbr[:E], (None if wout is None else wout[:E])


def pagerank(V, src, dst, max_iters=100, tol=1e-9, damping=0.85):
    src, dst = _c(src, np.int32), _c(dst, np.int32)
    out = np.zeros(V, np.float64)
    it = lib().or_pagerank(V, len(src), _p(src), _p(dst), max_iters, tol, damping, _p(out))
    return out, it


def pagerank_par(V, in_off, in_nbr, out_off, max_iters=100, tol=1e-9, damping=0.85):
    out = np.zeros(V, np.float64)
    it = lib().or_pagerank_par(V, _p(_c(in_off, np.int64)), _p(_c(in_nbr, np.int32)),
                               _p(_c(out_off, np.int64)), max_iters, tol, damping, _p(out))
    return out, it


def bfs_levels(V, off, nbr, source, parallel=False):
    out = np.zeros(V, np.int32)
    fn = lib().or_bfs_levels_par if parallel else lib().or_bfs_levels
    fn(V, _p(_c(off, np.int64)), _p(_c(nbr, np.int32)), source, _p(out))
    return out


def sssp_delta(V, off, nbr, w, source, delta):
    out = np.zeros(V, np.uint64)
    rounds = lib().or_sssp_delta(V, _p(_c(off, np.int64)), _p(_c(nbr, np.int32)),
                                 _p(_c(w, np.uint32)), source, delta, _p(out))
    return out, rounds


def cc(V, src, dst):
    src, dst = _c(src, np.int32), _c(dst, np.int32)
    out = np.zeros(V, np.int32)
    rounds = lib().or_cc(V, len(src), _p(src), _p(dst), _p(out))
    return out, rounds


def bc(V, off, nbr, sources):
    src = _c(sources, np.int64)
    out = np.zeros(V, np.float64)
    lib().or_bc(V, _p(_c(off, np.int64)), _p(_c(nbr, np.int32)), _p(src), len(src), _p(out))
    return out


def block_edges(V, dst, n):
    dst = _c(dst, np.int32)
    E = len(dst)
    S = (V + n - 1) // n
    perm = np.zeros(max(E, 1), np.int64)
    seg = np.zeros(max(S, 1), np.int64)
    lib().or_block_edges(V, E, _p(dst), n, _p(perm), _p(seg))
    return perm[:E], seg[:S]


def rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
    """C replica of the device RMAT generator (bit-identical, OpenMP)."""
    L = lib()
    L.or_rmat.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double,
                          C.c_uint64, C.c_void_p, C.c_void_p]
    V = 1 << scale
    E = V * edge_factor
    s = np.empty(E, np.int32)
    d = np.empty(E, np.int32)
    L.or_rmat(scale, E, a, b, c, seed, _p(s), _p(d))
    return V, s, d


# ---------------------------------------------------------------------------
# full-scale parity helpers (OpenMP; see the oracle.c section header)
# ---------------------------------------------------------------------------
def _par_lib():
    L = lib()
    if not getattr(L, "_par_ready", False):
        P, I64 = C.c_void_p, C.c_int64
        L.or_offsets_par.argtypes = [I64, I64, P, P]
        L.or_build_csr_par.argtypes = [I64, I64, P, P, P, P, P, P]
        L.or_bfs_levels_do.restype = I64
        L.or_bfs_levels_do.argtypes = [I64, P, P, P, P, I64, P]
        L.or_bfs_check_tree.restype = I64
        L.or_bfs_check_tree.argtypes = [I64, P, P, I64, P, P]
        L.or_cc_par.restype = I64
        L.or_cc_par.argtypes = [I64, I64, P, P, P]
        L.or_bc_par.argtypes = [I64, P, P, P, P, P, I64, P]
        L._par_ready = True
    return L


def offsets_par(V, keys):
    keys = _c(keys, np.int32)
    off = np.empty(V + 1, np.int64)
    _par_lib().or_offsets_par(V, len(keys), _p(keys), _p(off))
    return off


def csr_par(V, keys, vals, w=None):
    """CSR keys -> vals; neighbour order within a key unspecified."""
    keys, vals = _c(keys, np.int32), _c(vals, np.int32)
    E = len(keys)
    off = np.empty(V + 1, np.int64)
    nbr = np.empty(max(E, 1), np.int32)
    wi = wout = None
    if w is not None:
        wi = _c(w, np.uint32)
        wout = np.empty(max(E, 1), np.uint32)
    _par_lib().or_build_csr_par(V, E, _p(keys), _p(vals), _p(wi), _p(off), _p(nbr), _p(wout))
    return off, nbr[:E], (None if wout is None else wout[:E])


def bfs_levels_do(V, off, nbr, source, in_off=None, in_nbr=None):
    """Direction-optimising BFS levels (unique: equal to bfs_levels)."""
    if in_off is None:
        in_off, in_nbr = off, nbr
    out = np.empty(V, np.int32)
    _par_lib().or_bfs_levels_do(V, _p(_c(off, np.int64)), _p(_c(nbr, np.int32)),
                                _p(_c(in_off, np.int64)), _p(_c(in_nbr, np.int32)), source,
                                _p(out))
    return out


def bfs_check_tree(V, in_off, in_nbr, source, parents, levels):
    """Number of vertices violating BFS-tree legality (0 = legal tree)."""
    return int(_par_lib().or_bfs_check_tree(V, _p(_c(in_off, np.int64)), _p(_c(in_nbr, np.int32)),
                                            source, _p(_c(parents, np.int32)),
                                            _p(_c(levels, np.int32))))


def cc_par(V, src, dst):
    src, dst = _c(src, np.int32), _c(dst, np.int32)
    out = np.empty(V, np.int32)
    rounds = _par_lib().or_cc_par(V, len(src), _p(src), _p(dst), _p(out))
    return out, rounds


def bc_par(V, off, nbr, sources, in_off=None, in_nbr=None):
    """in_off/in_nbr default to off/nbr (symmetric graphs, as bc requires)."""
    if in_off is None:
        in_off, in_nbr = off, nbr
    src = _c(sources, np.int64)
    out = np.empty(V, np.float64)
    _par_lib().or_bc_par(V, _p(_c(off, np.int64)), _p(_c(nbr, np.int32)),
                         _p(_c(in_off, np.int64)), _p(_c(in_nbr, np.int32)), _p(src), len(src),
                         _p(out))
    return out
