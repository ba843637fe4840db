"""Graph container mirror (reference graphio.py).

A :class:`Graph` is uploaded once to HBM at construction: CSR-out, CSR-in and
the COO view in load order (graphio.py:58-81), built on the device by a stable
counting sort so neighbour order equals the reference's.  Host-side arrays are
numpy views fetched lazily from the device (never Python lists, which cost
~143 B/edge in the reference).  Loaders/symmetrisation are thin host helpers
kept for API parity; synthetic inputs are generated on the device
(``generate_rmat`` / ``generate_grid`` / ``generate_kronecker``).
"""

from __future__ import annotations

import ctypes as C
import random

import numpy as np

from . import _lib


class GraphLoadError(ValueError):
    """Unreadable or malformed graph input (graphio.py:15)."""


_ARR = {"out_offsets": (0, np.int64), "out_neighbors": (1, np.int32),
        "out_weights": (2, np.uint32), "in_offsets": (3, np.int64),
        "in_neighbors": (4, np.int32), "in_weights": (5, np.uint32),
        "coo_src": (6, np.int32), "coo_dst": (7, np.int32), "coo_weights": (8, np.uint32)}


class Graph:
    """Immutable directed multigraph resident on one GPU (graphio.py:19-92)."""

    def __init__(self, handle, device=0, diagnostics=None):
        self._h = handle
        V, E, w, s, d = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        _lib.call("gg_graph_info", handle, C.byref(V), C.byref(E), C.byref(w), C.byref(s),
                  C.byref(d))
        self.num_vertices = V.value
        self.num_edges = E.value
        self.weighted = bool(w.value)
        self.symmetric = bool(s.value)
        self.device = d.value
        self.diagnostics = diagnostics or {}
        self._host = {}

    # -- construction -----------------------------------------------------
    @classmethod
    def from_coo(cls, num_vertices, src, dst, weights=None, symmetric=False,
                 diagnostics=None, device=0):
        """Build all views from COO arrays (load order preserved).

        int32 numpy arrays (ideally in pinned memory) are uploaded as-is and
        range-checked on the device; other inputs are validated on the host.
        """
        fast = (isinstance(src, np.ndarray) and isinstance(dst, np.ndarray)
                and src.dtype == np.int32 and dst.dtype == np.int32
                and src.flags.c_contiguous and dst.flags.c_contiguous)
        if not fast:
            src = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
            dst = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
        if src.shape != dst.shape:
            raise GraphLoadError("src/dst length mismatch")
        if not fast and len(src) and (src.min() < 0 or dst.min() < 0
                                      or src.max() >= num_vertices
                                      or dst.max() >= num_vertices):
            raise GraphLoadError("vertex id out of range [0, %d)" % num_vertices)
        w = None
        if weights is not None:
            w64 = np.asarray(weights, dtype=np.int64)
            if w64.shape != src.shape:
                raise GraphLoadError("weights length mismatch")
            if len(w64) and w64.min() < 0:
                raise GraphLoadError("negative edge weight")
            if len(w64) and w64.max() > np.iinfo(np.uint32).max:
                raise GraphLoadError("edge weights must fit uint32 on the device")
            w = np.ascontiguousarray(w64.astype(np.uint32))
        s32 = src if fast else np.ascontiguousarray(src.astype(np.int32))
        d32 = dst if fast else np.ascontiguousarray(dst.astype(np.int32))
        h = C.c_void_p()
        try:
            _lib.call("gg_graph_create", device, int(num_vertices), len(s32), _lib.ptr(s32),
                      _lib.ptr(d32), _lib.ptr(w), 1 if symmetric else 0, C.byref(h))
        except ValueError as e:
            raise GraphLoadError(str(e)) from None
        g = cls(h, device, diagnostics)
        g._host.update({"coo_src": s32, "coo_dst": d32})
        if w is not None:
            g._host["coo_weights"] = w
        return g

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h is not None:
            _lib.load().gg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- host views (fetched lazily from the device) -----------------------
    def _array(self, name):
        a = self._host.get(name)
        if a is None:
            which, dt = _ARR[name]
            if name.endswith("weights") and not self.weighted:
                return None
            n = self.num_vertices + 1 if name.endswith("offsets") else self.num_edges
            a = np.empty(n, dtype=dt)
            if n:
                _lib.call("gg_graph_copy_array", self._h, which, _lib.ptr(a))
            self._host[name] = a
        return a

    def __getattr__(self, name):
        if name in _ARR and "_host" in self.__dict__:
            return self._array(name)
        raise AttributeError(name)

    def out_degrees(self):
        return np.diff(self._array("out_offsets"))

    def edges(self):
        w = self.coo_weights
        for i in range(self.num_edges):
            yield (int(self.coo_src[i]), int(self.coo_dst[i]),
                   None if w is None else int(w[i]))

    def edge_multiset(self):
        w = self.coo_weights if self.weighted else np.zeros(self.num_edges, np.uint32)
        return sorted(zip(self.coo_src.tolist(), self.coo_dst.tolist(), w.tolist()))

    def drop_coo(self):
        """Free the COO view on the device (CSR views stay)."""
        _lib.call("gg_graph_drop_coo", self._h)


def out_degree(g, v):
    if not 0 <= v < g.num_vertices:
        raise ValueError("vertex id %d out of range [0, %d)" % (v, g.num_vertices))
    off = g.out_offsets
    return int(off[v + 1] - off[v])


def in_degree(g, v):
    if not 0 <= v < g.num_vertices:
        raise ValueError("vertex id %d out of range [0, %d)" % (v, g.num_vertices))
    off = g.in_offsets
    return int(off[v + 1] - off[v])


def symmetrize_coo(src, dst, weights=None):
    """Each arc and its mirror once, first occurrence wins (graphio.py:118-140).

    Vectorised: candidates are emitted in the reference's order (u,v), (v,u)
    per input arc; a stable unique keeps the first occurrence.
    """
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    a = np.empty(2 * len(src), np.int64)
    b = np.empty(2 * len(src), np.int64)
    a[0::2], a[1::2] = src, dst
    b[0::2], b[1::2] = dst, src
    key = a * (int(max(a.max(initial=0), b.max(initial=0))) + 1) + b
    _, first = np.unique(key, return_index=True)
    keep = np.sort(first)
    w2 = None
    if weights is not None:
        w = np.asarray(weights, dtype=np.int64)
        w2 = np.repeat(w, 2)[keep]
    return a[keep], b[keep], w2, int(2 * len(src) - len(keep))


def load_edge_list(path, weighted=False, symmetrize=False, device=0):
    """Whitespace edge list ("src dst [w]"), '#'/'%' comments (graphio.py:143-191)."""
    src, dst, wts = [], [], [] if weighted else None
    comments = 0
    with open(path) as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.strip()
            if not line:
                continue
            if line[0] in "#%":
                comments += 1
                continue
            parts = line.split()
            if len(parts) < 2:
                raise GraphLoadError("%s:%d: malformed edge line %r" % (path, lineno, line))
            try:
                u, v = int(parts[0]), int(parts[1])
            except ValueError:
                raise GraphLoadError("%s:%d: non-integer vertex id in %r"
                                     % (path, lineno, line)) from None
            if u < 0 or v < 0:
                raise GraphLoadError("%s:%d: negative vertex id" % (path, lineno))
            if weighted:
                if len(parts) < 3:
                    raise GraphLoadError("%s:%d: missing weight token" % (path, lineno))
                try:
                    wt = int(parts[2])
                except ValueError:
                    raise GraphLoadError("%s:%d: non-integer weight %r"
                                         % (path, lineno, parts[2])) from None
                if wt < 0:
                    raise GraphLoadError("%s:%d: negative weight" % (path, lineno))
                wts.append(wt)
            src.append(u)
            dst.append(v)
    if not src:
        raise GraphLoadError("%s: no edges" % path)
    diag = {"comment_lines": comments, "input_edges": len(src)}
    if symmetrize:
        src, dst, wts, dropped = symmetrize_coo(src, dst, wts)
        diag["duplicates_collapsed"] = dropped
    n = int(max(max(src), max(dst))) + 1
    return Graph.from_coo(n, src, dst, wts, symmetric=symmetrize, diagnostics=diag,
                          device=device)


def load_matrix_market(path, weighted=False, device=0):
    """MatrixMarket coordinate file (graphio.py:193-261): 1-based ids, a
    'symmetric' banner mirrors every off-diagonal entry, integer values as
    weights; the declared dimensions bound the ids."""
    with open(path) as fh:
        banner = fh.readline()
        if not banner.startswith("%%MatrixMarket matrix coordinate"):
            raise GraphLoadError("%s: not a MatrixMarket coordinate file" % path)
        tok = banner.strip().lower().split()
        fld = tok[3] if len(tok) > 3 else "pattern"
        symmetric = len(tok) > 4 and tok[4] == "symmetric"
        if weighted and fld == "pattern":
            raise GraphLoadError("%s: pattern matrix has no weights" % path)
        lineno, dims = 1, None
        src, dst, wts = [], [], ([] if weighted else None)
        for raw in fh:
            lineno += 1
            line = raw.strip()
            if not line or line[0] == "%":
                continue
            parts = line.split()
            if dims is None:
                if len(parts) != 3:
                    raise GraphLoadError("%s:%d: bad size line %r" % (path, lineno, line))
                dims = [int(x) for x in parts]
                if dims[0] != dims[1]:
                    raise GraphLoadError("%s: adjacency matrix must be square" % path)
                continue
            if len(parts) < 2:
                raise GraphLoadError("%s:%d: malformed entry %r" % (path, lineno, line))
            i, j = int(parts[0]) - 1, int(parts[1]) - 1
            if i < 0 or j < 0:
                raise GraphLoadError("%s:%d: ids are 1-based" % (path, lineno))
            if weighted:
                if len(parts) < 3:
                    raise GraphLoadError("%s:%d: missing value token" % (path, lineno))
                val = float(parts[2])
                if val != int(val) or val < 0:
                    raise GraphLoadError("%s:%d: weights must be non-negative integers"
                                         % (path, lineno))
            pairs = [(i, j)] + ([(j, i)] if symmetric and i != j else [])
            for a, b in pairs:
                src.append(a)
                dst.append(b)
                if weighted:
                    wts.append(int(val))
    if dims is None:
        raise GraphLoadError("%s: missing size line" % path)
    if not src:
        raise GraphLoadError("%s: no edges" % path)
    n = dims[0]
    if max(max(src), max(dst)) >= n:
        raise GraphLoadError("%s: entry outside declared dimensions" % path)
    return Graph.from_coo(n, src, dst, wts, symmetric=symmetric,
                          diagnostics={"declared_nnz": dims[2]}, device=device)


def load_graph(path, weighted=False, symmetrize=False, device=0):
    """MatrixMarket banner or plain edge list (graphio.py:264-278)."""
    with open(path) as fh:
        first = fh.readline()
    if first.startswith("%%MatrixMarket"):
        g = load_matrix_market(path, weighted=weighted, device=device)
        if symmetrize and not g.symmetric:
            s, d, w, dropped = symmetrize_coo(g.coo_src, g.coo_dst, g.coo_weights)
            g = Graph.from_coo(g.num_vertices, s, d, w, symmetric=True,
                               diagnostics=dict(g.diagnostics, duplicates_collapsed=dropped),
                               device=device)
        return g
    return load_edge_list(path, weighted=weighted, symmetrize=symmetrize, device=device)


def with_random_weights(g, low=1, high=1000, seed=0):
    """Copy with uniform integer weights in [low, high] (graphio.py:279-284).

    Uses the same stdlib MT19937 stream as the reference, so the weights are
    identical for the same seed.
    """
    rng = random.Random(seed)
    w = [rng.randint(low, high) for _ in range(g.num_edges)]
    return Graph.from_coo(g.num_vertices, g.coo_src, g.coo_dst, w, symmetric=g.symmetric,
                          diagnostics=dict(g.diagnostics), device=g.device)


# ---------------------------------------------------------------------------
# Synthetic inputs generated on the device
# ---------------------------------------------------------------------------
GEN_RMAT, GEN_KRON, GEN_GRID = 0, 1, 2
F_SYMMETRIZE, F_PERMUTE, F_WEIGHTS, F_SORT_BY_SOURCE = 1, 2, 4, 8


def _generate(kind, scale, edge_factor, a, b, c, seed, flags, device):
    h = C.c_void_p()
    _lib.call("gg_generate", device, kind, scale, edge_factor, a, b, c, seed, flags,
              C.byref(h))
    return Graph(h, device, {"generator": kind, "scale": scale, "edge_factor": edge_factor,
                             "seed": seed, "flags": flags})


def generate_rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, symmetrize=False,
                  permute=False, weights=False, sort_by_source=False, device=0):
    flags = ((F_SYMMETRIZE if symmetrize else 0) | (F_PERMUTE if permute else 0)
             | (F_WEIGHTS if weights else 0) | (F_SORT_BY_SOURCE if sort_by_source else 0))
    return _generate(GEN_RMAT, scale, edge_factor, a, b, c, seed, flags, device)


def generate_kronecker(scale, edge_factor=16, seed=5, symmetrize=True, weights=False,
                       sort_by_source=False, device=0):
    flags = ((F_SYMMETRIZE if symmetrize else 0) | (F_WEIGHTS if weights else 0)
             | (F_SORT_BY_SOURCE if sort_by_source else 0))
    return _generate(GEN_KRON, scale, edge_factor, 0.57, 0.19, 0.19, seed, flags, device)


def generate_grid(side, seed=4, weights=True, device=0):
    return _generate(GEN_GRID, side, 0, 0.0, 0.0, 0.0, seed, F_WEIGHTS if weights else 0, device)
