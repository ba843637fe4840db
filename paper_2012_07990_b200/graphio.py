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
        if (isinstance(weights, np.ndarray) and weights.dtype == np.uint32
                and weights.flags.c_contiguous):
            # already the device's weight type: in range by construction,
            # uploaded as-is (no host passes over the arcs)
            if weights.shape != src.shape:
                raise GraphLoadError("weights length mismatch")
            w = weights
        elif weights is not None:
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

    def prepare_relabel(self):
        """Build the degree-ordered copy that cc_soman / bc query on large
        graphs (relabel.cu; cached on the graph) ahead of the queries and
        return its preprocessing time in ms."""
        ms = C.c_double(0.0)
        _lib.call("gg_relabel_prepare", self._h, C.byref(ms))
        return ms.value


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


def _records(path, skip_first=False):
    """(line number, tokens) of every non-blank, non-comment line."""
    with open(path) as fh:
        for lineno, raw in enumerate(fh, 1):
            if skip_first and lineno == 1:
                continue
            toks = raw.split()
            if toks and toks[0][0] not in "#%":
                yield lineno, toks


def _count_comments(path):
    with open(path) as fh:
        return sum(1 for raw in fh if raw.strip()[:1] in ("#", "%"))


def _as_int(tok, where, what):
    try:
        return int(tok)
    except ValueError:
        raise GraphLoadError("%s: non-integer %s %r" % (where, what, tok)) from None


class _Columns:
    """Growing src / dst / weight columns with the loaders' checks."""

    def __init__(self, weighted):
        self.src, self.dst = [], []
        self.w = [] if weighted else None

    def add(self, u, v, w=None):
        self.src.append(u)
        self.dst.append(v)
        if self.w is not None:
            self.w.append(w)

    def arrays(self):
        s = np.asarray(self.src, np.int64)
        d = np.asarray(self.dst, np.int64)
        return s, d, (None if self.w is None else np.asarray(self.w, np.int64))


def load_edge_list(path, weighted=False, symmetrize=False, device=0):
    """"src dst [weight]" per line, '#'/'%' comments (the reference's
    graphio.load_edge_list contract, graphio.py:143-191: same errors, a
    trailing weight ignored unless ``weighted``, ids from 0)."""
    cols = _Columns(weighted)
    for lineno, toks in _records(path):
        where = "%s:%d" % (path, lineno)
        if len(toks) < 2:
            raise GraphLoadError("%s: malformed edge line %r" % (where, " ".join(toks)))
        try:
            u, v = int(toks[0]), int(toks[1])
        except ValueError:
            raise GraphLoadError("%s: non-integer vertex id in %r"
                                 % (where, " ".join(toks))) from None
        if min(u, v) < 0:
            raise GraphLoadError("%s: negative vertex id" % where)
        w = None
        if weighted:
            if len(toks) < 3:
                raise GraphLoadError("%s: missing weight token" % where)
            w = _as_int(toks[2], where, "weight")
            if w < 0:
                raise GraphLoadError("%s: negative weight" % where)
        cols.add(u, v, w)
    if not cols.src:
        raise GraphLoadError("%s: no edges" % path)
    s, d, w = cols.arrays()
    diag = {"comment_lines": _count_comments(path), "input_edges": len(s)}
    if symmetrize:
        s, d, w, diag["duplicates_collapsed"] = symmetrize_coo(s, d, w)
    n = int(max(s.max(), d.max())) + 1
    return Graph.from_coo(n, s, d, w, symmetric=symmetrize, diagnostics=diag, device=device)


def load_matrix_market(path, weighted=False, device=0):
    """MatrixMarket coordinate file (graphio.py:193-261 contract): 1-based
    ids, a 'symmetric' banner mirrors off-diagonal entries, integer values
    are weights, the size line bounds the ids."""
    with open(path) as fh:
        banner = fh.readline()
    if not banner.startswith("%%MatrixMarket matrix coordinate"):
        raise GraphLoadError("%s: not a MatrixMarket coordinate file" % path)
    head = banner.lower().split()
    value_field = head[3] if len(head) > 3 else "pattern"
    mirror = len(head) > 4 and head[4] == "symmetric"
    if weighted and value_field == "pattern":
        raise GraphLoadError("%s: pattern matrix has no weights" % path)
    rows = None
    cols = _Columns(weighted)
    for lineno, toks in _records(path, skip_first=True):
        where = "%s:%d" % (path, lineno)
        if rows is None:  # the size line
            if len(toks) != 3:
                raise GraphLoadError("%s: bad size line %r" % (where, " ".join(toks)))
            rows, ncols, nnz = (int(x) for x in toks)
            if rows != ncols:
                raise GraphLoadError("%s: adjacency matrix must be square" % path)
            continue
        if len(toks) < 2:
            raise GraphLoadError("%s: malformed entry %r" % (where, " ".join(toks)))
        i, j = int(toks[0]) - 1, int(toks[1]) - 1
        if min(i, j) < 0:
            raise GraphLoadError("%s: ids are 1-based" % where)
        w = None
        if weighted:
            if len(toks) < 3:
                raise GraphLoadError("%s: missing value token" % where)
            val = float(toks[2])
            if val < 0 or val != int(val):
                raise GraphLoadError("%s: weights must be non-negative integers" % where)
            w = int(val)
        cols.add(i, j, w)
        if mirror and i != j:
            cols.add(j, i, w)
    if rows is None:
        raise GraphLoadError("%s: missing size line" % path)
    if not cols.src:
        raise GraphLoadError("%s: no edges" % path)
    s, d, w = cols.arrays()
    if max(s.max(), d.max()) >= rows:
        raise GraphLoadError("%s: entry outside declared dimensions" % path)
    return Graph.from_coo(rows, s, d, w, symmetric=mirror, diagnostics={"declared_nnz": nnz},
                          device=device)


def load_graph(path, weighted=False, symmetrize=False, device=0):
    """Dispatch on the first line: MatrixMarket banner or plain edge list
    (graphio.py:264-278)."""
    with open(path) as fh:
        is_mm = fh.readline().startswith("%%MatrixMarket")
    if not is_mm:
        return load_edge_list(path, weighted=weighted, symmetrize=symmetrize, device=device)
    g = load_matrix_market(path, weighted=weighted, device=device)
    if symmetrize and not g.symmetric:
        s, d, w, dropped = symmetrize_coo(g.coo_src, g.coo_dst, g.coo_weights)
        g = Graph.from_coo(g.num_vertices, s, d, w, symmetric=True,
                           diagnostics=dict(g.diagnostics, duplicates_collapsed=dropped),
                           device=device)
    return g


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
