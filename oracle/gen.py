"""Host (numpy) replicas of the device generators in csrc/graph.cu.

TEST INFRASTRUCTURE ONLY: lets tests generate the same synthetic graphs in
this container (no GPU) for the reference / oracle, and check that the device
generator is bit-identical.  Counter-based: edge i depends only on (seed, i).
"""

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _threshold(p):
    t = p * 4294967296.0
    return np.uint64(4294967295 if t >= 4294967296.0 else int(t))


def rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
    """k_rmat (graph.cu): returns (V, src int32, dst int32) in generation order."""
    V = 1 << scale
    E = V * edge_factor
    i = np.arange(E, dtype=np.uint64)
    ta, tab, tabc = _threshold(a), _threshold(a + b), _threshold(a + b + c)
    s = np.zeros(E, np.uint64)
    d = np.zeros(E, np.uint64)
    seed = np.uint64(seed)
    h = None
    for lvl in range(scale):
        if lvl % 2 == 0:
            with np.errstate(over="ignore"):
                h = mix64(seed ^ mix64(i * np.uint64(64) + np.uint64(lvl)))
        r = (h >> np.uint64(32)) if lvl % 2 else (h & np.uint64(0xFFFFFFFF))
        bs = (r >= tab).astype(np.uint64)
        bd = (((r >= ta) & (r < tab)) | (r >= tabc)).astype(np.uint64)
        s = (s << np.uint64(1)) | bs
        d = (d << np.uint64(1)) | bd
    return V, s.astype(np.int32), d.astype(np.int32)


def weights(E, seed):
    i = np.arange(E, dtype=np.uint64)
    k = mix64(np.uint64(seed ^ 0xA5A5A5A5) ^ mix64(i ^ np.uint64(0x5BD1E995)))
    return (np.uint64(1) + (k % np.uint64(1000))).astype(np.uint32)


def grid(side):
    """k_grid_arcs (graph.cu): CSR-ordered 4-neighbour grid."""
    V = side * side
    u = np.arange(V, dtype=np.int64)
    r, c = u // side, u % side
    cand = [(r > 0, u - side), (c > 0, u - 1), (c < side - 1, u + 1), (r < side - 1, u + side)]
    mask = np.stack([m for m, _ in cand], axis=1)
    nb = np.stack([x for _, x in cand], axis=1)
    src = np.repeat(u, mask.sum(axis=1))
    dst = nb[mask]
    return V, src.astype(np.int32), dst.astype(np.int32)


def sort_by_source(src, dst, w=None):
    order = np.argsort(src, kind="stable")
    return src[order], dst[order], (None if w is None else w[order])
