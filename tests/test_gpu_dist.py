"""Partitioned PageRank through NCCL on one GPU (world size 1 communicator);
the multi-rank data path is exercised by bench.py under torchrun."""

import numpy as np
import pytest

import oracle
from oracle import gen

pytestmark = pytest.mark.gpu


def test_pagerank_dist_single_rank_matches_oracle():
    import torch
    import paper_2012_07990_b200 as gg
    from paper_2012_07990_b200.dist import Comm, pagerank_dist
    V, s, d = gen.rmat(12, 16, seed=5)
    g = gg.Graph.from_coo(V, s, d)
    comm = Comm.create(0, 1, 0)
    ranks, st = pagerank_dist(comm, g, max_iters=20, tolerance=0.0)
    want, _ = oracle.pagerank(V, s, d, 20, 0.0)
    assert np.max(np.abs(ranks - want) / want) < 1e-6
    assert st.rounds == 20
    comm.close()
