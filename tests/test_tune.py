"""Autotuner: candidate lists equal the reference
tuner's (golden from oracle/make_golden.py), and a GPU-timed tune run."""

import json
import os

import numpy as np
import pytest

from paper_2012_07990_b200 import tune
from paper_2012_07990_b200.sched import schedule_key
from tests.conftest import GOLDEN


def test_candidates_match_reference_tuner():
    want = json.load(open(os.path.join(GOLDEN, "tune_candidates.json")))
    for algo, rec in want.items():
        c = tune.candidate_schedules(algo)
        assert len(c) == rec["n"], algo
        assert [schedule_key(s) for s in c[:5]] == rec["first5"], algo
        r = tune.candidate_schedules(algo, seed=3, strategy="random", limit=7)
        assert [schedule_key(s) for s in r] == rec["random3_7"], algo


def test_program_for_binds_fusion_loop():
    from paper_2012_07990_b200 import Schedule
    p = tune.program_for(Schedule(kernel_fusion=True))
    assert set(p.bindings) == {"s0", "s0:s1"} and p.bindings["s0"].kernel_fusion
    assert set(tune.program_for(Schedule()).bindings) == {"s0:s1"}
    with pytest.raises(ValueError):
        tune.candidate_schedules("nope")
    with pytest.raises(ValueError):
        tune.candidate_schedules("bfs", strategy="bogus")


@pytest.mark.gpu
def test_tune_on_device(tmp_path):
    import paper_2012_07990_b200 as gg
    g = gg.generate_rmat(10, 8, seed=4, symmetrize=True)
    import oracle
    V = g.num_vertices
    want_cc, _ = oracle.cc(V, g.coo_src, g.coo_dst)
    # every trial judged against the oracle's labels (not the default schedule)
    res = tune.tune("cc", g, budget_s=30.0, repeats=1, warmup=0, check=True,
                    expected=want_cc.tolist())
    assert res.best_program is not None and res.best_ms > 0
    assert all(t.passed == "true" for t in res.trials if not t.passed.startswith("error"))
    assert len(res.trials) == res.candidates
    res.write(str(tmp_path / "trials.csv"), str(tmp_path / "best.sched"))
    best = gg.parse_schedule(open(tmp_path / "best.sched").read())
    assert gg.cc_soman(g, best).array is not None
    off, nbr, _ = oracle.csr(V, g.coo_src, g.coo_dst)
    want_lv = oracle.bfs_levels(V, off, nbr, 1).tolist()
    resb = tune.tune("bfs", g, budget_s=5.0, source=1, repeats=1, warmup=0, check=True, limit=40,
                     expected=want_lv)
    assert all(t.passed == "true" or t.passed.startswith("error") for t in resb.trials)
    want_pr, _ = oracle.pagerank(V, g.coo_src, g.coo_dst, 10, 0.0)
    resp = tune.tune("pagerank", g, budget_s=30.0, repeats=1, warmup=0, check=True, max_iters=10,
                     expected=want_pr.tolist())
    assert all(t.passed == "true" for t in resp.trials if t.median_ms is not None)
    # a wrong expected answer fails every trial (the check is not self-referential)
    bad = tune.tune("cc", g, budget_s=5.0, repeats=1, warmup=0, check=True, limit=3,
                    expected=[0] * V)
    assert all(t.passed == "false" for t in bad.trials if t.median_ms is not None)
    assert bad.best_program is None
