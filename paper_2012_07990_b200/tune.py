"""GPU-backed schedule autotuner (reference `schedge tune`,
cli.py:210-283, over the space of sched.enumerate_space, sched.py:442-489).

Same candidate list as the reference -- the algorithm's default schedule
first, then the valid cross product of its observable dimensions (delta
variants for sssp), optionally shuffled and truncated -- but every trial runs
on the device and is timed by the library's CUDA events
(``RunStats.kernel_ms``), median of ``repeats`` runs after ``warmup``.

``check=True`` is the reference's ``--check`` (cli.py:262-270): every trial
is compared with the independent host checker (``checkers``, the reference's
oracle.py) when the graph is within its size guard, or with a caller-supplied
``expected`` answer; past the guard with no ``expected``, trials are compared
with the default schedule's device result (BFS levels, CC labels and SSSP
distances exactly, PageRank within 1e-6 and BC within 1e-5 relative).
"""

from __future__ import annotations

import csv
import random
import statistics
import time
from dataclasses import dataclass, field

import numpy as np

from . import algos, checkers
from .sched import Schedule, ScheduleError, ScheduleProgram, enumerate_space, pretty_print

# cli.py:21-29
ALGO_DIMENSIONS = {
    "bfs": ["direction", "pull_frontier_repr", "load_balance", "blocking",
            "frontier_creation", "dedup", "dedup_strategy", "kernel_fusion"],
    "pagerank": ["direction", "load_balance", "blocking", "kernel_fusion"],
    "sssp": ["load_balance", "blocking", "kernel_fusion"],
    "cc": ["direction", "load_balance", "blocking", "kernel_fusion"],
    "bc": ["direction", "pull_frontier_repr", "load_balance",
           "frontier_creation", "dedup", "dedup_strategy"],
}
SSSP_DELTA_CANDIDATES = (1, 4, 16, 64, 256)  # cli.py:31


def candidate_schedules(algo, seed=0, strategy="exhaustive", limit=None, deltas=None):
    """The default schedule, then the valid cross product (cli.py:210-229)."""
    if algo not in ALGO_DIMENSIONS:
        raise ValueError("unknown algorithm %r" % algo)
    candidates = list(enumerate_space(ALGO_DIMENSIONS[algo]).schedules)
    if algo == "sssp":
        extended = []
        for s in candidates:
            for delta in (deltas or SSSP_DELTA_CANDIDATES):
                c = s.copy()
                c.delta = delta
                extended.append(c)
        candidates = extended
    if strategy == "random":
        random.Random(seed).shuffle(candidates)
    elif strategy != "exhaustive":
        raise ValueError("strategy must be 'exhaustive' or 'random'")
    if limit is not None:
        candidates = candidates[:limit]
    return [algos.default_schedule(algo)] + candidates


def program_for(candidate):
    """s0:s1 = the candidate; s0 = a fusion-enabled loop when asked (cli.py:232-239)."""
    program = ScheduleProgram()
    program.bindings["s0:s1"] = candidate.copy()
    if candidate.kernel_fusion:
        program.bindings["s0"] = Schedule(kernel_fusion=True)
    return program


def _run(algo, g, program, source, sources, max_iters, exec_cfg):
    if algo == "bfs":
        return algos.bfs(g, source, program, exec_cfg)
    if algo == "pagerank":
        return algos.pagerank(g, program, exec_cfg, max_iters=max_iters, tolerance=0.0)
    if algo == "sssp":
        return algos.sssp_delta(g, source, program, exec_cfg)
    if algo == "cc":
        return algos.cc_soman(g, program, exec_cfg)
    return algos.bc(g, sources, program, exec_cfg)


def _agrees(algo, got, want):
    a, b = np.asarray(got.array), np.asarray(want.array)
    if algo == "bfs":
        return algos.bfs_levels(a) == algos.bfs_levels(b)
    if algo in ("cc", "sssp"):
        return bool(np.array_equal(a, b))
    tol = 1e-6 if algo == "pagerank" else 1e-5
    big = np.abs(b) > 1e-12
    rel = np.abs(a[big] - b[big]) / np.abs(b[big])
    return bool(rel.max(initial=0.0) <= tol and np.all(np.abs(a[~big] - b[~big]) <= 1e-9))


@dataclass
class Trial:
    schedule_id: int
    serialized_schedule: str
    median_ms: float | None
    passed: str  # "true" / "false" / "" (not checked) / "error: ..."


@dataclass
class TuneResult:
    best_program: ScheduleProgram | None
    best_ms: float | None
    trials: list = field(default_factory=list)
    candidates: int = 0
    seconds: float = 0.0

    def write(self, trials_path=None, out_path=None):
        """The reference's two artefacts: trials CSV and the best program text."""
        if trials_path:
            with open(trials_path, "w", newline="") as fh:
                w = csv.writer(fh)
                w.writerow(["schedule_id", "serialized_schedule", "median_ms", "pass"])
                for t in self.trials:
                    w.writerow([t.schedule_id, t.serialized_schedule,
                                "" if t.median_ms is None else "%.4f" % t.median_ms, t.passed])
        if out_path and self.best_program is not None:
            with open(out_path, "w") as fh:
                fh.write(pretty_print(self.best_program))


def _check_values(algo, result):
    a = np.asarray(result.array)
    return a.tolist()


def tune(algo, g, budget_s=60.0, *, source=0, sources=None, max_iters=20, exec_cfg=None,
         seed=0, strategy="exhaustive", limit=None, deltas=None, warmup=1, repeats=3,
         check=False, expected=None):
    """Time every candidate on the device within ``budget_s`` seconds (the
    first candidate always runs); the fastest median wins, among trials that
    pass the check when ``check`` is set.  ``expected``: the answer to check
    against, in ``checkers.compare`` form (levels for bfs, inf for sssp)."""
    if budget_s <= 0:
        raise ValueError("budget must be positive (seconds)")
    sources = list(sources) if sources is not None else [source]
    cands = candidate_schedules(algo, seed=seed, strategy=strategy, limit=limit, deltas=deltas)
    res = TuneResult(None, None, candidates=len(cands))
    reference = None
    if check and expected is None and g.num_vertices <= checkers.ORACLE_MAX_VERTICES:
        expected = checkers.expected(algo, g, source=source, sources=sources,
                                     max_iters=max_iters, tolerance=0.0)
    t0 = time.perf_counter()
    for idx, cand in enumerate(cands):
        if idx > 0 and time.perf_counter() - t0 > budget_s:
            break
        program = program_for(cand)
        text = pretty_print(program).replace("\n", " ").strip()
        try:
            for _ in range(warmup):
                _run(algo, g, program, source, sources, max_iters, exec_cfg)
            times, result = [], None
            for _ in range(max(1, repeats)):
                result = _run(algo, g, program, source, sources, max_iters, exec_cfg)
                times.append(result.stats.kernel_ms)
        except (ScheduleError, ValueError) as exc:
            res.trials.append(Trial(idx, text, None, "error: %s" % exc))
            continue
        med = statistics.median(times)
        ok = ""
        if check and expected is not None:
            ok = "true" if checkers.compare(algo, _check_values(algo, result), expected)[0] \
                else "false"
        elif check:
            if reference is None:
                reference = result
                ok = "true"
            else:
                ok = "true" if _agrees(algo, result, reference) else "false"
        res.trials.append(Trial(idx, text, med, ok))
        if ok != "false" and (res.best_ms is None or med < res.best_ms):
            res.best_ms, res.best_program = med, program
    res.seconds = time.perf_counter() - t0
    return res
