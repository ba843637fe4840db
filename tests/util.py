"""Shared helpers for the test-suite (graph records, schedule decoding)."""

import numpy as np

from paper_2012_07990_b200.sched import Schedule, ScheduleProgram


def sched_from(d):
    if d is None:
        return None
    return Schedule(**d)


def program_with(s, fusion=False):
    if s is None:
        return None
    p = ScheduleProgram({"s0:s1": s.copy()})
    if fusion:
        p.bindings["s0"] = Schedule(kernel_fusion=True)
    return p


def arrays(rec):
    src = np.asarray(rec["src"], np.int32)
    dst = np.asarray(rec["dst"], np.int32)
    w = None if rec["w"] is None else np.asarray(rec["w"], np.uint32)
    return rec["V"], src, dst, w


def max_rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    denom = np.maximum(np.abs(want), 1e-300)
    return float(np.max(np.abs(got - want) / denom)) if len(want) else 0.0
