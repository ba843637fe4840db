"""Schedule language parity with the reference DSL (sched.py); host only."""

import pytest

from paper_2012_07990_b200.sched import (DIMENSIONS, HybridSchedule, ParseError, Schedule,
                                         ScheduleError, ScheduleProgram, enumerate_space,
                                         parse_schedule, pretty_print, schedule_key, validate,
                                         validate_hybrid)

HYBRID_BFS_TEXT = """
SimpleGPUSchedule s1;
s1.configDirection(PUSH);
s1.configLoadBalance(VERTEX_BASED);
SimpleGPUSchedule s2 = s1;
s2.configDirection(PULL, BITMAP);
s2.configDeduplication(DISABLED);
s2.configLoadBalance(VERTEX_BASED);
s2.configFrontierCreation(UNFUSED_BITMAP);
HybridGPUSchedule h1(VERTEXSET_SIZE, "argv[3]", s1, s2);
apply("s0:s1", h1);
"""


def test_hybrid_program_structure():
    h = parse_schedule(HYBRID_BFS_TEXT).binding("s0:s1")
    assert isinstance(h, HybridSchedule)
    assert h.criteria == "INPUT_VERTEXSET_SIZE" and h.threshold == "argv[3]"
    assert h.s1.direction == "PUSH" and h.s1.load_balance == "VERTEX_BASED"
    assert h.s2.direction == "PULL" and h.s2.pull_frontier_repr == "BITMAP"
    assert h.s2.dedup is False and h.s2.frontier_creation == "UNFUSED_BITMAP"


def test_defaults_and_empty():
    assert parse_schedule("").bindings == {}
    s = Schedule()
    assert (s.direction, s.pull_frontier_repr, s.load_balance, s.blocking,
            s.frontier_creation, s.dedup, s.dedup_strategy, s.kernel_fusion) == (
        "PUSH", "BOOLMAP", "VERTEX_BASED", False, "FUSED", True, "MONOTONIC_COUNTERS", False)
    assert validate(s) == []


def test_errors_carry_positions():
    with pytest.raises(ParseError, match="invalid direction value 'SIDEWAYS'") as err:
        parse_schedule("SimpleGPUSchedule s1;\ns1.configDirection(SIDEWAYS);")
    assert err.value.line == 2
    with pytest.raises(ParseError, match="line 1"):
        parse_schedule("SimpleGPUSchedule ;")
    with pytest.raises(ParseError, match="unknown config function"):
        parse_schedule("SimpleGPUSchedule s;\ns.configApplyDirection(PUSH);")
    with pytest.raises(ParseError, match="argument"):
        parse_schedule("SimpleGPUSchedule s;\ns.configDelta(1, 2);")
    with pytest.raises(ParseError, match="unknown SimpleGPUSchedule"):
        parse_schedule("s1.configDirection(PUSH);")
    with pytest.raises(ParseError, match="unknown schedule"):
        parse_schedule('apply("s0", nope);')
    with pytest.raises(ParseError, match="delta"):
        parse_schedule("SimpleGPUSchedule s;\ns.configDelta(0);")
    with pytest.raises(ParseError, match="bound twice"):
        parse_schedule('SimpleGPUSchedule s;\napply("a", s);\napply("a", s);')
    with pytest.raises(ParseError, match="unexpected character"):
        parse_schedule("SimpleGPUSchedule s; @")


def test_copy_is_deep_and_comments():
    p = parse_schedule("// c\nSimpleGPUSchedule s1; // t\ns1.configDirection(PULL, BITMAP);\n"
                       "SimpleGPUSchedule s2 = s1;\ns2.configDirection(PUSH);\ns2.configDelta(9);\n"
                       'apply("a", s1);\napply("b", s2);\n')
    assert p.binding("a").direction == "PULL" and p.binding("a").delta == 1
    assert p.binding("b").direction == "PUSH" and p.binding("b").delta == 9


def test_validation_rules():
    assert any("EDGE_ONLY" in m for m in validate(Schedule(load_balance="ETWC", blocking=True)))
    assert validate(Schedule(load_balance="EDGE_ONLY", blocking=True)) == []
    assert any("delta" in m for m in validate(Schedule(delta=0)))
    assert any("threshold" in m for m in validate_hybrid(HybridSchedule(threshold=1.5)))


def test_space_counts_and_round_trip():
    space = enumerate_space()
    assert space.raw_count == 2016 and space.valid_count == 1152
    for field, values in DIMENSIONS.values():
        for value in values:
            s = Schedule(**{field: value})
            if s.blocking:
                s.load_balance = "EDGE_ONLY"
            p = ScheduleProgram({"s0:s1": s})
            assert parse_schedule(pretty_print(p)).binding("s0:s1") == s
    for s in space.schedules[::97]:
        p = ScheduleProgram({"s0:s1": s})
        assert parse_schedule(pretty_print(p)).binding("s0:s1") == s
    h = parse_schedule(HYBRID_BFS_TEXT)
    assert parse_schedule(pretty_print(h)).binding("s0:s1") == h.binding("s0:s1")


def test_resolve_args_and_keys():
    p = parse_schedule(HYBRID_BFS_TEXT)
    with pytest.raises(ScheduleError, match="argv"):
        p.resolve_args({})
    p.resolve_args({3: "0.2"})
    assert p.binding("s0:s1").threshold == 0.2
    assert schedule_key(Schedule(direction="PULL", delta=4)) == \
        "PULL/BOOLMAP/VERTEX_BASED/FUSED/DEDUP/MONOTONIC_COUNTERS/UNBLOCKED/NOFUSE/delta4"
