"""Stream programs, host side (no GPU): validation and planning
(contract of the reference's tests/test_tasks.py, re-expressed)."""

import pytest

from paper_2504_19442_b200 import SynchronizationFault, UsageError
from paper_2504_19442_b200.tasks import Stream, TaskRole, copy_async, plan, stream_wait


def names(order):
    return [(s.name, op[1] if op[0] == "call" else "join") for s, op in order]


def test_cross_rank_join_rejected():
    with pytest.raises(UsageError):
        stream_wait(Stream(1, "s1"), Stream(0, "s0"))


def test_copy_engine_stream_roles():
    with pytest.raises(UsageError):
        copy_async(Stream(0, "comm", TaskRole.COMM_BLOCK), None, None)
    ce = Stream(0, "ce", TaskRole.COPY_ENGINE)
    with pytest.raises(UsageError):
        ce.enqueue(lambda pe: None, "gemm", kind="compute")
    ce.enqueue(lambda pe: None, "signal")  # signals / transfers are fine
    assert ce.task_count() == 1


def test_join_count_fixed_when_recorded():
    s0, s1 = Stream(0, "s0"), Stream(0, "s1")
    s0.enqueue(lambda pe: None, "a")
    s1.wait(s0)              # the one task s0 holds now
    s0.enqueue(lambda pe: None, "b")
    s1.wait(s0, upto=3)      # an explicit count may name later tasks
    assert [op[2] for op in s1.ops] == [1, 3]
    assert s0.task_count() == 2 and s1.task_count() == 0


def test_plan_respects_fifo_and_joins():
    s0, s1 = Stream(0, "s0"), Stream(0, "s1")
    s1.enqueue(lambda pe: None, "E")
    s1.wait(s0, upto=1)
    s1.enqueue(lambda pe: None, "B")
    s0.enqueue(lambda pe: None, "A")
    order = names(plan([s1, s0]))
    assert order.index(("s1", "E")) < order.index(("s1", "B"))
    assert order.index(("s0", "A")) < order.index(("s1", "B"))


def test_plan_chained_joins_transitive():
    s0, s1, s2 = (Stream(0, f"s{i}") for i in range(3))
    s0.enqueue(lambda pe: None, "t0")
    s1.wait(s0)
    s1.enqueue(lambda pe: None, "t1")
    s2.wait(s1)
    s2.enqueue(lambda pe: None, "t2")
    calls = [n for n in names(plan([s2, s1, s0])) if n[1] != "join"]
    assert calls == [("s0", "t0"), ("s1", "t1"), ("s2", "t2")]


def test_plan_refuses_a_cycle_naming_both_streams():
    s0, s1 = Stream(0, "s0"), Stream(0, "s1")
    s0.wait(s1, upto=1)
    s0.enqueue(lambda pe: None, "a")
    s1.wait(s0, upto=1)
    s1.enqueue(lambda pe: None, "b")
    with pytest.raises(SynchronizationFault) as info:
        plan([s0, s1])
    assert "s0" in str(info.value) and "s1" in str(info.value)


def test_plan_refuses_a_join_outside_the_program():
    s0, other = Stream(0, "s0"), Stream(0, "elsewhere")
    other.enqueue(lambda pe: None, "x")
    s0.wait(other)
    with pytest.raises(SynchronizationFault, match="not in this program"):
        plan([s0])


def test_join_on_empty_stream_is_noop():
    s0, s1 = Stream(0, "s0"), Stream(0, "s1")
    s1.wait(s0)
    s1.enqueue(lambda pe: None, "only")
    assert names(plan([s0, s1])) == [("s1", "join"), ("s1", "only")]
