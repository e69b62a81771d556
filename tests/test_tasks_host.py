"""Task-layer validation that needs no GPU (reference tests/test_tasks.py)."""

import pytest

from paper_2504_19442_b200 import UsageError
from paper_2504_19442_b200.tasks import (BlockAssignment, Stream, TaskRole, copy_async,
                                         stream_wait)


def test_cross_rank_wait_rejected():
    s0 = Stream(0, "s0")
    s1 = Stream(1, "s1")
    with pytest.raises(UsageError):
        stream_wait(s1, s0)


def test_copy_async_requires_copy_engine_role():
    comm = Stream(0, "comm", TaskRole.COMM_BLOCK)
    with pytest.raises(UsageError):
        copy_async(comm, None, None)
    ce = Stream(0, "ce", TaskRole.COPY_ENGINE)
    with pytest.raises(UsageError):
        ce.enqueue(lambda pe: None, "compute", kind="compute")


def test_role_mapping_block_assignment():
    BlockAssignment({0: "send", 1: "recv"})
    with pytest.raises(UsageError):
        BlockAssignment({0: "send", 2: "recv"})


def test_wait_watermarks_recorded_at_construction():
    s0, s1 = Stream(0, "s0"), Stream(0, "s1")
    s0.enqueue(lambda pe: None, "a")
    s1.wait(s0)              # waits for the one task s0 holds now
    s0.enqueue(lambda pe: None, "b")
    s1.wait(s0, upto=3)      # explicit count, may reference later tasks
    assert s1.items[0].watermark == 1 and s1.items[1].watermark == -3
    assert s0.task_count() == 2 and s1.task_count() == 0
