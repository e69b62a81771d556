"""Tuner aggregation rules (reference tests/test_tuning.py), on CPU with a
stand-in world; the GPU run is in test_gpu_cli_tuning.py."""

import numpy as np
import pytest

from paper_2504_19442_b200.tuning import ConfigSpace, TuneReport, TuningError, tune


class _Pe:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank

    def putmem(self, handle, arr, peer, dst_off=0):
        self.world.mem[peer][:] = np.asarray(arr, dtype=np.int64)[0]

    def barrier_all(self):
        pass

    def local_view(self, handle, dtype, shape):
        import torch

        return torch.tensor([int(self.world.mem[self.rank][0])] * shape[0])


class FakeWorld:
    """Just enough World for tune(): sequential ranks, host memory."""

    _dist = False

    def __init__(self, n):
        self.world_size = n
        self.local_ranks = list(range(n))
        self.mem = [np.zeros(1, dtype=np.int64) for _ in range(n)]
        self.resets = 0
        self.recovered = 0

    def pe(self, r):
        return _Pe(self, r)

    def run(self, fn, timeout=None):
        return [fn(self.pe(r)) for r in range(self.world_size)]

    def zero_all_signals(self):
        self.resets += 1

    def sweep_signals(self):
        return {}

    def recover(self):
        self.recovered += 1

    def alloc_symmetric(self, n, align=8):
        return object()


def injected(table):
    return lambda pe, cfg, it: table[cfg["x"]][pe.rank][it]


def noop(pe, cfg):
    pass


def test_hand_evaluated_aggregation_rule():
    table = {0: [[10.0], [9.0]], 1: [[8.0], [11.0]]}
    w = FakeWorld(2)
    report = tune(w, noop, ConfigSpace({"x": [0, 1]}), iterations=1, warmup=0,
                  measure=injected(table))
    assert report.scores == [10.0, 11.0]
    assert report.chosen_index == 0 and report.per_rank_chosen == [0, 0]


def test_median_then_max():
    table = {0: [[1.0, 9.0, 2.0], [3.0, 3.0, 3.0]], 1: [[2.5, 2.5, 2.5], [2.5, 2.5, 2.5]]}
    report = tune(FakeWorld(2), noop, ConfigSpace({"x": [0, 1]}), iterations=3, warmup=0,
                  measure=injected(table))
    assert report.scores == [3.0, 2.5] and report.chosen_config == {"x": 1}


def test_tie_breaks_to_first_config():
    table = {0: [[5.0], [5.0]], 1: [[5.0], [5.0]]}
    report = tune(FakeWorld(2), noop, ConfigSpace({"x": [0, 1]}), iterations=1, warmup=0,
                  measure=injected(table))
    assert report.chosen_index == 0


def test_every_measurement_starts_from_reset_signals():
    w = FakeWorld(2)
    tune(w, noop, ConfigSpace({"x": [0, 1, 2]}), iterations=2, warmup=1,
         measure=lambda pe, cfg, it: 1.0)
    assert w.resets == 3 * 3


def test_faulting_config_is_marked_invalid():
    from paper_2504_19442_b200 import ArgumentError

    def target(pe, cfg):
        if cfg["x"] == 1:
            raise ArgumentError("bad tile")

    w = FakeWorld(2)
    report = tune(w, target, ConfigSpace({"x": [0, 1]}), iterations=1, warmup=0,
                  measure=lambda pe, cfg, it: 1.0)
    assert report.scores[1] is None and "ArgumentError" in report.invalid[1]
    assert w.recovered == 1


def test_all_invalid_raises():
    def target(pe, cfg):
        from paper_2504_19442_b200 import ShmemError

        raise ShmemError("nope")

    with pytest.raises(TuningError):
        tune(FakeWorld(1), target, ConfigSpace({"x": [0]}), iterations=1, warmup=0,
             measure=lambda pe, cfg, it: 1.0)


def test_space_enumeration_and_validation():
    space = ConfigSpace({"a": [1, 2], "b": ["x", "y"]})
    assert space.configs() == [{"a": 1, "b": "x"}, {"a": 1, "b": "y"},
                               {"a": 2, "b": "x"}, {"a": 2, "b": "y"}]
    assert space.size() == 4
    with pytest.raises(TuningError):
        ConfigSpace({})
    with pytest.raises(TuningError):
        ConfigSpace({"a": []})


def test_report_json_roundtrip():
    import json

    r = TuneReport({"x": [0]}, [{"x": 0}], [[[1.0]]], [1.0], 0, {"x": 0}, [0], {})
    doc = json.loads(r.to_json())
    assert doc["chosen_config"] == {"x": 0} and doc["invalid"] == {}


def test_kernel_config_environment_knobs_restore(monkeypatch):
    # the sub-chunking and reduction-form knobs travel through the library's
    # environment for the block and are restored afterwards
    import os

    from paper_2504_19442_b200 import ConfigurationError
    from paper_2504_19442_b200.tuning import kernel_config

    monkeypatch.setenv("SHB_AG_SUB", "2")
    monkeypatch.delenv("SHB_RS_UNFUSED", raising=False)
    with kernel_config(subchunks=4, rs_reduce="separate"):
        assert os.environ["SHB_AG_SUB"] == "4" and os.environ["SHB_RS_UNFUSED"] == "1"
    assert os.environ["SHB_AG_SUB"] == "2" and "SHB_RS_UNFUSED" not in os.environ
    with kernel_config(subchunks=0, rs_reduce="fused"):
        assert "SHB_AG_SUB" not in os.environ and os.environ["SHB_RS_UNFUSED"] == "0"
    assert os.environ["SHB_AG_SUB"] == "2"
    with pytest.raises(ConfigurationError):
        with kernel_config(rs_reduce="sometimes"):
            pass
