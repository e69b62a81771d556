"""verify / tune on the GPU (reference cli.py verify scenarios + tuning.tune)."""

import json

import pytest

torch = pytest.importorskip("torch")

from paper_2504_19442_b200 import cli  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("doc", [
    {"scenario": "ag-gemm", "world": {"world_size": 4}, "trials": 2},
    {"scenario": "gemm-rs", "world": {"world_size": 4}, "trials": 2},
    {"scenario": "allgather-push", "world": {"world_size": 8}, "trials": 2},
    {"scenario": "allgather-pull", "world": {"world_size": 4}, "trials": 2},
    {"scenario": "reducescatter", "world": {"world_size": 8}, "trials": 2},
])
def test_verify_scenarios_pass(tmp_path, capsys, doc):
    p = tmp_path / "s.json"
    p.write_text(json.dumps(doc))
    rc = cli.main(["verify", "--config", str(p), "--out", str(tmp_path), "--seed", "3"])
    out = json.loads(capsys.readouterr().out)
    assert rc == cli.EXIT_OK and out["ok"] and out["mismatches"] == []
    assert (tmp_path / f"{doc['scenario']}_summary.json").exists()


def test_tune_ag_gemm_tile(tmp_path, capsys):
    doc = {"scenario": "ag-gemm-tile", "world": {"world_size": 2, "heap_bytes": 1 << 26},
           "problem": {"m": 2560, "n": 2048, "k": 1024}, "iterations": 2,
           "axes": {"bn": [256, 128], "stream_k": [0, 1]}}
    p = tmp_path / "t.json"
    p.write_text(json.dumps(doc))
    rc = cli.main(["tune", "--config", str(p), "--out", str(tmp_path)])
    out = json.loads(capsys.readouterr().out)
    assert rc == cli.EXIT_OK
    assert out["chosen_config"] in [{"bn": b, "stream_k": s} for b in (256, 128) for s in (0, 1)]
    report = json.loads((tmp_path / "ag-gemm-tile_report.json").read_text())
    assert len(report["configs"]) == 4 and all(sc > 0 for sc in report["scores"])
    assert report["per_rank_chosen"] == [report["chosen_index"]] * 2


def test_tune_subchunk_and_reduction_knobs(tmp_path, capsys):
    # the ag-gemm-tile scenario over the sub-chunking knob (AG) on a W=2
    # world; every candidate runs bit-exact and the choice is unanimous
    doc = {"scenario": "ag-gemm-tile", "world": {"world_size": 2, "heap_bytes": 1 << 26},
           "problem": {"m": 1024, "n": 512, "k": 512}, "iterations": 2,
           "axes": {"subchunks": [0, 2], "rs_reduce": ["auto", "separate"]}}
    p = tmp_path / "t.json"
    p.write_text(json.dumps(doc))
    rc = cli.main(["tune", "--config", str(p), "--out", str(tmp_path)])
    out = json.loads(capsys.readouterr().out)
    assert rc == cli.EXIT_OK, out
    report = json.loads((tmp_path / "ag-gemm-tile_report.json").read_text())
    assert len(report["configs"]) == 4 and all(sc and sc > 0 for sc in report["scores"])
    assert report["per_rank_chosen"] == [report["chosen_index"]] * 2
