"""CLI contract on CPU: list-scenarios, usage errors and exit codes
(reference tests/test_cli.py); GPU scenarios in test_gpu_cli_tuning.py."""

import json

from paper_2504_19442_b200 import cli


def test_list_scenarios(capsys):
    assert cli.main(["list-scenarios"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    for name in ("ag-gemm", "gemm-rs", "allgather-push", "allgather-pull", "reducescatter",
                 "ag-gemm-tile"):
        assert name in out


def test_missing_config_file_is_usage_error(tmp_path, capsys):
    assert cli.main(["verify", "--config", str(tmp_path / "nope.json")]) == cli.EXIT_USAGE


def test_bad_json_is_usage_error(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text("{not json")
    assert cli.main(["verify", "--config", str(p)]) == cli.EXIT_USAGE


def test_unknown_keys_and_scenarios_are_usage_errors(tmp_path):
    p = tmp_path / "s.json"
    p.write_text(json.dumps({"scenario": "ag-gemm", "bogus": 1}))
    assert cli.main(["verify", "--config", str(p)]) == cli.EXIT_USAGE
    p.write_text(json.dumps({"scenario": "nope"}))
    assert cli.main(["verify", "--config", str(p)]) == cli.EXIT_USAGE
    p.write_text(json.dumps({"scenario": "ag-gemm", "world": {"cores": 3}}))
    assert cli.main(["verify", "--config", str(p)]) == cli.EXIT_USAGE
    p.write_text(json.dumps({"scenario": "ag-gemm"}))
    assert cli.main(["tune", "--config", str(p)]) == cli.EXIT_USAGE


def test_emitted_documents_are_schema_checked(tmp_path):
    """Every file the CLI writes is validated against its contract first
    (reference cli.py:78-85): a conforming summary is written, a broken one
    is a usage error naming the document."""
    import pytest

    from paper_2504_19442_b200 import schemas
    from paper_2504_19442_b200.errors import ConfigurationError

    ok = {"scenario": "ag-gemm", "kind": "verify", "ok": True, "mismatches": []}
    path = cli._emit(tmp_path, "s_summary.json", ok, "summary")
    assert json.loads(open(path).read()) == ok
    with pytest.raises(ConfigurationError, match="summary schema"):
        cli._emit(tmp_path, "bad_summary.json", {"scenario": "x", "kind": "bogus", "ok": 1},
                  "summary")
    report = {"axes": {"bn": [128, 256]}, "configs": [{"bn": 128}, {"bn": 256}],
              "timings_us": [[[1.0, 2.0]], None], "scores": [1.5, None], "chosen_index": 0,
              "chosen_config": {"bn": 128}, "per_rank_chosen": [0], "invalid": {"1": "bad"}}
    schemas.validate(report, "tune_report", "r")
    with pytest.raises(ConfigurationError):
        schemas.validate({**report, "extra": 1}, "tune_report", "r")
    with pytest.raises(ConfigurationError):
        schemas.validate({"scenario": "ag-gemm", "trials": 0}, "scenario", "s")
    schemas.validate({"scenario": "ag-gemm", "world": {"world_size": 2},
                      "problem": {"m": 8, "n": 8, "k": 8, "dtype": "bfloat16"}, "trials": 2},
                     "scenario", "s")
