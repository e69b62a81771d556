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
