"""JSON document contracts of the CLI outputs and inputs (§8 row f4).

The drop-in's verify / tune commands emit the same documents as the
reference CLI (pkg/src/minishmem/cli.py:78-85 validates every emitted file
against its packaged schemas: run summary, tune report, Chrome-trace event
list, scenario input).  The contracts are restated here as JSON Schema
(draft 2020-12) dictionaries and checked with ``jsonschema`` before anything
is written; a violation is a ``ConfigurationError`` naming the document.
"""

from __future__ import annotations

from .errors import ConfigurationError

_DRAFT = "https://json-schema.org/draft/2020-12/schema"
_NUM_MAP = {"type": "object", "additionalProperties": {"type": "number"}}
_POS_INT = {"type": "integer", "minimum": 1}

SUMMARY = {
    "$schema": _DRAFT,
    "title": "run summary (verify / tune)",
    "type": "object",
    "required": ["scenario", "kind", "ok"],
    "additionalProperties": True,
    "properties": {
        "scenario": {"type": "string"},
        "kind": {"enum": ["verify", "simulate", "tune"]},
        "ok": {"type": "boolean"},
        "seed": {"type": "integer"},
        "scheduler": {"type": "string"},
        "trials": {"type": "integer"},
        "world": {"type": "object"},
        "mismatches": {"type": "array"},
        "chosen_index": {"type": "integer"},
        "chosen_config": {"type": "object"},
        "outputs": {"type": "object", "additionalProperties": {"type": "string"}},
        "makespan_us": {"type": "number"},
        "ideal_makespan_us": {"type": "number"},
        "critical_path": {"type": "array", "items": {"type": "string"}},
        "threshold_gbps": {"type": "number"},
        "tails_us": _NUM_MAP,
        "slacks_us": _NUM_MAP,
        "total_tail_us": {"type": "number"},
        "stage_durations_us": _NUM_MAP,
    },
}

TUNE_REPORT = {
    "$schema": _DRAFT,
    "title": "tune report",
    "type": "object",
    "required": ["axes", "configs", "timings_us", "scores", "chosen_index", "chosen_config",
                 "per_rank_chosen", "invalid"],
    "additionalProperties": False,
    "properties": {
        "axes": {"type": "object", "additionalProperties": {"type": "array", "minItems": 1}},
        "configs": {"type": "array", "items": {"type": "object"}},
        # [config][rank][iteration] in us; null for a config that failed
        "timings_us": {"type": "array", "items": {"oneOf": [
            {"type": "null"},
            {"type": "array", "items": {"type": "array", "items": {"type": "number"}}}]}},
        "scores": {"type": "array", "items": {"oneOf": [{"type": "null"}, {"type": "number"}]}},
        "chosen_index": {"type": "integer", "minimum": 0},
        "chosen_config": {"type": "object"},
        "per_rank_chosen": {"type": "array", "items": {"type": "integer"}},
        "invalid": {"type": "object", "additionalProperties": {"type": "string"}},
    },
}

TRACE = {
    "$schema": _DRAFT,
    "title": "Chrome trace event list",
    "type": "array",
    "items": {
        "type": "object",
        "required": ["name", "ph", "ts", "dur", "pid", "tid"],
        "additionalProperties": False,
        "properties": {
            "name": {"type": "string"},
            "ph": {"const": "X"},
            "ts": {"type": "number", "minimum": 0},
            "dur": {"type": "number", "minimum": 0},
            "pid": {"type": "integer", "minimum": 0},
            "tid": {"type": "string"},
        },
    },
}

SCENARIO = {
    "$schema": _DRAFT,
    "title": "scenario configuration",
    "type": "object",
    "required": ["scenario"],
    "additionalProperties": False,
    "properties": {
        "scenario": {"type": "string"},
        "world": {"type": "object", "additionalProperties": False, "properties": {
            "world_size": _POS_INT, "n_nodes": _POS_INT, "local_world_size": _POS_INT,
            "heap_bytes": _POS_INT, "signal_count": _POS_INT,
            "timeout_s": {"type": "number", "exclusiveMinimum": 0}}},
        "params": {"oneOf": [{"type": "string"}, {"type": "object"}]},
        "problem": {"type": "object", "additionalProperties": False, "properties": {
            "m": _POS_INT, "n": _POS_INT, "k": _POS_INT, "dtype": {"type": "string"},
            "tile_m": {"type": "integer", "minimum": 0}, "tile_n": {"type": "integer", "minimum": 0},
            "bytes_per_rank": {"type": "integer", "minimum": 4}, "elems_per_rank": _POS_INT,
            "tokens_per_rank": {"type": "integer", "minimum": 0}, "experts": _POS_INT,
            "topk": _POS_INT, "hidden": _POS_INT, "dtype_bytes": _POS_INT, "m_per_rank": _POS_INT}},
        "trials": _POS_INT,
        "iterations": _POS_INT,
        "axes": {"type": "object", "additionalProperties": {"type": "array", "minItems": 1}},
        "measure": {"enum": ["model", "wall"]},
        "allocations": {"type": "object", "additionalProperties": {"type": "integer", "minimum": 0}},
        "sm_total": _POS_INT,
        "inject_corrupt": {"type": "boolean"},
    },
}

BY_NAME = {"summary": SUMMARY, "tune_report": TUNE_REPORT, "trace": TRACE, "scenario": SCENARIO}


def validate(doc, schema_name, what):
    """Raise ConfigurationError unless ``doc`` satisfies the named contract."""
    try:
        import jsonschema
    except ImportError as exc:  # the reference CLI depends on it too (pyproject.toml)
        raise ConfigurationError(f"jsonschema is required to validate {what}") from exc
    try:
        jsonschema.validate(doc, BY_NAME[schema_name])
    except jsonschema.ValidationError as exc:
        raise ConfigurationError(f"{what} violates the {schema_name} schema: {exc.message}")
