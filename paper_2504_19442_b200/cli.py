"""Parity / tuning command line on the GPU drop-in (§8 row f4; reference
pkg/src/minishmem/cli.py:59-560, verify and tune commands).

    python -m paper_2504_19442_b200.cli verify --config scenario.json [--out DIR]
    python -m paper_2504_19442_b200.cli tune --config scenario.json
    python -m paper_2504_19442_b200.cli list-scenarios

A scenario is the reference's JSON document (``{"scenario": "ag-gemm",
"world": {...}, "problem": {...}, "trials": 3}``).  ``verify`` runs the GPU
path against the dense numpy oracle with small-integer payloads (exact in
bf16) and reports mismatch coordinates; exit codes 0 ok / 1 mismatch or
tuning failure / 2 usage or configuration error, as cli.py:59-61.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

from . import schemas
from .errors import ConfigurationError, ShmemError

EXIT_OK = 0
EXIT_FAIL = 1
EXIT_USAGE = 2
_MISMATCH_LIMIT = 20

_WORLD_KEYS = {"world_size", "n_nodes", "local_world_size", "heap_bytes", "signal_count",
               "timeout_s"}
_PROBLEM_KEYS = {"m", "n", "k", "dtype", "tile_m", "tile_n", "bytes_per_rank", "elems_per_rank"}
_TOP_KEYS = {"scenario", "world", "problem", "trials", "iterations", "axes", "measure", "params",
             "allocations", "sm_total", "inject_corrupt"}

_DESCRIPTIONS = {
    "allgather-push": "push-mode AllGather on the GPU heap vs byte concatenation",
    "allgather-pull": "pull-mode AllGather (one barrier) vs byte concatenation",
    "reducescatter": "push-mode ReduceScatter (int64) vs the dense sum",
    "ag-gemm": "fused AllGather+GEMM (bf16 exact ints) vs vstack(shards) @ b",
    "gemm-rs": "fused GEMM+ReduceScatter (bf16 exact ints) vs row blocks of sum A_r @ B",
    "ag-gemm-tile": "tune the AG+GEMM kernel knobs (bn, stream_k, group_m, subchunks, ...) on device time",
}


def _validate_scenario(doc, what):
    if not isinstance(doc, dict) or "scenario" not in doc:
        raise ConfigurationError(f"{what}: a scenario object with a 'scenario' key is required")
    schemas.validate(doc, "scenario", what)
    extra = set(doc) - _TOP_KEYS
    if extra:
        raise ConfigurationError(f"{what}: unknown keys {sorted(extra)}")
    if set(doc.get("world", {})) - _WORLD_KEYS:
        raise ConfigurationError(f"{what}: unknown world keys {sorted(set(doc['world']) - _WORLD_KEYS)}")
    if set(doc.get("problem", {})) - _PROBLEM_KEYS:
        raise ConfigurationError(
            f"{what}: unknown problem keys {sorted(set(doc['problem']) - _PROBLEM_KEYS)}")
    for k in ("trials", "iterations"):
        if k in doc and (not isinstance(doc[k], int) or doc[k] < 1):
            raise ConfigurationError(f"{what}: {k} must be an integer >= 1")


def _world_from(doc, defaults, args):
    from .core import WorldSpec, init_world

    cfg = dict(defaults)
    cfg.update(doc.get("world", {}))
    if args.timeout_ms is not None:
        cfg["timeout_s"] = args.timeout_ms / 1000.0
    return init_world(WorldSpec(**cfg))


def _mismatches(trial, rank, got, want):
    got = np.asarray(got).reshape(-1)
    want = np.asarray(want).reshape(-1)
    if got.shape != want.shape:
        return [{"trial": trial, "rank": rank, "index": -1, "got": int(got.size),
                 "want": int(want.size)}]
    bad = np.nonzero(got != want)[0]
    return [{"trial": trial, "rank": rank, "index": int(i), "got": float(got[i]),
             "want": float(want[i])} for i in bad[:_MISMATCH_LIMIT]]


def _to_np(results):
    return [r.float().cpu().numpy() if hasattr(r, "cpu") else r for r in results]


def _verify_allgather(doc, args, pull):
    from .collectives import allgather_pull_intra, allgather_push_intra

    trials = doc.get("trials", 3)
    world = _world_from(doc, {"world_size": 8, "heap_bytes": 1 << 20}, args)
    n = doc.get("problem", {}).get("bytes_per_rank", 64)
    rng = np.random.default_rng(args.seed or 0)
    out = []
    with world:
        dst = world.alloc_symmetric(world.world_size * n)
        sigs = world.alloc_signals(world.world_size)
        for trial in range(trials):
            shards = [rng.integers(0, 256, size=n).astype(np.uint8) for _ in range(world.world_size)]

            def body(pe):
                fn = allgather_pull_intra if pull else allgather_push_intra
                fn(pe, dst, sigs, shards[pe.rank].tobytes())
                return pe.local_view(dst).clone()

            want = np.concatenate(shards)
            for rank, got in enumerate(world.run(body)):
                out += _mismatches(trial, rank, got.cpu().numpy(), want)
    return out


def _verify_reducescatter(doc, args):
    import torch

    from .collectives import reducescatter_push_intra
    from .primitives import SignalOp

    trials = doc.get("trials", 3)
    world = _world_from(doc, {"world_size": 8, "heap_bytes": 1 << 20}, args)
    w = world.world_size
    chunk = doc.get("problem", {}).get("elems_per_rank", 64)
    rng = np.random.default_rng(args.seed or 0)
    out = []
    with world:
        staging = world.alloc_symmetric(w * chunk * 8)
        psig, rsig = world.alloc_signals(w), world.alloc_signals(w)
        for trial in range(trials):
            vals = [rng.integers(-2 ** 31, 2 ** 31, w * chunk).astype(np.int64) for _ in range(w)]

            def body(pe):
                for c in range(w):
                    pe.signal_op(pe.rank, psig.at(c), SignalOp.SET, 1)
                res = torch.zeros(chunk, dtype=torch.int64, device=pe.torch_device)
                reducescatter_push_intra(pe, staging, psig, rsig,
                                         torch.from_numpy(vals[pe.rank]).to(pe.torch_device), res)
                return res

            oracle = sum(v.reshape(w, chunk) for v in vals)
            for rank, got in enumerate(world.run(body)):
                out += _mismatches(trial, rank, got.cpu().numpy(), oracle[rank])
    return out


def _shape(doc, defaults):
    from .pipelines import ProblemShape

    prob = dict(defaults)
    prob.update({k: v for k, v in doc.get("problem", {}).items() if k in ("m", "n", "k", "tile_m",
                                                                         "tile_n", "dtype")})
    prob.setdefault("dtype", "bfloat16")
    return ProblemShape(**prob)


def _dev(x, pe):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x).astype(np.float32)).to(torch.bfloat16).to(
        pe.torch_device)


def _verify_ag_gemm(doc, args):
    from .pipelines import ag_gemm, make_ag_gemm_buffers
    from .swizzle import ag_order_switch

    trials = doc.get("trials", 3)
    world = _world_from(doc, {"world_size": 4, "heap_bytes": 1 << 24}, args)
    shape = _shape(doc, {"m": 1024, "n": 256, "k": 256})
    w = world.world_size
    rows = shape.rows_per_rank(w)
    rng = np.random.default_rng(args.seed or 0)
    out = []
    with world:
        bufs = make_ag_gemm_buffers(world, shape)
        for trial in range(trials):
            shards = [rng.integers(-2, 3, size=(rows, shape.k)) for _ in range(w)]
            b = rng.integers(-1, 2, size=(shape.k, shape.n))

            def body(pe):
                x, bb = _dev(shards[pe.rank], pe), _dev(b, pe)
                return ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, w), bufs)

            oracle = np.vstack(shards) @ b
            for rank, got in enumerate(_to_np(world.run(body))):
                out += _mismatches(trial, rank, got, oracle)
    return out


def _verify_gemm_rs(doc, args):
    from .pipelines import gemm_rs, make_gemm_rs_buffers
    from .swizzle import rs_inter_order

    trials = doc.get("trials", 3)
    world = _world_from(doc, {"world_size": 4, "heap_bytes": 1 << 24}, args)
    shape = _shape(doc, {"m": 1024, "n": 256, "k": 128})
    w = world.world_size
    rows = shape.rows_per_rank(w)
    rng = np.random.default_rng(args.seed or 0)
    out = []
    with world:
        bufs = make_gemm_rs_buffers(world, shape)
        for trial in range(trials):
            mats = [rng.integers(-1, 2, size=(shape.m, shape.k)) for _ in range(w)]
            b = rng.integers(-1, 2, size=(shape.k, shape.n))

            def body(pe):
                a, bb = _dev(mats[pe.rank], pe), _dev(b, pe)
                return gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, w), bufs)

            oracle = sum(a @ b for a in mats)
            for rank, got in enumerate(_to_np(world.run(body))):
                out += _mismatches(trial, rank, got, oracle[rank * rows:(rank + 1) * rows])
    return out


VERIFY_SCENARIOS = {
    "allgather-push": lambda doc, args: _verify_allgather(doc, args, pull=False),
    "allgather-pull": lambda doc, args: _verify_allgather(doc, args, pull=True),
    "reducescatter": _verify_reducescatter,
    "ag-gemm": _verify_ag_gemm,
    "gemm-rs": _verify_gemm_rs,
}


def _tune_ag_gemm_tile(doc, args):
    from .pipelines import ag_gemm, make_ag_gemm_buffers
    from .swizzle import ag_order_switch
    from .tuning import ConfigSpace, tune

    shape = _shape(doc, {"m": 8192, "n": 3584, "k": 8192})
    axes = doc.get("axes", {"bn": [256, 128], "stream_k": [-1, 0]})
    world = _world_from(doc, {"world_size": 1, "heap_bytes": 1 << 30}, args)
    w = world.world_size
    rows = shape.rows_per_rank(w)
    rng = np.random.default_rng(args.seed or 0)
    shards = [rng.standard_normal((rows, shape.k)).astype(np.float32) for _ in range(w)]
    b = (rng.standard_normal((shape.k, shape.n)) * 0.02).astype(np.float32)
    with world:
        bufs = make_ag_gemm_buffers(world, shape)
        staged = world.run(lambda pe: (_dev(shards[pe.rank], pe), _dev(b, pe)))

        def target(pe, cfg):
            x, bb = staged[world.local_ranks.index(pe.rank)]
            ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, w), bufs)

        return tune(world, target, ConfigSpace(axes), iterations=doc.get("iterations", 3))


def _load(args):
    if not args.config:
        raise ConfigurationError("--config is required")
    text = args.config
    path = Path(text)
    if path.exists():
        text = path.read_text()
    elif not text.lstrip().startswith("{"):
        raise ConfigurationError(f"config file {path} not found")
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ConfigurationError(f"config is not valid JSON: {exc}")
    _validate_scenario(doc, str(args.config)[:60])
    return doc


def _emit(out_dir, filename, doc, schema_name):
    """Validate ``doc`` against its contract (reference cli.py:78-85), then
    write it (when an output directory was given)."""
    schemas.validate(doc, schema_name, filename)
    if out_dir is None:
        return None
    out_dir.mkdir(parents=True, exist_ok=True)
    path = out_dir / filename
    path.write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")
    return str(path)


def cmd_verify(args):
    doc = _load(args)
    name = doc["scenario"]
    runner = VERIFY_SCENARIOS.get(name)
    if runner is None:
        raise ConfigurationError(
            f"unknown verify scenario {name!r}; choices: {sorted(VERIFY_SCENARIOS)}")
    mismatches = runner(doc, args)
    summary = {"scenario": name, "kind": "verify", "ok": not mismatches, "seed": args.seed or 0,
               "scheduler": "free", "trials": doc.get("trials", 3), "mismatches": mismatches}
    path = _emit(Path(args.out) if args.out else None, f"{name}_summary.json", summary, "summary")
    print(json.dumps(summary if not path else {**summary, "written": path}, indent=2))
    return EXIT_OK if not mismatches else EXIT_FAIL


def cmd_tune(args):
    doc = _load(args)
    name = doc["scenario"]
    if name != "ag-gemm-tile":
        raise ConfigurationError(f"unknown tune scenario {name!r}; choices: ['ag-gemm-tile']")
    report = _tune_ag_gemm_tile(doc, args)
    out_dir = Path(args.out) if args.out else None
    path = _emit(out_dir, f"{name}_report.json", json.loads(report.to_json()), "tune_report")
    summary = {"scenario": name, "kind": "tune", "ok": True, "seed": args.seed or 0,
               "scheduler": "free", "chosen_index": report.chosen_index,
               "chosen_config": report.chosen_config, "scores_us": report.scores}
    if path:
        summary["outputs"] = {"report": path}
    _emit(out_dir, f"{name}_summary.json", summary, "summary")
    print(json.dumps(summary, indent=2))
    return EXIT_OK


def cmd_list(args):
    rows = [(n, "verify", _DESCRIPTIONS[n]) for n in sorted(VERIFY_SCENARIOS)]
    rows.append(("ag-gemm-tile", "tune", _DESCRIPTIONS["ag-gemm-tile"]))
    width = max(len(r[0]) for r in rows)
    for name, kind, desc in rows:
        print(f"{name:<{width}}  {kind:<8}  {desc}")
    return EXIT_OK


def build_parser():
    parser = argparse.ArgumentParser(prog="paper_2504_19442_b200",
                                     description="Verify or tune the GPU AG+GEMM / GEMM+RS path.")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, fn in (("verify", cmd_verify), ("tune", cmd_tune), ("list-scenarios", cmd_list)):
        p = sub.add_parser(name)
        p.set_defaults(fn=fn)
        if name != "list-scenarios":
            p.add_argument("--config", required=True, help="scenario JSON file or inline JSON")
            p.add_argument("--seed", type=int, default=None)
            p.add_argument("--out", default=None, help="output directory")
            p.add_argument("--timeout-ms", type=int, default=None)
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    from .tuning import TuningError

    try:
        return args.fn(args)
    except TuningError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_FAIL
    except (ConfigurationError, ShmemError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
