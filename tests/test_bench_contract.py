"""The bench.py contract the driver depends on, checked without a GPU: the
reference arm's JSON line, the C5 sweep shapes, the BASELINE roofline
arithmetic."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ, OPENBLAS_NUM_THREADS="2", OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         env=env, timeout=300, check=True)
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the unmodified reference package when it is installed under baseline/_ref
    # (the driver's offline install), else the numpy port of the same path
    installed = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "minishmem"))
    assert d["cpu_baseline"]["kind"] == ("reference" if installed else "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["steps"] == 1 and d["warmup"] == 0  # the driver's K / W, as given
    assert d["config"]["workload"].startswith("Llama-3-70B MLP TP pair")


def test_sweep_shapes_follow_c5():
    for tp in (1, 2, 4, 8):
        shapes = list(bench.sweep_shapes(tp))
        assert [(op, M) for op, M, _ in shapes] == [
            (op, M) for M in (1024, 4096, 16384) for op in ("ag_gemm", "gemm_rs")]
        for op, M, s in shapes:
            if op == "ag_gemm":
                assert s == dict(m=M, n=28672 // tp, k=8192)
            else:
                assert s == dict(m=M, n=8192, k=28672 // tp)
        assert bench.sweep_heap_bytes(tp) > 0


@pytest.mark.parametrize("tp", [1, 2, 8])
def test_tp_roofline_is_max_of_gemm_and_nvlink(tp):
    r = bench.tp_roofline(tp, 1000.0, ag_ms=1.0, rs_ms=1.0, step_ms=2.0)
    t_gemm = bench.flops(bench.AG) / 1e15 * 1e6
    assert r["ag"]["t_gemm_us"] == pytest.approx(t_gemm)
    t_nvl = (tp - 1) / tp * bench.AG["m"] * bench.AG["k"] * 2 / (bench.NVLINK_GBS * 1e9) * 1e6
    assert r["ag"]["t_nvlink_us"] == pytest.approx(t_nvl)
    assert r["ag"]["frac"] == pytest.approx(max(t_gemm, t_nvl) / 1000.0)
    assert r["ag"]["bound"] == ("tensor" if t_gemm >= t_nvl else "nvlink")
