"""Host side of the timeline emitter: events -> Chrome trace / exposed-comm
summary (the device side is covered by test_gpu_timeline.py)."""

import json

from paper_2504_19442_b200 import schemas
from paper_2504_19442_b200.timeline import exposed_comm, to_chrome_trace


def ev(op, cta, t0, t1, rank=0, launch=0, kernel="ag_gemm", chunk=None):
    return {"rank": rank, "launch": launch, "kernel": kernel, "op": op, "cta": cta,
            "chunk": chunk, "item_kind": None, "tile": 0, "t0_ns": t0, "t1_ns": t1}


def test_chrome_trace_shape_matches_reference_timeline():
    events = [ev("cta", 0, 1000, 9000), ev("chunk_wait", 0, 2000, 2500, chunk=3),
              ev("tile_epilogue", 1, 4000, 4400, chunk=0)]
    evs = to_chrome_trace(events)
    json.dumps(evs)
    schemas.validate(evs, "trace", "trace")  # the reference's trace contract
    assert {e["ph"] for e in evs} == {"X"}
    assert {"name", "ph", "ts", "dur", "pid", "tid"} == set(evs[0])
    wait = next(e for e in evs if "chunk_wait" in e["name"])
    assert wait["ts"] == 1.0 and wait["dur"] == 0.5 and wait["tid"] == "cta0" and "[c3]" in wait["name"]
    assert to_chrome_trace([]) == []


def test_exposed_comm_per_launch():
    events = [ev("cta", 0, 0, 10_000), ev("cta", 1, 500, 12_000),
              ev("chunk_wait", 0, 100, 1100, chunk=1), ev("chunk_wait", 0, 2000, 2500, chunk=2),
              ev("chunk_wait", 1, 600, 700, chunk=1),
              ev("cta", 0, 20_000, 30_000, launch=1, kernel="gemm_rs"),
              ev("peer_wait", 0, 25_000, 27_000, launch=1, kernel="gemm_rs", chunk=0)]
    s = exposed_comm(events)
    ag = next(x for x in s if x["kernel"] == "ag_gemm")
    rs = next(x for x in s if x["kernel"] == "gemm_rs")
    assert ag["span_us"] == 12.0 and ag["wait_max_us"] == 1.5 and ag["wait_mean_us"] == 0.8
    assert rs["span_us"] == 10.0 and rs["wait_max_us"] == 2.0
