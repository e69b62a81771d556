"""Device-timeline breakdown of the proxy kernels (preset flags): per CTA the
MMA warp's waits for a free accumulator (epilogue-bound) and for operand
stages (load-bound), epilogue windows by tile kind, CTA span.
Usage: python scripts/proxy_trace.py W [ag|rs]   (PROXY_M = per-job M, default 8192)"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tp_proxy  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mode = os.environ.get("PROXY_MODE", "preset")
ops = sys.argv[2:] or ["ag", "rs"]
M = int(os.environ.get("PROXY_M", "8192"))
if W == 1:
    px = tp_proxy.TpProxy(1, M, 3584, 8192, 8192, 3584)
else:
    px = tp_proxy.TpProxy(W, M, 28672 // W, 8192, 8192, 28672 // W)
out = {}
try:
    for op in ops:
        if mode == "paced0":
            px.rs_done_us = [0.0] * px.W  # every release right at the origin
        px.time_op(op, mode.rstrip("0"), 5, subchunks=1)
        px.world.start_trace(records_per_cta=1024, launches=2)
        px.time_op(op, mode.rstrip("0"), 1, warmup=0, subchunks=1)
        ev = px.world.stop_trace()
        kern = "ag_gemm" if op == "ag" else "gemm_rs"
        last = max(e["launch"] for e in ev if e["kernel"] == kern)
        red = [e for e in ev if e["kernel"] == "rs_reduce" and e["launch"] > last]
        ev = [e for e in ev if e["launch"] == last]
        t0 = min(e["t0_ns"] for e in ev if e["op"] == "cta")
        per = {}
        for e in ev:
            d = per.setdefault(e["cta"], {"acc_wait": 0, "stage_wait": 0, "items": 0, "epi": [],
                                          "epi_own": [], "end": 0})
            if e["op"] == "mma_item":
                d["acc_wait"] += e["t1_ns"] - e["t0_ns"]
                d["stage_wait"] += e["stage_wait_ns"] or 0
                d["items"] += 1
            elif e["op"] == "tile_epilogue":
                (d["epi_own"] if e["chunk"] == 0 and W > 1 else d["epi"]).append(e["t1_ns"] - e["t0_ns"])
                d["last_acc"] = max(d.get("last_acc", 0), e["t0_ns"] - t0)
            elif e["op"] == "own_reduce":
                d.setdefault("red", []).append(((e["t1_ns"] - e["t0_ns"]) / 1e3, e["drain_ns"] / 1e3))
            elif e["op"] == "cta":
                d["end"] = e["t1_ns"] - t0
                d["start"] = e["t0_ns"] - t0
            if e["op"] == "mma_item":
                d["first_mma"] = min(d.get("first_mma", 1 << 62), e["t0_ns"] - t0)
        lead = [d for d in per.values() if d["items"]]
        allepi = [x for d in per.values() for x in d["epi"]]
        allown = [x for d in per.values() for x in d["epi_own"]]
        out[op] = {
            "span_us": max(d["end"] for d in per.values()) / 1e3,
            "mma_acc_wait_us_mean": statistics.mean(d["acc_wait"] for d in lead) / 1e3,
            "mma_stage_wait_us_mean": statistics.mean(d["stage_wait"] for d in lead) / 1e3,
            "items_per_cluster": statistics.mean(d["items"] for d in lead),
            "epi_us_median": statistics.median(allepi) / 1e3 if allepi else None,
            "epi_us_p90": sorted(allepi)[int(0.9 * len(allepi))] / 1e3 if allepi else None,
            "epi_own_us_median": statistics.median(allown) / 1e3 if allown else None,
            "epi_own_us_max": max(allown) / 1e3 if allown else None,
            "own_reduce_us": sorted(x for d in per.values() for x in d.get("red", []))[::16],
            # tail: last accumulator ready (final MMA done) -> CTA end
            "tail_us": sorted(round((d["end"] - d.get("last_acc", d["end"])) / 1e3, 1)
                              for d in per.values() if "last_acc" in d)[::12],
            # ramp: CTA start spread, first MMA work item start
            "cta_start_us_max": max(d.get("start", 0) for d in per.values()) / 1e3,
            "first_mma_us": sorted(round(d["first_mma"] / 1e3, 1) for d in lead if "first_mma" in d)[::12],
            "end_us": sorted(round(d["end"] / 1e3, 1) for d in per.values())[::12],
            "last_acc_us_max": max(d.get("last_acc", 0) for d in per.values()) / 1e3,
            "peer_wait_us_max": max((e["t1_ns"] - e["t0_ns"]) / 1e3 for e in ev
                                    if e["op"] == "peer_wait") if any(e["op"] == "peer_wait" for e in ev) else 0,
            # separate RS reduction kernel: its CTAs' wait for the peers'
            # rows (kind 3) after the GEMM, and its span
            "reduce_wait_us_max": max(((e["t1_ns"] - e["t0_ns"]) / 1e3 for e in red
                                       if e["op"] == "peer_wait"), default=None),
            "reduce_span_us": ((max(e["t1_ns"] for e in red if e["op"] == "cta")
                                - min(e["t0_ns"] for e in red if e["op"] == "cta")) / 1e3
                               if any(e["op"] == "cta" for e in red) else None),
            "event_us": statistics.median(px.time_op(op, mode.rstrip("0"), 10, subchunks=1)),
        }
finally:
    px.close()
print(json.dumps(out))
