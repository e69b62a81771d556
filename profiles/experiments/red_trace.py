"""Timeline of the in-kernel column-streamed RS reduction on the TP=W proxy
(preset or paced): per unit the claim time, counter wait and duration
relative to the kernel start, and when the GEMM tiles ended.
Usage: python scripts/red_trace.py [preset|paced]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tp_proxy  # noqa: E402  (needs the patch in profiles/experiments)

mode = sys.argv[1] if len(sys.argv) > 1 else "preset"
px = tp_proxy.TpProxy(8, 8192, 28672 // 8, 8192, 8192, 28672 // 8)
try:
    px.time_op("rs", mode, 3)
    px.world.start_trace(records_per_cta=1024, launches=2)
    px.time_op("rs", mode, 1, warmup=0)
    ev = px.world.stop_trace()
    last = max(e["launch"] for e in ev)
    ev = [e for e in ev if e["launch"] == last]
    t0 = min(e["t0_ns"] for e in ev if e["op"] == "cta")
    units = sorted((e for e in ev if e["op"] == "reduce_unit"), key=lambda e: e["t0_ns"])
    epi = [e for e in ev if e["op"] == "tile_epilogue"]
    us = lambda x: round((x - t0) / 1e3, 1)  # noqa: E731
    out = {
        "units": len(units),
        "tiles_end_us": us(max(e["t1_ns"] for e in epi)),
        "cta_end_us": us(max(e["t1_ns"] for e in ev if e["op"] == "cta")),
        "unit_dur_us_median": statistics.median((e["t1_ns"] - e["t0_ns"] - e["ready_wait_ns"]) / 1e3
                                                for e in units) if units else None,
        "unit_done_us_deciles": [us(sorted(e["t1_ns"] for e in units)[int(q * (len(units) - 1))])
                                 for q in (0, .1, .2, .3, .4, .5, .6, .7, .8, .9, 1.0)] if units else None,
        "by_warp": {w: sum(1 for e in units if e["tile"] >> 16 == w) for w in range(7)},
        "first_units": [(e["tile"] & 0xFFFF, us(e["t0_ns"]), round(e["ready_wait_ns"] / 1e3, 1),
                         us(e["t1_ns"])) for e in units[:12]],
        "event_us": statistics.median(px.time_op("rs", mode, 5)),
    }
    print(json.dumps(out))
finally:
    px.close()
