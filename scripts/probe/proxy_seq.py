"""The bench's proxy sequence (TP=8, 2, 4) in one process: does an earlier
proxy disturb a later one's paced RS?  Prints per W the RS preset/paced and
the release times of one paced call."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tp_proxy

for W in [int(x) for x in (sys.argv[1:] or ["8", "2", "4"])]:
    px = tp_proxy.TpProxy(W, 8192, 28672 // W, 8192, 8192, 28672 // W)
    try:
        px._ensure_rs_estimate()
        pre = statistics.median(px.time_op("rs", "preset", 8))
        pac = px.time_op("rs", "paced", 8)
        print(json.dumps({"W": W, "done": [round(x, 1) for x in px.rs_done_us], "preset": round(pre, 1),
                          "paced": [round(x, 1) for x in pac], "arr": px.arrivals("rs"),
                          "lat_ns": px.release_lat_ns}), flush=True)
    finally:
        px.close()
