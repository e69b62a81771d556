"""Paced vs preset on the TP proxy at a large per-rank M (default TP=2,
M=16384): release times of one paced call per op and the device timeline's
waits, to separate pacer effects from kernel waits."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tp_proxy

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
M = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
px = tp_proxy.TpProxy(W, M, 28672 // W, 8192, 8192, 28672 // W)
try:
    cal = px.calibrate()
    out = {"W": W, "M": M, "pacing": cal}
    for op in ("ag", "rs"):
        pre = statistics.median(px.time_op(op, "preset", 5))
        pac = px.time_op(op, "paced", 5)
        out[op] = {"preset": round(pre, 1), "paced": [round(x, 1) for x in pac],
                   "arrivals": px.arrivals(op), "trace": px.trace_waits(op)}
        if op == "rs":
            out[op]["done"] = [round(x, 1) for x in px.rs_done_us]
    print(json.dumps(out))
finally:
    px.close()
