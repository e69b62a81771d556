import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import tp_proxy
for trial in range(2):
    px = tp_proxy.TpProxy(4, 8192, 7168, 8192, 8192, 7168)
    try:
        px._ensure_rs_estimate()
        pre = statistics.median(px.time_op("rs", "preset", 8))
        pac = px.time_op("rs", "paced", 8)
        print(json.dumps({"trial": trial, "done": [round(x,1) for x in px.rs_done_us], "preset": round(pre,1), "paced": [round(x,1) for x in pac], "arr": px.arrivals("rs")}))
    finally:
        px.close()
