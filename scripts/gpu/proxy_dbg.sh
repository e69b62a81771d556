PROXY_DEBUG=1 timeout 300 python - > gpurun_out/proxy_dbg.log 2>&1 <<'PY'
import statistics, tp_proxy, sys
px = tp_proxy.TpProxy(8, 8192, 3584, 8192, 8192, 3584, timeout_s=2.0)
print("preset", statistics.median(px.time_op("rs", "preset", 10)), flush=True)
print("free", px.time_op("rs", "free", 5), flush=True)
print("arr free", px.arrivals("rs", mode="free"), flush=True)
print("paced", px.time_op("rs", "paced", 5), flush=True)
print("ag preset", statistics.median(px.time_op("ag", "preset", 10)), flush=True)
print("ag arr free1", px.arrivals("ag", 1, mode="free"), flush=True)
print("ag arr free4", px.arrivals("ag", 4, mode="free"), flush=True)
PY
echo rc=$?; tail -40 gpurun_out/proxy_dbg.log | cut -c1-1500
