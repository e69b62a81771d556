timeout 600 python tp_proxy.py 30 > gpurun_out/proxy.json 2> gpurun_out/proxy.err; echo "proxy rc=$?"; tail -3 gpurun_out/proxy.err
for m in preset paced; do
PROXY_MODE=$m timeout 300 python scripts/proxy_trace.py 8 > gpurun_out/trace_$m.json 2> gpurun_out/trace_$m.err; echo "$m rc=$?"; cat gpurun_out/trace_$m.json; tail -2 gpurun_out/trace_$m.err
done
