for m in preset paced paced0; do
PROXY_MODE=$m timeout 300 python scripts/proxy_trace.py 8 rs > gpurun_out/trace_$m.json 2> gpurun_out/trace_$m.err; echo "$m rc=$?"; cat gpurun_out/trace_$m.json; tail -2 gpurun_out/trace_$m.err
done
