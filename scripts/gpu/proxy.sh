set -x
timeout 600 python tp_proxy.py 30 > gpurun_out/proxy.json 2> gpurun_out/proxy.err; echo "proxy rc=$?"
tail -20 gpurun_out/proxy.err; cat gpurun_out/proxy.json
