timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_r2.log
timeout 600 python tp_proxy.py 30 > gpurun_out/proxy_r2.json 2> gpurun_out/proxy_r2.err; echo "proxy rc=$?"; tail -2 gpurun_out/proxy_r2.err
timeout 420 ncu --set full --clock-control none --import-source on -k regex:gemm_tp_kernel -c 4 -o gpurun_out/r2_proxy_tp8_v2 python scripts/proxy_ncu.py both 8 > gpurun_out/proxy_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-proxy --no-cpu-baseline --no-unfused > gpurun_out/bench_ncu.log 2>&1; echo "ncu-bench rc=$?"
