mkdir -p gpurun_out
timeout 420 ncu --set full --clock-control none --import-source on -k regex:gemm_tp_kernel -c 4 -o gpurun_out/r2_proxy_tp8 python scripts/proxy_ncu.py both 8 > gpurun_out/proxy_ncu.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/proxy_ncu.log
timeout 300 ncu --set full --clock-control none -k regex:gemm_tp_kernel -c 2 -o gpurun_out/r2_proxy_tp1 python scripts/proxy_ncu.py rs 1 > gpurun_out/proxy_ncu1.log 2>&1; echo "ncu1 rc=$?"
tail -3 gpurun_out/proxy_ncu1.log
