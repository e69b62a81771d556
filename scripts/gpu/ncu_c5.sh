for M in 1024 16384; do
timeout 600 ncu --set full --clock-control none -k regex:"gemm_tp_kernel|nvjet|gemm|Kernel" --launch-skip 1 -c 3 -o gpurun_out/r2_c5_rs_M$M python scripts/ncu_c5.py rs $M > gpurun_out/ncu_c5_$M.log 2>&1; echo "M=$M rc=$?"; tail -2 gpurun_out/ncu_c5_$M.log
done
