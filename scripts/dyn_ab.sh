for d in 0 1; do
  echo "== SHB_DYN=$d"
  SHB_DYN=$d ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_tp -s 6 -c 3 python scripts/profile_vs_cublas.py 2>&1 | grep -E "gpu__time|dram|per_second|sm__pipe" | awk '{print $(NF-1), $NF}' | paste -sd' '
done
