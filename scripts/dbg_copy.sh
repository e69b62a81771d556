for d in 0; do
  echo "== SHB_DBG=$d"
  SHB_DBG=$d ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k regex:gemm_tp -s 14 -c 7 python scripts/profile_variants.py 2>&1 | grep -E "gpu__time|sm__pipe|dram" | awk '{print $NF}' | paste -sd' '
done
