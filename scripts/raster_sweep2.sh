for g in 4 6 8 10 12 16; do
  echo "== G=$g"
  SHB_GROUP_M=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tp -s 2 -c 1 python scripts/profile_vs_cublas.py 2>&1 | grep -E "gpu__time|dram|per_second" | awk '{print $(NF-1), $NF}' | paste -sd' '
done
