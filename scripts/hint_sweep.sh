for a in normal last first; do for b in normal last first; do
  echo "== A=$a B=$b"
  SHB_HINT_A=$a SHB_HINT_B=$b ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tp -s 6 -c 3 python scripts/profile_vs_cublas.py 2>&1 | grep -E "gpu__time|dram|per_second" | awk '{print $(NF-1), $NF}' | paste -sd' '
done; done
