M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for g in 8 16 32; do
  echo "== G=$g"
  SHB_GROUP_M=$g ncu --metrics $M --clock-control none --csv -k regex:"gemm_tp|nvjet" -s 2 -c 2 python scripts/probe/rs_big.py > /tmp/p.csv 2>&1
  python scripts/ncu_table.py /tmp/p.csv
done
