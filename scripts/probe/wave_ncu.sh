M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second"
for wv in 0 1; do
  echo "== SHB_WAVE=$wv  RS M=16384"
  SHB_WAVE=$wv ncu --metrics $M --clock-control none --csv -k regex:"gemm_tp" -s 1 -c 1 python scripts/probe/rs_big.py > /tmp/p.csv 2>&1
  python scripts/ncu_table.py /tmp/p.csv
  echo "== SHB_WAVE=$wv  C3 AG / C4 RS"
  SHB_WAVE=$wv ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  python scripts/ncu_table.py /tmp/p.csv
done
