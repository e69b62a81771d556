M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for g in 4 6 8 11 16; do
  SHB_GROUP_M=$g ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "G=$g $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
