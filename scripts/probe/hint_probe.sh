# AG C3 DRAM reads vs raster group and L2 eviction hints of the operand loads
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for cfg in "8 normal normal" "8 last first" "12 last first" "16 last first" "6 last first" "8 last normal" "8 normal first"; do
  set -- $cfg
  SHB_GROUP_M=$1 SHB_HINT_A=$2 SHB_HINT_B=$3 ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "G=$1 A=$2 B=$3: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
