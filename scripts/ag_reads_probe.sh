#!/bin/bash
# What drives the AG kernel's DRAM reads: stream-K tail, own-slot copy, raster.
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second"
for v in "SHB_SK=1" "SHB_SK=0" "SHB_OWN_COPY_CE=1" "SHB_SK=0 SHB_GROUP_M=32" "SHB_SK=0 SHB_GROUP_M=1" "SHB_SK=0 SHB_OWN_COPY_CE=1 SHB_GROUP_M=8"; do
  echo "== $v"
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  python scripts/ncu_table.py /tmp/p.csv
done
echo "== core C3 / C4"
ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py core > /tmp/p.csv 2>&1
python scripts/ncu_table.py /tmp/p.csv
