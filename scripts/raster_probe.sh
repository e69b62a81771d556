#!/bin/bash
# DRAM traffic and time per launch of the fused ops / GEMM core / cuBLAS for a
# sweep of raster settings.  Output: gpurun_out/raster_probe_<tag>.csv
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second"
mkdir -p gpurun_out
ncu --metrics $M --clock-control none --csv -c 80 python scripts/raster_probe.py ag,rs,cublas \
  > gpurun_out/raster_probe_cublas.csv 2>&1
for g in ${RASTER_GROUPS:-1 2 3 4 8}; do
  for hb in ${HINTS_B:-normal last}; do
    SHB_GROUP_M=$g SHB_HINT_B=$hb ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 \
      python scripts/raster_probe.py ag,rs > gpurun_out/raster_probe_g${g}_${hb}.csv 2>&1
  done
done
