M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__cycles_elapsed.avg.per_second,lts__cycles_elapsed.avg.per_second"
nvidia-smi --query-gpu=name,pci.bus_id,serial,clocks.max.sm,clocks.max.mem,power.limit,temperature.gpu --format=csv,noheader
for v in "SHB_KSERP=0 SHB_SERPENTINE=0 SHB_PDL=0 SHB_GROUP_M=8" "SHB_KSERP=0 SHB_SERPENTINE=0" "SHB_KSERP=0" "SHB_PDL=1"; do
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "$v"; python scripts/ncu_table.py /tmp/p.csv
done
ncu --metrics $M --clock-control none --csv -k regex:nvjet -c 2 python scripts/raster_probe.py cublas > /tmp/p.csv 2>&1; echo cublas; python scripts/ncu_table.py /tmp/p.csv
