M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
nvidia-smi --query-gpu=pci.bus_id,serial --format=csv,noheader
for v in "SHB_OWN_COPY_CE=1" "SHB_SK=0" "SHB_OWN_COPY_CE=1 SHB_SK=0" "SHB_HINT_A=normal"; do
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "$v: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 2 python scripts/raster_probe.py core > /tmp/p.csv 2>&1
echo "core:"; python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/'
