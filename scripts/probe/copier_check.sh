nvidia-smi --query-gpu=pci.bus_id,serial --format=csv,noheader
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for v in "SHB_PDL=1" "SHB_OWN_COPY_CE=1"; do
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "$v: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
AB_STEPS=600 python scripts/probe/long_blocks.py ag,step 2>&1 | grep steady
