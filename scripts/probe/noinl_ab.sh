nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for L in scripts/probe/lib_base.so scripts/probe/lib_noinl.so scripts/probe/lib_base.so scripts/probe/lib_noinl.so; do
  SHB_LIB=$L ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "$L"; python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/'
done
