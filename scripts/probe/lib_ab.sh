nvidia-smi --query-gpu=pci.bus_id,serial --format=csv,noheader
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for L in scripts/probe/lib_209f8c8.so scripts/probe/lib_285beae.so paper_2504_19442_b200/libshmem_b200.so; do
  SHB_LIB=$L ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "$L: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
