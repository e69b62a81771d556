nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for cfg in "scripts/probe/lib_base.so 0" "scripts/probe/lib_dup.so 0" "scripts/probe/lib_dup.so 1" "scripts/probe/lib_base.so 0"; do
  set -- $cfg
  SHB_LIB=$1 SHB_COPY_DUP=$2 ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "$1 dup=$2: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
