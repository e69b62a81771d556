# RS C4: DRAM traffic per launch and steady-state time vs the L2 policy of the epilogue stores
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for h in normal first; do
  SHB_HINT_STORE=$h ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py rs > /tmp/p.csv 2>&1
  echo "store=$h: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
for h in normal first normal first; do
  echo "== steady SHB_HINT_STORE=$h"
  SHB_HINT_STORE=$h AB_STEPS=600 python scripts/probe/long_blocks.py rs 2>&1 | grep steady
done
