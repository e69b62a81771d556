# L2 promotion of the TMA loads: DRAM traffic per launch and steady-state time
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for pr in 3 2 0; do
  SHB_L2_PROMO=$pr ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "promo=$pr"; python scripts/ncu_table.py /tmp/p.csv
done
for pr in 3 2 3 2; do
  echo "== SHB_L2_PROMO=$pr"
  SHB_L2_PROMO=$pr AB_STEPS=600 python scripts/probe/long_blocks.py ag,rs 2>&1 | grep "ours  "
done
