# AG C output stores evict-last vs normal (does RS read H from L2?): DRAM per launch, steady step
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for h in normal last; do
  SHB_HINT_STORE_AG=$h ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/profile_step.py 3 > /tmp/p.csv 2>&1
  echo "ag_store=$h"; python scripts/ncu_table.py /tmp/p.csv
done
for h in normal last normal last normal last; do
  echo "== SHB_HINT_STORE_AG=$h"
  SHB_HINT_STORE_AG=$h AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  "
done
