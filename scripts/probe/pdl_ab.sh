# steady-state step time with / without programmatic dependent launch; kernel gaps via CUPTI
for v in 0 1 0 1; do
  echo "== SHB_PDL=$v"
  SHB_PDL=$v AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  "
done
