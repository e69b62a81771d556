# steady-state ag / rs calls with the static stride schedule vs the dynamic tile hand-out
for v in 0 1 0 1; do
  echo "== SHB_DYN=$v"
  SHB_DYN=$v AB_STEPS=600 python scripts/probe/long_blocks.py ag,rs 2>&1 | grep "ours  "
done
