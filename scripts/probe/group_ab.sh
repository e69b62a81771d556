# steady-state AG C3 call vs raster group (auto = 8)
for g in 8 1 4 8 1 4; do
  echo "== SHB_GROUP_M=$g"
  SHB_GROUP_M=$g AB_STEPS=600 python scripts/probe/long_blocks.py ag 2>&1 | grep "ag ours"
done
