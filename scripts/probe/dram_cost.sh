# what DRAM read traffic costs in the power-capped steady state: AG C3 with
# raster group 8 (530 MB/launch) vs 32 (894 MB/launch)
for g in 8 32 8 32; do
  echo "== SHB_GROUP_M=$g"
  SHB_GROUP_M=$g AB_STEPS=600 python scripts/probe/long_blocks.py ag 2>&1 | grep "ag ours"
done
