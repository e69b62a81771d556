timeout 300 python -m pytest tests/test_gpu_gemm_core.py tests/test_gpu_pipelines.py tests/test_gpu_fuzz.py -q 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1; python scripts/ncu_table.py /tmp/p.csv
for g in 17 0 17 0 17 0; do
  echo "== SHB_GROUP_M=$g"
  if [ $g = 0 ]; then AB_STEPS=600 python scripts/probe/long_blocks.py rs 2>&1 | grep "rs ours"; else SHB_GROUP_M=$g AB_STEPS=600 python scripts/probe/long_blocks.py rs 2>&1 | grep "rs ours"; fi
done
