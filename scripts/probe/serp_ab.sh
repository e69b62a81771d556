# serpentine raster (SHB_SERPENTINE=1) vs default: exactness, DRAM per launch, steady state
SHB_SERPENTINE=1 timeout 300 python -m pytest tests/test_gpu_gemm_core.py tests/test_gpu_pipelines.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for sp in 0 1; do
  SHB_SERPENTINE=$sp ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "serp=$sp"; python scripts/ncu_table.py /tmp/p.csv
done
for sp in 0 1 0 1; do
  echo "== SHB_SERPENTINE=$sp"
  SHB_SERPENTINE=$sp AB_STEPS=600 python scripts/probe/long_blocks.py ag,rs 2>&1 | grep "ours  "
done
