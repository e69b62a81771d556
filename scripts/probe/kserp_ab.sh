# K-direction serpentine (SHB_KSERP=1): exactness, DRAM per launch, steady state
SHB_KSERP=1 timeout 300 python -m pytest tests/test_gpu_gemm_core.py tests/test_gpu_pipelines.py tests/test_gpu_fuzz.py tests/test_gpu_baseline_configs.py -q 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for v in 0 1; do
  SHB_KSERP=$v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "kserp=$v"; python scripts/ncu_table.py /tmp/p.csv
done
for v in 0 1 0 1 0 1; do
  echo "== SHB_KSERP=$v"
  SHB_KSERP=$v AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  "
done
