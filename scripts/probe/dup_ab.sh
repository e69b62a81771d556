nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
SHB_COPY_DUP=1 timeout 300 python -m pytest tests/test_gpu_pipelines.py tests/test_gpu_fuzz.py tests/test_gpu_baseline_configs.py tests/test_gpu_golden.py -q 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for v in 0 1; do
  SHB_COPY_DUP=$v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/raster_probe.py ag > /tmp/p.csv 2>&1
  echo "dup=$v: $(python scripts/ncu_table.py /tmp/p.csv | sed 's/.*bytes_read/read/')"
done
for v in 0 1 0 1 0 1; do
  echo "== SHB_COPY_DUP=$v"; SHB_COPY_DUP=$v AB_STEPS=600 python scripts/probe/long_blocks.py ag 2>&1 | grep "ag ours"
done
