SHB_SERPENTINE=1 timeout 300 python -m pytest tests/test_gpu_gemm_core.py tests/test_gpu_pipelines.py tests/test_gpu_fuzz.py -q 2>&1 | tail -1
for sp in 0 1 0 1 0 1 0 1; do
  echo "== SHB_SERPENTINE=$sp"
  SHB_SERPENTINE=$sp AB_STEPS=600 python scripts/probe/long_blocks.py ag 2>&1 | grep "ours  "
done
