for i in 1 2 3 4 5 6; do
timeout 300 python -m pytest tests/test_gpu_dist.py -x -q -p no:cacheprovider 2>&1 | grep -E "AssertionError|rank [0-9]|passed|failed" | head -5
done
for i in 1 2; do
timeout 600 python -m pytest tests/test_gpu_baseline_configs.py tests/test_gpu_bench_configs.py -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -2
done
