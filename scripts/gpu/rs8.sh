for i in 1 2 3; do
timeout 400 python -m pytest tests/test_gpu_bench_configs.py -x -q -p no:cacheprovider -k "w8 or w1" 2>&1 | tail -2
done
