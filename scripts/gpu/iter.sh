timeout 900 python -m pytest tests/test_gpu_litmus.py -q -p no:cacheprovider --durations=3 > gpurun_out/litmus.log 2>&1; echo rc=$?
grep -E "^E |passed|failed|call" gpurun_out/litmus.log | head -30
