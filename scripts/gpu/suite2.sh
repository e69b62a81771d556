for i in 1 2; do
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$i.log 2>&1; echo "pytest#$i rc=$?"; tail -3 gpurun_out/pytest_gpu_$i.log; grep -E "^FAILED|^E  .*(Error|Fault|assert)" gpurun_out/pytest_gpu_$i.log | head -8
done
