for cfg in "" "SHB_FLAG_KERNEL=1"; do echo "== $cfg"; env $cfg timeout 200 python scripts/debug_rs.py 8 ag 30 device 2>&1 | tail -1; env $cfg timeout 200 python scripts/debug_rs.py 8 rs 30 device 2>&1 | tail -1;  done
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_pipelines.py -q 2>&1 | grep -E "^E |^FAILED|passed|failed" | cut -c1-300; done
