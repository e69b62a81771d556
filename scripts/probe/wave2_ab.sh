# NOTE: SHB_WAVE=2 (k-granular lockstep) was measured with this script and then
# removed from the kernel (profiles/README.md, r1_wave_kgran_ab.log); it needs
# the sources of that experiment to run again.
# k-granular wave lockstep (SHB_WAVE=2): exactness, DRAM per launch, steady
# state vs the default and vs the HEAD library (code-layout check)
nvidia-smi --query-gpu=pci.bus_id,serial --format=csv,noheader
timeout 300 python -m pytest tests/test_gpu_pipelines.py -q -k wave 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
for v in "SHB_WAVE=0" "SHB_WAVE=2 SHB_WAVE_D=16" "SHB_WAVE=2 SHB_WAVE_D=32" "SHB_WAVE=2 SHB_WAVE_D=64"; do
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "== $v"; python scripts/ncu_table.py /tmp/p.csv
done
for v in "SHB_WAVE=0" "SHB_WAVE=2"; do
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 2 -c 1 python scripts/probe/rs_big.py > /tmp/p.csv 2>&1
  echo "== C5 RS $v"; python scripts/ncu_table.py /tmp/p.csv
done
for r in 1 2 3; do
  echo "== head lib"; SHB_LIB=scripts/probe/lib_head.so AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  "
  echo "== new lib"; AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  "
  echo "== new lib wave2"; SHB_WAVE=2 AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  "
done
AB_ROUNDS=3 python scripts/ab_sweep.py "gemm_rs:16384,ag_gemm:16384" "-" "SHB_WAVE=2" "SHB_WAVE=2,SHB_WAVE_D=64" 2>&1 | tail -12
