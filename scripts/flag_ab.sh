for M in 1024 8192; do
  PROXY_MODES=preset PROXY_M=$M timeout 300 python scripts/proxy_ab.py ag,rs 4 10 first= barall=SHB_FLAG_BARRIER_ALL:1 kernel=SHB_FLAG_KERNEL:1 > gpurun_out/flag_ab_$M.json 2> gpurun_out/flag_ab_$M.err
done
