for lib in build_ab/lib_old.so paper_2504_19442_b200/libshmem_b200.so build_ab/lib_old.so paper_2504_19442_b200/libshmem_b200.so; do
  echo "== $lib"
  SHB_LIB=$lib ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tp -s 14 -c 7 python scripts/profile_variants.py 2>&1 | grep -E "gpu__time|sm__pipe|per_second" | awk '{print $NF}' | paste -sd' '
done
