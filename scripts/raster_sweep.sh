for g in 4 8 12 16 32; do
  echo "== group_m $g"
  SHB_GROUP_M=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_tp -s 4 -c 2 python scripts/profile_step.py 3 2>&1 | grep -E "dram__|gpu__time" | tr -s ' ' | paste -sd' '
done
