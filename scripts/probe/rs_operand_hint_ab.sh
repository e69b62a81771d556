# RS operand L2 hints (H = A re-read over 32 n-blocks, B over 32 m-blocks):
# DRAM per launch, then steady step
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for v in "X=0" "SHB_HINT_A_RS=last" "SHB_HINT_B_RS=last" "SHB_HINT_A_RS=last SHB_HINT_B_RS=first" "SHB_HINT_A_RS=first SHB_HINT_B_RS=last"; do
  env $v ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/profile_step.py 3 > /tmp/p.csv 2>&1
  echo "== $v"; python scripts/ncu_table.py /tmp/p.csv
done
for v in "X=0" "SHB_HINT_A_RS=last" "X=0" "SHB_HINT_A_RS=last" "X=0" "SHB_HINT_A_RS=last"; do
  echo "== $v"
  env $v AB_STEPS=600 python scripts/probe/long_blocks.py step 2>&1 | grep "ours  " | tail -1
done
