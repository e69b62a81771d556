# die-aware m-split (SHB_DIE=1) vs default: exactness, DRAM per launch, steady state
SHB_DIE=1 SHB_TRACE=1 python -c "
import torch, paper_2504_19442_b200 as sb
a=torch.randn(4096,2048,device='cuda').bfloat16(); b=torch.randn(2048,4096,device='cuda').bfloat16()
c=sb.gemm(a,b); torch.cuda.synchronize(); ref=a.float()@b.float()
print('core rel err', ((c.float()-ref).norm()/ref.norm()).item())" 2>&1 | grep -E "die map|rel err"
SHB_DIE=1 timeout 300 python -m pytest tests/test_gpu_gemm_core.py tests/test_gpu_pipelines.py -q -x -k "not weighted and not wave" 2>&1 | tail -2
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for dd in 0 1; do
  SHB_DIE=$dd ncu --metrics $M --clock-control none --csv -k regex:gemm_tp -s 4 -c 2 python scripts/raster_probe.py ag,rs > /tmp/p.csv 2>&1
  echo "die=$dd"; python scripts/ncu_table.py /tmp/p.csv
done
for dd in 0 1 0 1; do
  echo "== SHB_DIE=$dd"
  SHB_DIE=$dd AB_STEPS=600 python scripts/probe/long_blocks.py ag,rs 2>&1 | grep "ours  "
done
