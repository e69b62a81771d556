# ncu metric pass of the TP=W proxy kernels under SHB_* knob settings.
# Usage: bash scripts/ncu_knob_ab.sh OP W "ENV=V ENV2=V" ["ENV=V" ...]
# Output: gpurun_out/ncuab_<op>_<cfg>.csv (read with scripts/ncu_csv.py)
op=$1; W=$2; shift 2
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_tp_kernel --launch-skip 1 -c 1 --csv \
    python scripts/proxy_ncu.py $op $W 2>/dev/null | grep -v "^==" > "gpurun_out/ncuab_${op}_$(echo $cfg | tr ' =' '_-').csv"
done
