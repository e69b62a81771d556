# A/B of the bulk reduction's CTAs per SM x ring stages on the TP=8 proxy RS
# (event time via proxy_ab; the ncu loop needs --launch-skip 0 to catch the
# two rs_reduce launches of proxy_ncu.py)
for cfg in "2 3" "1 6" "1 4" "2 2" "1 3"; do set -- $cfg; SHB_RB_CTAS=$1 SHB_RB_STAGES=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed -k regex:rs_reduce -c 2 --clock-control none --csv --log-file gpurun_out/rb_c$1_s$2.csv python scripts/proxy_ncu.py rs 8 8192 > /dev/null 2>&1; done
PROXY_MODES=preset python scripts/proxy_ab.py rs 4 20 base= c1s6=SHB_RB_CTAS:1,SHB_RB_STAGES:6 c1s4=SHB_RB_CTAS:1,SHB_RB_STAGES:4 c2s2=SHB_RB_STAGES:2 > gpurun_out/rb_ab.json 2> gpurun_out/rb_ab.err
