timeout 300 python scripts/ab_wide.py rs 1024
SHB_PDL=0 timeout 300 python scripts/ab_wide.py rs 1024
