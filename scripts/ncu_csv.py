"""Print the metric table of `ncu --metrics ... --csv` logs (one row per
kernel launch).  Usage: python scripts/ncu_csv.py FILE..."""
import csv
import sys

SHORT = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "dram_rd_MB",
         "dram__bytes_write.sum": "dram_wr_MB",
         "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor%",
         "lts__t_sector_hit_rate.pct": "l2hit%", "sm__cycles_elapsed.avg.per_second": "GHz"}
SCALE = {"us": 1e-3, "dram_rd_MB": 1e-6, "dram_wr_MB": 1e-6, "GHz": 1e-9}

for fn in sys.argv[1:]:
    lines = [ln for ln in open(fn) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"][:48])
        name = SHORT.get(r["Metric Name"], r["Metric Name"])
        try:
            v = float(r["Metric Value"].replace(",", "")) * SCALE.get(name, 1.0)
        except ValueError:
            continue
        per.setdefault(key, {})[name] = round(v, 3)
    print("==", fn)
    for (i, k), d in per.items():
        print("  ", i, k, d)
