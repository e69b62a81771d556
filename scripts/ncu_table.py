"""Summarise an ncu --csv metrics dump: one row per launch, metrics as columns.

    python scripts/ncu_table.py file.csv [name-regex]
"""
import csv
import re
import sys


def rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    launches = {}
    for r in rd:
        key = int(r["ID"])
        d = launches.setdefault(key, {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    return [launches[k] for k in sorted(launches)]


def short(name):
    m = re.match(r"(?:void )?(?:[\w:]+::)?(\w+)(<[^(]*>)?", name)
    base = m.group(1) if m else name[:40]
    if "gemm_tp_kernel" in name:
        return "gemm_tp<" + name.split("<", 1)[1].split(">")[0] + ">"
    return base[:48]


def main():
    path = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    for d in rows(path):
        if pat and not pat.search(d["name"]):
            continue
        cols = []
        for k, vu in d.items():
            if k in ("name", "grid"):
                continue
            v, u = vu
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                cols.append(f"{k}={v}")
                continue
            if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                cols.append(f"{k.split('__')[1] if '__' in k else k}={fv * mult / 1e6:.1f}MB")
            elif u in ("nsecond", "usecond", "msecond"):
                mult = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}[u]
                cols.append(f"time={fv * mult:.1f}us")
            elif "hz" in u.lower():
                mult = {"hz": 1e-6, "khz": 1e-3, "mhz": 1, "ghz": 1e3}.get(u.lower().split("/")[0], 1)
                cols.append(f"clk={fv * mult:.0f}MHz")
            else:
                cols.append(f"{k.split('.')[0][-24:]}={fv:g}{u}")
        print(f"{short(d['name']):40s} grid={d['grid']:>12s} " + " ".join(cols))


if __name__ == "__main__":
    main()
