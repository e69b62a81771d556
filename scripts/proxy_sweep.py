"""C5 on the TP proxy: both ops at TP = 2, 4, 8 for M in {1024, 4096, 16384}
(per-rank shapes AG (M, 28672/TP, 8192), RS (M, 8192, 28672/TP)), rank 0's
real kernels with the peers emulated (tp_proxy.py), against the roofline
(GEMM at the measured burst peak vs shard bytes at 900 GB/s) and the
modelled unfused sequence (measured cuBLAS + the collective's bytes at
770 GB/s).  One JSON line per point.
Usage: python scripts/proxy_sweep.py [iters] [W,W,...] [M,M,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tp_proxy  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
worlds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 8]
ms = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1024, 4096, 16384]
peak = 1700.9
mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(mp):
    peak = json.load(open(mp)).get("bf16_tflops", peak)
for W in worlds:
    for M in ms:
        try:
            r = tp_proxy.run(W=W, m=M, iters=iters, peak_tflops=peak, ab=False)
            out = {"W": W, "M": M, "parity": r["parity"]}
            for op in ("ag", "rs"):
                out[op] = {k: r[op][k] for k in ("preset_us", "paced_us", "tflops", "roofline_us",
                                                 "roofline_frac", "unfused_modelled_us",
                                                 "speedup_vs_unfused_modelled")}
        except Exception as e:  # noqa: BLE001
            out = {"W": W, "M": M, "error": f"{type(e).__name__}: {e}"[:300]}
        sys.stdout.write(json.dumps(out) + "\n")
        sys.stdout.flush()
