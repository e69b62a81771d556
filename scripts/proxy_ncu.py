"""ncu target: the TP=W proxy's rank-0 kernels in preset mode (every flag set
before the launch, so a kernel-serialising profiler cannot deadlock them).
Usage: ncu ... python scripts/proxy_ncu.py [ag|rs|both] [W] [M]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tp_proxy  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
M = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
px = tp_proxy.TpProxy(W, M, 28672 // W, 8192, 8192, 28672 // W)
try:
    for op in ("ag", "rs"):
        if which in (op, "both"):
            px.time_op(op, "preset", 2, warmup=0, subchunks=1)
finally:
    px.close()
print("done")
