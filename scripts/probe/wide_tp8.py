import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tp_proxy
from paper_2504_19442_b200 import _lib
lib = _lib.load()
px = tp_proxy.TpProxy(8, 8192, 3584, 8192, 8192, 3584)
res = {}
try:
    for r in range(4):
        for bn in (0, 512):
            _lib.check(lib.sh_set_tile_config(bn, 2 if bn else 0))
            for op in ("ag", "rs"):
                t = statistics.median(px.time_op(op, "preset", 10))
                res.setdefault(f"{op}/{bn}", []).append(round(t, 1))
finally:
    _lib.check(lib.sh_set_tile_config(0, 0))
    px.close()
print(json.dumps({k: (statistics.median(v), v) for k, v in res.items()}))
