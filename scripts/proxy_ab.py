"""Same-process A/B of library knobs on the TP=W proxy (tp_proxy.py).

Each config is a set of SHB_* environment overrides (read per launch by the
C ABI); configs are interleaved round by round and the per-config median of
the per-round medians is reported, preset and paced.

Usage: python scripts/proxy_ab.py OPS ROUNDS ITERS label=ENV:V,ENV:V ...
       e.g. python scripts/proxy_ab.py rs 3 20 base= help0=SHB_RED_HELP:0
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tp_proxy  # noqa: E402

ops = sys.argv[1].split(",")
rounds = int(sys.argv[2])
iters = int(sys.argv[3])
W = int(os.environ.get("PROXY_W", "8"))
modes = os.environ.get("PROXY_MODES", "preset,paced").split(",")
cfgs = []
for a in sys.argv[4:]:
    label, _, spec = a.partition("=")
    env = dict(kv.split(":", 1) for kv in spec.split(",") if kv)
    cfgs.append((label, env))

M = int(os.environ.get("PROXY_M", "8192"))
px = tp_proxy.TpProxy(W, M, 28672 // W, 8192, 8192, 28672 // W)
res = {}
try:
    base_env = {k: os.environ.get(k) for _, e in cfgs for k in e}
    for r in range(rounds):
        for label, env in cfgs:
            for k, v in base_env.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
            os.environ.update(env)
            for op in ops:
                for mode in modes:
                    t = px.time_op(op, mode, iters)
                    res.setdefault(f"{op}/{mode}/{label}", []).append(statistics.median(t))
    out = {k: {"median_us": round(statistics.median(v), 1), "rounds": [round(x, 1) for x in v]}
           for k, v in res.items()}
    print(json.dumps(out, indent=1))
finally:
    px.close()
