"""Interleaved A/B of the W=1 bench step (C3 ag_gemm then C4 gemm_rs) under
different tile configurations (sh_set_tile_config: bn, cta_group) against
the unfused torch.matmul pair, in blocks of AB_STEPS back-to-back steps
(AB_SETTLE untimed first), AB_ROUNDS rounds; SM clock median per block.
Usage: python scripts/tile_step_ab.py AGBN,AGCG/RSBN,RSCG ...  (0,0 = automatic)
       e.g. 0,0/0,0 0,0/512,2"""
import json
import os
import statistics
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402
from paper_2504_19442_b200 import _lib  # noqa: E402

STEPS = int(os.environ.get("AB_STEPS", "200"))
SETTLE = int(os.environ.get("AB_SETTLE", "100"))
ROUNDS = int(os.environ.get("AB_ROUNDS", "4"))
cfgs = [tuple(tuple(int(x) for x in half.split(",")) for half in a.split("/"))
        for a in sys.argv[1:]] or [((0, 0), (0, 0)), ((0, 0), (512, 2))]
cur = [((0, 0), (0, 0))]
lib = _lib.load()
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags = sb.ProblemShape(m=8192, n=3584, k=8192, dtype="bfloat16")
rss = sb.ProblemShape(m=8192, n=8192, k=3584, dtype="bfloat16")
agb, rsb = sb.make_ag_gemm_buffers(w, ags), sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
h = torch.empty(8192, 3584, device="cuda", dtype=torch.bfloat16)
y = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
stream = pe.stream()

import pynvml  # noqa: E402

pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)


def ours():
    (abn, acg), (rbn, rcg) = cur[0]
    lib.sh_set_tile_config(abn, acg)
    sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False, out=h)
    lib.sh_set_tile_config(rbn, rcg)
    sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False, out=y)


def unfused():
    torch.matmul(torch.matmul(x, wu), wd)


def block(fn, s):
    for _ in range(SETTLE):
        fn()
    clk, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
            stop.wait(0.01)
    th = threading.Thread(target=sampler)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    e0.record(s)
    for _ in range(STEPS):
        fn()
    e1.record(s)
    e1.synchronize()
    stop.set()
    th.join()
    return e0.elapsed_time(e1) * 1e3 / STEPS, statistics.median(clk) if clk else None


res = {}
for r in range(ROUNDS):
    for cfg in cfgs:
        cur[0] = cfg
        with torch.cuda.stream(stream):
            t, c = block(ours, stream)
        res.setdefault(f"ours ag={cfg[0]} rs={cfg[1]}", []).append((t, c))
    _lib.check(lib.sh_set_tile_config(0, 0))
    t, c = block(unfused, torch.cuda.current_stream())
    res.setdefault("unfused", []).append((t, c))
out = {k: {"us_per_step": round(statistics.median(t for t, _ in v), 1),
           "sm_mhz": statistics.median(c for _, c in v if c),
           "rounds": [round(t, 1) for t, _ in v]} for k, v in res.items()}
print(json.dumps(out, indent=1))
w.close()
