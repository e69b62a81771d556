"""Interleaved A/B of the full W=1 bench step under env variants + unfused torch."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb
import torch
AG = dict(m=8192, n=3584, k=8192); RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags = sb.ProblemShape(dtype="bfloat16", **AG); rss = sb.ProblemShape(dtype="bfloat16", **RS)
agb = sb.make_ag_gemm_buffers(w, ags); rsb = sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
stream = pe.stream()
variants = sys.argv[1:] or ["-"]
keys = {kv.split("=")[0] for v in variants if v != "-" for kv in v.split(",")}
def setenv(v):
    for k in keys: os.environ.pop(k, None)
    if v != "-":
        for kv in v.split(","):
            k, val = kv.split("="); os.environ[k] = val
def ours():
    h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
    sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
def torch_step():
    torch.matmul(torch.matmul(x, wu), wd)
def run(fn, iters=30):
    with torch.cuda.stream(stream):
        fn(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(iters): fn()
        e.record(stream); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
res = {v: [] for v in variants + ["torch"]}
for _ in range(7):
    for v in variants:
        setenv(v); res[v].append(run(ours))
    res["torch"].append(run(torch_step))
fl = 2 * (8192 * 3584 * 8192) * 2
for v, ts in res.items():
    print(f"{v:30s} median {statistics.median(ts)*1e3:7.1f} us  {fl/statistics.median(ts)/1e9:7.1f} TF  min {min(ts)*1e3:7.1f} us")
