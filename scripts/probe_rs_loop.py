"""Diagnostic: per-call time of gemm_rs C4 (W=1) in back-to-back loops, with a
fresh output per call vs a preallocated out=, and the AG C3 likewise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

AG = dict(m=8192, n=3584, k=8192)
RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags, rss = sb.ProblemShape(dtype="bfloat16", **AG), sb.ProblemShape(dtype="bfloat16", **RS)
agb, rsb = sb.make_ag_gemm_buffers(w, ags), sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
stream = pe.stream()
hbuf = torch.empty(8192, 3584, dtype=torch.bfloat16, device="cuda")
ybuf = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")


def loop(name, fn, k=20):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
    torch.cuda.synchronize()
    evs[0].record(stream)
    for i in range(k):
        fn()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    ts = [evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(k)]
    print(f"{name:28s} mean {sum(ts)/k:7.1f} us  first {ts[0]:7.1f}  min {min(ts):7.1f}  "
          f"max {max(ts):7.1f}", flush=True)


with torch.cuda.stream(stream):
    h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
    for rep in range(2):
        loop("ag alloc", lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False))
        loop("ag out=", lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False, out=hbuf))
        loop("rs alloc", lambda: sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False))
        loop("rs out=", lambda: sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False, out=ybuf))
        loop("rs alloc hbuf", lambda: sb.gemm_rs(pe, hbuf, wd, rss, sr, rsb, reset=False))
        loop("cublas rs", lambda: torch.matmul(h, wd))
w.close()
