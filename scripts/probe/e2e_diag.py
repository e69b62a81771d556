"""e2e loop (pinned H2D of X, compute, D2H of Y; double-buffered) with our fused
pair, with the unfused cuBLAS pair, and copies only -- which ones slow down?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb
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
x_host = x.cpu().pin_memory()
y_host = torch.empty((8192, 8192), dtype=torch.bfloat16).pin_memory()
x_dev = [torch.empty_like(x) for _ in range(2)]
y_fixed = torch.empty((8192, 8192), dtype=torch.bfloat16, device="cuda")
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()

def ours(xin):
    h = sb.ag_gemm(pe, xin, wu, ags, sa, agb, reset=False)
    return sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)

def unfused(xin):
    return torch.matmul(torch.matmul(xin, wu), wd)

def nocompute(xin):
    return y_fixed

def loop(step, k=40):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done_h2d = [torch.cuda.Event() for _ in range(2)]
    done_use = [torch.cuda.Event() for _ in range(2)]
    for i in range(k):
        slot = i % 2
        h2d.wait_event(e0)
        if i >= 2:
            h2d.wait_event(done_use[slot])
        with torch.cuda.stream(h2d):
            x_dev[slot].copy_(x_host, non_blocking=True)
        done_h2d[slot].record(h2d)
        stream.wait_event(done_h2d[slot])
        with torch.cuda.stream(stream):
            yd = step(x_dev[slot])
        done_use[slot].record(stream)
        d2h.wait_stream(stream)
        with torch.cuda.stream(d2h):
            y_host.copy_(yd, non_blocking=True)
            yd.record_stream(d2h)
    stream.wait_stream(d2h)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k

with torch.cuda.stream(stream):
    for _ in range(5): ours(x); unfused(x)
print(os.popen("nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader").read().strip())
for r in range(2):
    for name, fn in [("copies only", nocompute), ("ours", ours), ("unfused", unfused)]:
        print(f"round {r} {name:12s} {loop(fn):7.3f} ms/step", flush=True)
