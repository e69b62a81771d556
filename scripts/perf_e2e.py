import os, sys, time
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
x_host = x.cpu().pin_memory(); y_host = torch.empty(8192, 8192, dtype=torch.bfloat16).pin_memory()
x_dev = [torch.empty_like(x) for _ in range(2)]
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
def step(xin):
    h = sb.ag_gemm(pe, xin, wu, ags, sa, agb, reset=False)
    return sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
def loop(k, compute=True, copies=True):
    done_h2d = [torch.cuda.Event() for _ in range(2)]; done_use = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(k):
        slot = i % 2
        if i >= 2: h2d.wait_event(done_use[slot])
        if copies:
            with torch.cuda.stream(h2d): x_dev[slot].copy_(x_host, non_blocking=True)
        done_h2d[slot].record(h2d)
        stream.wait_event(done_h2d[slot])
        with torch.cuda.stream(stream):
            yd = step(x_dev[slot]) if compute else x_dev[slot]
        done_use[slot].record(stream)
        d2h.wait_stream(stream)
        if copies:
            with torch.cuda.stream(d2h):
                y_host.copy_(yd.view(torch.bfloat16) if compute else yd, non_blocking=True)
                yd.record_stream(d2h)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
with torch.cuda.stream(stream):
    step(x)
loop(3)
print("full      %.2f ms" % loop(20))
print("copies    %.2f ms" % loop(20, compute=False))
print("compute   %.2f ms" % loop(20, copies=False))
mode = os.environ.get("STEP", "")
if mode == "gemm":
    def step(xin):
        return sb.gemm(sb.gemm(xin, wu), wd)
    print("gemm-only full %.2f ms" % loop(20))
if mode == "ag":
    def step(xin):
        h = sb.ag_gemm(pe, xin, wu, ags, sa, agb, reset=False)
        return sb.gemm(h, wd)
    print("ag+gemm full %.2f ms" % loop(20))
if mode == "rs":
    def step(xin):
        return sb.gemm_rs(pe, sb.gemm(xin, wu), wd, rss, sr, rsb, reset=False)
    print("gemm+rs full %.2f ms" % loop(20))
