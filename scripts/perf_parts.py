"""Time the parts of one bench step (W=1) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb
import torch

def bench(fn, iters=30, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3

AG = dict(m=8192, n=3584, k=8192); RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=30))
pe = w.pe(0)
ags = sb.ProblemShape(dtype="bfloat16", **AG); rss = sb.ProblemShape(dtype="bfloat16", **RS)
agb = sb.make_ag_gemm_buffers(w, ags); rsb = sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
h = sb.gemm(x, wu)
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
dst = torch.empty_like(x)
print("gemm AG shape      %7.1f us" % bench(lambda: sb.gemm(x, wu)))
print("gemm RS shape      %7.1f us" % bench(lambda: sb.gemm(h, wd)))
print("torch AG shape     %7.1f us" % bench(lambda: torch.matmul(x, wu)))
print("torch RS shape     %7.1f us" % bench(lambda: torch.matmul(h, wd)))
print("d2d copy 128MB     %7.1f us" % bench(lambda: dst.copy_(x)))
print("ag_gemm W=1        %7.1f us" % bench(lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)))
os.environ["SHB_OWN_COPY_CE"] = "1"
print("ag_gemm CE copy    %7.1f us" % bench(lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)))
del os.environ["SHB_OWN_COPY_CE"]
os.environ["SHB_RS_UNFUSED"] = "1"
print("gemm_rs unfused    %7.1f us" % bench(lambda: sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)))
del os.environ["SHB_RS_UNFUSED"]
print("gemm_rs W=1        %7.1f us" % bench(lambda: sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)))
def step():
    hh = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
    sb.gemm_rs(pe, hh, wd, rss, sr, rsb, reset=False)
print("step               %7.1f us" % bench(step))
import time
t0 = time.perf_counter()
for _ in range(200): sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
t1 = time.perf_counter()
print("host us per ag_gemm call (enqueue) %.1f" % ((t1 - t0) / 200 * 1e6))
torch.cuda.synchronize()
