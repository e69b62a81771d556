"""Long-block A/B (default 1000 steps per block, alternating, 3 rounds each):
does ours lose to the unfused pair only in long blocks?  Prints per-block
ms/step, and the per-100-step profile inside each block (CUDA events)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb
STEPS = int(os.environ.get("AB_STEPS", "1000"))
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
def ours():
    h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
    sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
def unfused():
    torch.matmul(torch.matmul(x, wu), wd)
def block(fn):
    with torch.cuda.stream(stream):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(STEPS // 100 + 1)]
        evs[0].record(stream)
        for i in range(STEPS):
            fn()
            if (i + 1) % 100 == 0:
                evs[(i + 1) // 100].record(stream)
        torch.cuda.synchronize()
    seg = [evs[i].elapsed_time(evs[i + 1]) / 100 * 1e3 for i in range(len(evs) - 1)]
    return sum(seg) / len(seg), seg
h0 = torch.randn(8192, 3584, device="cuda").bfloat16()
pairs = {
    "step": [("ours", ours), ("unfused", unfused)],
    "ag": [("ag ours", lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)),
           ("ag cublas", lambda: torch.matmul(x, wu))],
    "rs": [("rs ours", lambda: sb.gemm_rs(pe, h0, wd, rss, sr, rsb, reset=False)),
           ("rs cublas", lambda: torch.matmul(h0, wd))],
    "core4": [("core C4", lambda: sb.gemm(h0, wd)), ("cublas C4", lambda: torch.matmul(h0, wd))],
    "core3": [("core C3", lambda: sb.gemm(x, wu)), ("cublas C3", lambda: torch.matmul(x, wu))],
}
modes = (sys.argv[1] if len(sys.argv) > 1 else "step").split(",")
for _ in range(10):
    ours(); unfused()
torch.cuda.synchronize()
for mode in modes:
    pair = pairs[mode]
    steady = {n: [] for n, _ in pair}
    for r in range(3):
        for name, fn in (pair if r % 2 == 0 else pair[::-1]):
            avg, seg = block(fn)
            steady[name].append(sum(seg[1:]) / len(seg[1:]))
            print(f"round {r} {name:10s} {avg:7.1f} us  per-100: " + " ".join(f"{v:.0f}" for v in seg), flush=True)
    for name in steady:
        print(f"  {name:10s} steady (last 900 of each block) median {statistics.median(steady[name]):7.1f} us", flush=True)
