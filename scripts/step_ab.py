"""Interleaved A/B of the whole W=1 bench step (ours) against the unfused
torch.matmul pair, in blocks of STEPS back-to-back steps, ROUNDS rounds;
also each op alone against its cuBLAS call.  Medians per variant."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb

STEPS = int(os.environ.get("AB_STEPS", "200"))
ROUNDS = int(os.environ.get("AB_ROUNDS", "6"))
AG = dict(m=8192, n=3584, k=8192); RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags = sb.ProblemShape(dtype="bfloat16", **AG); rss = sb.ProblemShape(dtype="bfloat16", **RS)
agb = sb.make_ag_gemm_buffers(w, ags); rsb = sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
h0 = torch.randn(8192, 3584, device="cuda").bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
stream = pe.stream()

def ours():
    h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
    sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)

def unfused():
    torch.matmul(torch.matmul(x, wu), wd)

variants = {
    "step ours": ours, "step unfused": unfused,
    "ag ours": lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False),
    "ag cublas": lambda: torch.matmul(x, wu),
    "rs ours": lambda: sb.gemm_rs(pe, h0, wd, rss, sr, rsb, reset=False),
    "rs cublas": lambda: torch.matmul(h0, wd),
}

def run(fn):
    with torch.cuda.stream(stream):
        fn(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(STEPS):
            fn()
        e.record(stream); torch.cuda.synchronize()
    return s.elapsed_time(e) / STEPS

res = {k: [] for k in variants}
for r in range(ROUNDS):
    keys = list(variants)
    if r % 2:
        keys = keys[::-1]  # alternate who goes first
    for k in keys:
        res[k].append(run(variants[k]))
for k, ts in res.items():
    print(f"{k:14s} median {statistics.median(ts)*1e3:7.1f} us  min {min(ts)*1e3:7.1f}  max {max(ts)*1e3:7.1f}", flush=True)
