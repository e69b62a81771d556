"""One W=1 bench step (ag_gemm + gemm_rs, Llama MLP per-rank shapes) for ncu:
    ncu --set full -k regex:gemm_tp_kernel -s 2 -c 2 python scripts/profile_step.py"""
import os, sys
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
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(steps):
    h = sb.ag_gemm(pe, x, wu, ags, sb.ag_order_switch(0, 1), agb, reset=False)
    y = sb.gemm_rs(pe, h, wd, rss, sb.rs_inter_order(w.ranks[0], 1, 1), rsb, reset=False)
torch.cuda.synchronize()
print("done")
