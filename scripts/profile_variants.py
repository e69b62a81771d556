"""One launch per variant for ncu metric comparison (same process, same data)."""
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
h = torch.randn(8192, 3584, device="cuda").bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
def env(**kv):
    for k in ["SHB_SK", "SHB_OWN_COPY_CE", "SHB_RS_UNFUSED"]: os.environ.pop(k, None)
    os.environ.update(kv)
runs = [
    ("ag_call_epi_copy_sk1_first", lambda: (env(SHB_SK="1"), sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False))),
    ("gemm_ag_sk1", lambda: (env(SHB_SK="1"), sb.gemm(x, wu))),
    ("gemm_ag_sk0", lambda: (env(SHB_SK="0"), sb.gemm(x, wu))),
    ("ag_call_epi_copy_sk1", lambda: (env(SHB_SK="1"), sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False))),
    ("ag_call_ce_copy_sk1", lambda: (env(SHB_SK="1", SHB_OWN_COPY_CE="1"), sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False))),
    ("gemm_rs_shape", lambda: (env(), sb.gemm(h, wd))),
    ("rs_call_fused", lambda: (env(), sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False))),
]
for _ in range(2):  # warm
    for name, fn in runs: fn()
torch.cuda.synchronize()
for name, fn in runs:
    print("RUN", name, flush=True)
    fn(); torch.cuda.synchronize()
