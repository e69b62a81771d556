"""cProfile of 300 small ag_gemm calls (host side)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2504_19442_b200 as sb
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=256 << 20, timeout_s=60))
pe = w.pe(0)
m, n, k = 1024, 3584, 8192
shape = sb.ProblemShape(dtype="bfloat16", m=m, n=n, k=k)
agb = sb.make_ag_gemm_buffers(w, shape); rsb = sb.make_gemm_rs_buffers(w, shape)
a = torch.randn(m, k, device="cuda").bfloat16(); b = (torch.randn(k, n, device="cuda") * .02).bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
with torch.cuda.stream(pe.stream()):
    for _ in range(10):
        sb.ag_gemm(pe, a, b, shape, sa, agb, reset=False); sb.gemm_rs(pe, a, b, shape, sr, rsb, reset=False)
    torch.cuda.synchronize()
    pr = cProfile.Profile(); pr.enable()
    for _ in range(300):
        sb.ag_gemm(pe, a, b, shape, sa, agb, reset=False)
        sb.gemm_rs(pe, a, b, shape, sr, rsb, reset=False)
    pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
