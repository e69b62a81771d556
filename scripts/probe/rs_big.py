"""One RS call at M=16384 (C5, TP=1) + cuBLAS, for ncu DRAM/L2 counters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2504_19442_b200 as sb
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
FFN, HID = 28672, 8192
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=M * HID * 2 + (64 << 20), timeout_s=60))
pe = w.pe(0)
shape = sb.ProblemShape(dtype="bfloat16", m=M, n=HID, k=FFN)
bufs = sb.make_gemm_rs_buffers(w, shape)
a = torch.randn(M, FFN, device="cuda").bfloat16()
b = (torch.randn(FFN, HID, device="cuda") * .02).bfloat16()
sr = sb.rs_inter_order(w.ranks[0], 1, 1)
with torch.cuda.stream(pe.stream()):
    for _ in range(2):
        sb.gemm_rs(pe, a, b, shape, sr, bufs, reset=False)
        torch.matmul(a, b)
    torch.cuda.synchronize()
