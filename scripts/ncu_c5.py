"""ncu target for the C5 TP=1 points: gemm_rs / ag_gemm at M in {1024, 16384}
(ProblemShape(M, 8192, 28672) / (M, 28672, 8192)) and torch.matmul of the same
GEMM for comparison.  Usage: python scripts/ncu_c5.py rs|ag M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

op, M = sys.argv[1], int(sys.argv[2])
m, n, k = (M, 8192, 28672) if op == "rs" else (M, 28672, 8192)
dev = torch.device("cuda", 0)
a = (torch.randn(m, k, device=dev) * 0.1).to(torch.bfloat16)
b = (torch.randn(k, n, device=dev) * 0.02).to(torch.bfloat16)
shape = sb.ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
with sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=m * max(n, k) * 2 + (16 << 20),
                                timeout_s=30.0, devices=(0,))) as w:
    bufs = sb.make_gemm_rs_buffers(w, shape) if op == "rs" else sb.make_ag_gemm_buffers(w, shape)
    for _ in range(2):
        if op == "rs":
            w.run(lambda pe: sb.gemm_rs(pe, a, b, shape, sb.rs_inter_order(pe.ctx, 1, 1), bufs))
        else:
            w.run(lambda pe: sb.ag_gemm(pe, a, b, shape, sb.ag_order_switch(0, 1), bufs))
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
print("done")
