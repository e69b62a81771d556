import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb
import torch
shapes = [(8192, 8192, 8192), (8192, 8192, 3584), (8192, 3584, 8192)]
for m, n, k in shapes:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(k, n, device="cuda").bfloat16()
    for _ in range(2):
        torch.matmul(a, b); sb.gemm(a, b)
    torch.cuda.synchronize()
    print("SHAPE", m, n, k, flush=True)
    torch.matmul(a, b); sb.gemm(a, b)
    torch.cuda.synchronize()
