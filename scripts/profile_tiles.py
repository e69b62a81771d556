"""ncu target: the C3 / C4 GEMM under several kernel configs (one launch each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb
from paper_2504_19442_b200.tuning import kernel_config
import torch
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
h = torch.randn(8192, 3584, device="cuda").bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
cfgs = [dict(bn=256, stream_k=1), dict(bn=256, stream_k=0), dict(bn=224, stream_k=0),
        dict(bn=224, stream_k=1)]
for _ in range(2):
    for c in cfgs:
        with kernel_config(**c):
            sb.gemm(x, wu); sb.gemm(h, wd)
torch.cuda.synchronize()
for c in cfgs:
    print("CFG", c, flush=True)
    with kernel_config(**c):
        sb.gemm(x, wu); sb.gemm(h, wd)
    torch.cuda.synchronize()
