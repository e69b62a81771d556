import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_19442_b200 as sb
import torch
os.environ["SHB_SK"] = sys.argv[1] if len(sys.argv) > 1 else "1"
m, n, k = 2560, 2048, 512
shape = sb.ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=1 << 26))
bufs = sb.make_ag_gemm_buffers(w, shape)
x = torch.randint(-2, 3, (m, k), device="cuda").bfloat16()
b = torch.randint(-1, 2, (k, n), device="cuda").bfloat16()
pe = w.pe(0)
out = sb.ag_gemm(pe, x, b, shape, sb.ag_order_switch(0, 1), bufs, reset=False)
torch.cuda.synchronize()
g = w.read_tensor(0, bufs.gathered, torch.bfloat16, (m, k))
bad = (g != x)
print("bad elems", int(bad.sum()), "of", bad.numel())
if bad.any():
    rows = bad.any(1).nonzero().flatten().tolist(); cols = bad.any(0).nonzero().flatten().tolist()
    print("bad rows", rows[:5], "...", len(rows), " bad cols", cols[:5], "...", len(cols))
    rb = sorted({r // 128 for r in rows}); cb = sorted({c // 64 for c in cols})
    print("row blocks(128)", rb, "k blocks", cb)
print("out ok", bool((out.float() == x.float() @ b.float()).all()))
