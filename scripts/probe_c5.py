"""One C5 sweep point (TP=1) for ncu: ``python scripts/probe_c5.py OP M [impls]``.

OP is ag_gemm (ProblemShape(M, 28672, 8192)) or gemm_rs (ProblemShape(M,
8192, 28672)); impls is a comma list of ``ours``, ``core`` (plain GEMM core)
and ``cublas``.  Two warm-up passes, then the profiled one (ncu -s/-c)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

op, M = sys.argv[1], int(sys.argv[2])
impls = sys.argv[3].split(",") if len(sys.argv) > 3 else ["ours", "cublas"]
reps = int(os.environ.get("PROBE_REPS", "3"))
FFN, HID = 28672, 8192
s = dict(m=M, n=FFN, k=HID) if op == "ag_gemm" else dict(m=M, n=HID, k=FFN)
heap = M * (s["k"] if op == "ag_gemm" else s["n"]) * 2 + (8 << 20)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=heap, timeout_s=60))
pe = w.pe(0)
shape = sb.ProblemShape(dtype="bfloat16", **s)
a = torch.randn(M, s["k"], device="cuda").bfloat16()
b = (torch.randn(s["k"], s["n"], device="cuda") * .02).bfloat16()
if op == "ag_gemm":
    bufs = sb.make_ag_gemm_buffers(w, shape)
    ours = lambda: sb.ag_gemm(pe, a, b, shape, sb.ag_order_switch(0, 1), bufs, reset=False)  # noqa: E731
else:
    bufs = sb.make_gemm_rs_buffers(w, shape)
    ours = lambda: sb.gemm_rs(pe, a, b, shape, sb.rs_inter_order(w.ranks[0], 1, 1), bufs,  # noqa: E731
                              reset=False)
stream = pe.stream()
with torch.cuda.stream(stream):
    for rep in range(reps):
        if "ours" in impls:
            ours()
        if "core" in impls:
            sb.gemm(a, b)
        if "cublas" in impls:
            torch.matmul(a, b)
        torch.cuda.synchronize()
w.close()
print("done", flush=True)
