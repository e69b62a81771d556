"""One launch each of: fused ag_gemm (C3), fused gemm_rs (C4), the plain GEMM
core on both shapes and cuBLAS on both shapes, after warm-up.  Meant to run
under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,...` (see
scripts/raster_probe.sh) to compare DRAM traffic per raster setting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

AG = dict(m=8192, n=3584, k=8192)
RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags = sb.ProblemShape(dtype="bfloat16", **AG)
rss = sb.ProblemShape(dtype="bfloat16", **RS)
agb = sb.make_ag_gemm_buffers(w, ags)
rsb = sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
h = torch.randn(8192, 3584, device="cuda").bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ag", "rs", "core", "cublas"]
stream = pe.stream()
with torch.cuda.stream(stream):
    for rep in range(3):  # 2 warm-up passes, then the profiled one (ncu -s/-c pick it)
        if "ag" in which:
            sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
        if "rs" in which:
            sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
        if "core" in which:
            sb.gemm(x, wu)
            sb.gemm(h, wd)
        if "cublas" in which:
            torch.matmul(x, wu)
            torch.matmul(h, wd)
        torch.cuda.synchronize()
print("done", flush=True)
