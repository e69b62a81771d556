"""Kernel timeline (CUPTI via torch.profiler) of back-to-back gemm_rs calls,
fused vs SHB_RS_UNFUSED=1: real overlap, no ncu serialisation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2504_19442_b200 as sb
RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=300 << 20, timeout_s=60))
pe = w.pe(0)
shape = sb.ProblemShape(dtype="bfloat16", **RS)
bufs = sb.make_gemm_rs_buffers(w, shape)
h = torch.randn(8192, 3584, device="cuda").bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
sr = sb.rs_inter_order(w.ranks[0], 1, 1)
stream = pe.stream()
for unf, ns in [("0", "0"), ("1", "0"), ("1", "1")]:
    os.environ["SHB_DIAG_NOSPIN"] = ns
    os.environ["SHB_RS_UNFUSED"] = unf
    with torch.cuda.stream(stream):
        for _ in range(3):
            sb.gemm_rs(pe, h, wd, shape, sr, bufs, reset=False)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(4):
                sb.gemm_rs(pe, h, wd, shape, sr, bufs, reset=False)
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    print(f"== unfused={unf} nospin={ns}")
    for e in evs:
        print(f"  {e.time_range.start - t0:9.1f} +{e.time_range.elapsed_us():8.1f} us  {e.name[:70]}")
