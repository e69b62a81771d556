"""Host vs device time per gemm_rs call, fused vs SHB_RS_UNFUSED=1 (W=1, C4)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
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
for unf in ["0", "1", "0", "1"]:
    os.environ["SHB_RS_UNFUSED"] = unf
    with torch.cuda.stream(stream):
        for _ in range(3):
            sb.gemm_rs(pe, h, wd, shape, sr, bufs, reset=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(20):
            sb.gemm_rs(pe, h, wd, shape, sr, bufs, reset=False)
        t1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    print(f"unfused={unf} host enqueue {(t1-t0)/20*1e6:.0f} us/call, device {e0.elapsed_time(e1)/20*1e3:.0f} us/call, wall {(t2-t0)/20*1e6:.0f}")
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(20):
            sb.gemm_rs(pe, h, wd, shape, sr, bufs, reset=True)
        e1.record(stream)
        torch.cuda.synchronize()
    print(f"unfused={unf} reset=True device {e0.elapsed_time(e1)/20*1e3:.0f} us/call")
