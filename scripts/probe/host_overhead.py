"""Host enqueue time vs device time per call for a small TP=8-sized shape
(ag_gemm m=1024 n=3584 k=8192 at W=1: 60 GFLOP, ~45 us on the GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=256 << 20, timeout_s=60))
pe = w.pe(0)
for (m, n, k) in [(1024, 3584, 8192), (1024, 8192, 3584), (8192, 3584, 8192)]:
    shape = sb.ProblemShape(dtype="bfloat16", m=m, n=n, k=k)
    agb = sb.make_ag_gemm_buffers(w, shape)
    rsb = sb.make_gemm_rs_buffers(w, shape)
    a = torch.randn(m, k, device="cuda").bfloat16(); b = (torch.randn(k, n, device="cuda") * .02).bfloat16()
    sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
    for name, fn in [("ag_gemm", lambda: sb.ag_gemm(pe, a, b, shape, sa, agb, reset=False)),
                     ("gemm_rs", lambda: sb.gemm_rs(pe, a, b, shape, sr, rsb, reset=False)),
                     ("cublas", lambda: torch.matmul(a, b))]:
        with torch.cuda.stream(pe.stream()):
            for _ in range(10): fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter(); e0.record()
            for _ in range(200): fn()
            t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
        print(f"{m}x{n}x{k} {name:8s} host {(t1-t0)/200*1e6:6.1f} us/call  device {e0.elapsed_time(e1)/200*1e3:7.1f} us/call", flush=True)
