"""A/B of the RS C5 point M=1024 (ProblemShape(1024, 8192, 28672), TP=1):
auto (256x512 wide tile) vs forced 256x256 (stream-K) vs torch.matmul,
interleaved blocks of back-to-back calls, CUDA events."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402
from paper_2504_19442_b200 import _lib  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "rs"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
m, n, k = (M, 8192, 28672) if op == "rs" else (M, 28672, 8192)
dev = torch.device("cuda", 0)
a = (torch.randn(m, k, device=dev) * 0.1).to(torch.bfloat16)
b = (torch.randn(k, n, device=dev) * 0.02).to(torch.bfloat16)
out_c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
shape = sb.ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
lib = _lib.load()
res = {"wide": [], "sk256": [], "cublas": []}
with sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=m * max(n, k) * 2 * 2 + (16 << 20),
                                timeout_s=30.0, devices=(0,))) as w:
    pe = w.pe(0)
    bufs = sb.make_gemm_rs_buffers(w, shape) if op == "rs" else sb.make_ag_gemm_buffers(w, shape)
    y = torch.empty((m, n), device=dev, dtype=torch.bfloat16)
    s = pe.stream()

    def ours():
        if op == "rs":
            sb.gemm_rs(pe, a, b, shape, sb.rs_inter_order(pe.ctx, 1, 1), bufs, reset=False, out=y)
        else:
            sb.ag_gemm(pe, a, b, shape, sb.ag_order_switch(0, 1), bufs, reset=False, out=y)

    import threading

    import pynvml

    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = {}

    def block(fn, n_=200, settle=20, name=None):
        for _ in range(settle):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        samples, stop = [], threading.Event()

        def sampler():
            while not stop.is_set():
                samples.append((pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(hnd) / 1e3))
                stop.wait(0.005)
        th = threading.Thread(target=sampler)
        e0.record(s)
        for _ in range(n_):
            fn()
        e1.record(s)
        th.start()
        s.synchronize()
        stop.set()
        th.join()
        if name and samples:
            clk.setdefault(name, []).append((statistics.median(x[0] for x in samples),
                                             statistics.median(x[1] for x in samples)))
        return e0.elapsed_time(e1) / n_ * 1e3

    with torch.cuda.stream(s):
        for rnd in range(4):
            for name in (("wide", "sk256", "cublas") if rnd % 2 == 0 else ("cublas", "sk256", "wide")):
                if name == "cublas":
                    res[name].append(block(lambda: torch.matmul(a, b, out=out_c), name=name))
                else:
                    _lib.check(lib.sh_set_tile_config(0 if name == "wide" else 256, 0 if name == "wide" else 2))
                    res[name].append(block(ours, name=name))
    _lib.check(lib.sh_set_tile_config(0, 0))
flops = 2.0 * m * n * k
print({kk: (round(statistics.median(v), 1), round(flops / statistics.median(v) / 1e6, 1),
            "MHz/W", [(round(c), round(p_)) for c, p_ in clk.get(kk, [])]) for kk, v in res.items()})
