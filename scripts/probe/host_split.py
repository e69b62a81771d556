"""Host time per call: the Python wrapper vs the bare C-ABI call (tiny shape,
so the GPU is never the bottleneck)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2504_19442_b200 as sb
from paper_2504_19442_b200 import _lib
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=64 << 20, timeout_s=60))
pe = w.pe(0)
m = n = k = 512
shape = sb.ProblemShape(dtype="bfloat16", m=m, n=n, k=k)
agb = sb.make_ag_gemm_buffers(w, shape); rsb = sb.make_gemm_rs_buffers(w, shape)
a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(k, n, device="cuda").bfloat16()
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
sa = sb.ag_order_switch(0, 1)
lib = _lib.load()
order = _lib.int_array([0])
stream = pe.stream()
with torch.cuda.stream(stream):
    for _ in range(20): sb.ag_gemm(pe, a, b, shape, sa, agb, reset=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(1000): sb.ag_gemm(pe, a, b, shape, sa, agb, reset=False)
    t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"python ag_gemm: {(t1-t0)*1e3:.1f} us/call")
    ep = 10_000
    t0 = time.perf_counter()
    for i in range(1000):
        _lib.check(lib.sh_ag_gemm(w.handle, 0, a.data_ptr(), b.data_ptr(), c.data_ptr(),
                                  agb.gathered.offset, agb.ready.base, agb.done.base,
                                  m, n, k, 0, order, ep + i, stream.cuda_stream))
    t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"bare C call: {(t1-t0)*1e3:.1f} us/call")
