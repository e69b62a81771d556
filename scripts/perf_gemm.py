"""Quick GEMM-core perf probe: our tcgen05 kernel vs torch.matmul (cuBLAS)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb  # noqa: E402
from paper_2504_19442_b200 import _lib  # noqa: E402
import torch  # noqa: E402


def bench(fn, iters=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


shapes = [(8192, 3584, 8192), (8192, 8192, 3584), (8192, 8192, 8192), (4096, 4096, 4096),
          (1024, 3584, 8192)]
cfgs = [(256, 2)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]]
for m, n, k in shapes:
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(k, n, device="cuda").to(torch.bfloat16)
    fl = 2 * m * n * k
    t_ref = bench(lambda: torch.matmul(a, b))
    line = f"{m}x{n}x{k}: cublas {fl / t_ref / 1e9:7.1f} TF"
    for bn, cg in cfgs:
        _lib.check(_lib.load().sh_set_tile_config(bn, cg))
        for sk in ("0", "1"):
            os.environ["SHB_SK"] = sk
            t = bench(lambda: sb.gemm(a, b))
            line += f" | bn={bn} sk={sk} {fl / t / 1e9:7.1f}"
        del os.environ["SHB_SK"]
    c = sb.gemm(a, b)
    ref = (a.float() @ b.float())
    err = ((c.float() - ref).norm() / ref.norm()).item()
    print(line, f"relerr={err:.2e}", flush=True)
_lib.check(_lib.load().sh_set_tile_config(0, 0))
