"""compute-sanitizer target: the fused ops at W=1 (the bench's own world) and
W=2 on one GPU (the phased protocol the library picks under a
kernel-serialising tool), small shapes, checked against the oracle; and one
rank of a W=4 world with the full GPU (tp_proxy.py, preset flags): the
one-rank-per-GPU RS path (scattering GEMM with chunk-pair tiles, bulk-DMA
reduction kernel), checked bit for bit.

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402
from oracle import minishmem_oracle as oracle  # noqa: E402


def run(W, m, n, k, calls=2):
    rows = m // W
    g = np.random.default_rng(W)
    xs = [g.integers(-2, 3, (rows, k)) for _ in range(W)]
    bs = [g.integers(-1, 2, (k, n)) for _ in range(W)]
    amats = [g.integers(-1, 2, (m, k)) for _ in range(W)]
    ag = sb.ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 24, timeout_s=60,
                                    devices=(0,) * W)) as w:
        agb, rsb = sb.make_ag_gemm_buffers(w, ag), sb.make_gemm_rs_buffers(w, ag)
        t = lambda a: torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).cuda(0)  # noqa: E731
        ops = w.run(lambda pe: (t(xs[pe.rank]), t(bs[pe.rank]), t(amats[pe.rank])))
        for _ in range(calls):
            res = w.run(lambda pe: (
                sb.ag_gemm(pe, ops[pe.rank][0], ops[pe.rank][1], ag, sb.ag_order_switch(pe.rank, W), agb),
                sb.gemm_rs(pe, ops[pe.rank][2], ops[pe.rank][1], ag, sb.rs_inter_order(pe.ctx, 1, W), rsb)))
            ys = oracle.gemm_rs_reference(amats, bs)
            for r in range(W):
                assert np.array_equal(res[r][0].float().cpu().numpy(), oracle.ag_gemm_reference(xs, bs[r]))
                assert np.array_equal(res[r][1].float().cpu().numpy(), ys[r])
        print(f"W={W} {m}x{n}x{k}: {calls} calls exact (phased={w.phased})", flush=True)


def run_proxy():
    import tp_proxy

    px = tp_proxy.TpProxy(4, 512, 512, 512, 512, 512, timeout_s=60.0)
    try:
        for op in ("ag", "rs"):
            px.time_op(op, "preset", 1, warmup=0)
        torch.cuda.synchronize()
        stag = px.world.heap_view(0, px.rsb.staging, torch.bfloat16, (px.W, px.rows, px.rs.n))
        acc = torch.zeros(px.rows, px.rs.n, device=stag.device)
        for s in range(px.W):
            acc += stag[s].float()
        assert torch.equal(px.y.view(torch.int16), acc.to(torch.bfloat16).view(torch.int16))
        print("proxy W=4 rank 0 (separate GPUs path): RS bits exact", flush=True)
    finally:
        px.close()


run(1, 512, 512, 256)
run(2, 512, 256, 256)
run_proxy()
print("sanitize target ok")
