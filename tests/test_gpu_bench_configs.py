"""Parity at the configurations bench.py times (BASELINE.json C3 / C4 / C5).

* W=1, the exact bench calls: ag_gemm ProblemShape(8192, 3584, 8192) and
  gemm_rs ProblemShape(8192, 8192, 3584) with the automatic tile / stream-K
  choice, random-normal bf16 operands against the fp32 oracle within the
  north-star tolerance (relative Frobenius error <= 1e-2); gathered slot 0 is
  the shard bit for bit; the RS output equals its own staging slot bit for
  bit (a world of one reduces one slot).
* W=8 on cuda:0 with the TP=8 per-rank chunking (1024-row chunks, 7
  flag-gated remote chunks, the weighted stream-K partition and sub-chunk
  flags at their defaults): same tolerance per rank; gathered bit-exact on
  every rank; the fused RS output is bit-for-bit the ascending-source fp32
  sum of the staging slots it read (the reference's reduction order,
  collectives.py:163-171); a one-hot payload checks the scatter layout
  bit-exactly against the oracle.
* C5 at TP=1: both ops for M in {1024, 4096, 16384}.
"""

import contextlib
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import minishmem_oracle as oracle  # noqa: E402
from paper_2504_19442_b200 import (ProblemShape, WorldSpec, ag_gemm,  # noqa: E402
                                   ag_order_switch, gemm_rs, init_world,
                                   make_ag_gemm_buffers, make_gemm_rs_buffers, rs_inter_order)

pytestmark = pytest.mark.gpu
BF16 = torch.bfloat16
TOL = 1e-2
AG = dict(m=8192, n=3584, k=8192)   # C3 per-rank ProblemShape
RS = dict(m=8192, n=8192, k=3584)   # C4 per-rank ProblemShape


def rel_frobenius(out, ref):
    return float(np.linalg.norm(out.astype(np.float64) - ref) / np.linalg.norm(ref))


def normal_bf16(g, shape, scale=1.0):
    """Seeded N(0, scale^2) rounded to bf16; returns (fp32 numpy for the
    oracle, the same values as a CPU bf16 tensor)."""
    x = torch.from_numpy((g.standard_normal(shape, dtype=np.float32) * scale)).to(BF16)
    return x.float().numpy(), x


@contextlib.contextmanager
def world(W, heap, timeout_s=60.0):
    w = init_world(WorldSpec(world_size=W, heap_bytes=heap, timeout_s=timeout_s,
                             devices=(0,) * W))
    try:
        yield w
    finally:
        w.close()


def test_c3_ag_gemm_w1_exact_bench_call():
    g = np.random.default_rng(0)
    a32, a = normal_bf16(g, (AG["m"], AG["k"]))
    b32, b = normal_bf16(g, (AG["k"], AG["n"]), 0.02)
    shape = ProblemShape(dtype="bfloat16", **AG)
    with world(1, AG["m"] * AG["k"] * 2 + (1 << 20)) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        out = w.run(lambda pe: ag_gemm(pe, a.cuda(), b.cuda(), shape, ag_order_switch(0, 1), bufs,
                                       reset=False))[0]
        gathered = w.read_tensor(0, bufs.gathered, BF16, (AG["m"], AG["k"]))
        assert torch.equal(gathered.cpu(), a)
    ref = oracle.ag_gemm_reference([a32], b32)
    assert rel_frobenius(out.float().cpu().numpy(), ref) <= TOL


def test_c4_gemm_rs_w1_exact_bench_call():
    g = np.random.default_rng(1)
    a32, a = normal_bf16(g, (RS["m"], RS["k"]))
    b32, b = normal_bf16(g, (RS["k"], RS["n"]), 0.02)
    shape = ProblemShape(dtype="bfloat16", **RS)
    with world(1, RS["m"] * RS["n"] * 2 + (1 << 20)) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        out = w.run(lambda pe: gemm_rs(pe, a.cuda(), b.cuda(), shape,
                                       rs_inter_order(pe.ctx, 1, 1), bufs, reset=False))[0]
        staging = w.read_tensor(0, bufs.staging, BF16, (RS["m"], RS["n"]))
        assert torch.equal(staging, out)
    ref = oracle.gemm_rs_reference([a32], [b32])[0]
    assert rel_frobenius(out.float().cpu().numpy(), ref) <= TOL


@pytest.mark.timeout(900)
def test_c3_ag_gemm_w8_tp8_chunking():
    W = 8
    rows = AG["m"] // W
    g = np.random.default_rng(2)
    shards = [normal_bf16(g, (rows, AG["k"])) for _ in range(W)]
    bs = [normal_bf16(g, (AG["k"], AG["n"]), 0.02) for _ in range(W)]
    shape = ProblemShape(dtype="bfloat16", **AG)
    heap = W * rows * AG["k"] * 2 + (1 << 20)
    with world(W, heap) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        staged = w.run(lambda pe: (shards[pe.rank][1].cuda(), bs[pe.rank][1].cuda()))
        outs = w.run(lambda pe: ag_gemm(pe, *staged[pe.rank], shape,
                                        ag_order_switch(pe.rank, W), bufs))
        outs = [o.float().cpu().numpy() for o in outs]
        gathered = [w.read_tensor(r, bufs.gathered, BF16, (AG["m"], AG["k"])).cpu()
                    for r in range(W)]
    expect = torch.cat([s[1] for s in shards])
    allA = np.vstack([s[0] for s in shards])
    for r in range(W):
        assert torch.equal(gathered[r], expect), r
        assert rel_frobenius(outs[r], allA @ bs[r][0]) <= TOL, r


@pytest.mark.timeout(900)
def test_c4_gemm_rs_w8_tp8_chunking():
    W = 8
    rows = RS["m"] // W
    g = np.random.default_rng(3)
    amats = [normal_bf16(g, (RS["m"], RS["k"])) for _ in range(W)]
    bs = [normal_bf16(g, (RS["k"], RS["n"]), 0.02) for _ in range(W)]
    shape = ProblemShape(dtype="bfloat16", **RS)
    heap = W * rows * RS["n"] * 2 + (1 << 20)
    with world(W, heap) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        staged = w.run(lambda pe: (amats[pe.rank][1].cuda(), bs[pe.rank][1].cuda()))
        outs = w.run(lambda pe: gemm_rs(pe, *staged[pe.rank], shape,
                                        rs_inter_order(pe.ctx, 1, W), bufs))
        outs = [o.cpu() for o in outs]
        staging = [w.read_tensor(r, bufs.staging, BF16, (W, rows, RS["n"])).cpu()
                   for r in range(W)]
    ref = oracle.gemm_rs_reference([a[0] for a in amats], [b[0] for b in bs])
    for r in range(W):
        assert rel_frobenius(outs[r].float().numpy(), ref[r]) <= TOL, r
        # the fused reduction: ascending-source fp32 sum of the bf16 slots
        acc = torch.zeros((rows, RS["n"]), dtype=torch.float32)
        for s in range(W):
            acc += staging[r][s].float()
        assert torch.equal(acc.to(BF16), outs[r]), r


@pytest.mark.timeout(900)
def test_c4_gemm_rs_w8_scatter_layout_one_hot():
    # one-hot A rows pick rows of B: every product exact, so the staging
    # layout is checked bit for bit against the oracle at the TP=8 shape
    W = 8
    rows = RS["m"] // W
    g = np.random.default_rng(4)
    amats, bs = [], []
    for _ in range(W):
        a = np.zeros((RS["m"], RS["k"]), dtype=np.float32)
        a[np.arange(RS["m"]), g.integers(0, RS["k"], RS["m"])] = 1.0
        amats.append(a)
        bs.append(g.integers(-8, 9, (RS["k"], RS["n"])).astype(np.float32))
    shape = ProblemShape(dtype="bfloat16", **RS)
    with world(W, W * rows * RS["n"] * 2 + (1 << 20)) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        staged = w.run(lambda pe: (torch.from_numpy(amats[pe.rank]).to(BF16).cuda(),
                                   torch.from_numpy(bs[pe.rank]).to(BF16).cuda()))
        outs = w.run(lambda pe: gemm_rs(pe, *staged[pe.rank], shape,
                                        rs_inter_order(pe.ctx, 1, W), bufs))
        outs = [o.float().cpu().numpy() for o in outs]
        for r in (0, 3, 7):
            staging = w.read_tensor(r, bufs.staging, BF16, (W, rows, RS["n"])).float().cpu().numpy()
            assert np.array_equal(staging, oracle.staging_layout(amats, bs, r)), r
    ref = oracle.gemm_rs_reference(amats, bs)
    for r in range(W):
        assert np.array_equal(outs[r], ref[r]), r


C5 = [("ag_gemm", M) for M in (1024, 4096, 16384)] + [("gemm_rs", M) for M in (1024, 4096, 16384)]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("op,M", C5)
def test_c5_tp1_points(op, M):
    FFN, HID = 28672, 8192
    s = dict(m=M, n=FFN, k=HID) if op == "ag_gemm" else dict(m=M, n=HID, k=FFN)
    g = np.random.default_rng(M + (op == "gemm_rs"))
    a32, a = normal_bf16(g, (s["m"], s["k"]))
    b32, b = normal_bf16(g, (s["k"], s["n"]), 0.02)
    shape = ProblemShape(dtype="bfloat16", **s)
    heap = s["m"] * (s["k"] if op == "ag_gemm" else s["n"]) * 2 + (1 << 20)
    with world(1, heap) as w:
        if op == "ag_gemm":
            bufs = make_ag_gemm_buffers(w, shape)
            out = w.run(lambda pe: ag_gemm(pe, a.cuda(), b.cuda(), shape, ag_order_switch(0, 1),
                                           bufs))[0]
        else:
            bufs = make_gemm_rs_buffers(w, shape)
            out = w.run(lambda pe: gemm_rs(pe, a.cuda(), b.cuda(), shape,
                                           rs_inter_order(pe.ctx, 1, 1), bufs))[0]
        out = out.float().cpu().numpy()
    t0 = time.time()
    ref = a32 @ b32
    assert rel_frobenius(out, ref) <= TOL, (op, M, time.time() - t0)
