"""BASELINE.json configs C1 and C2 on the GPU path, against the oracle.

C1: AG+GEMM, world_size=2, M=N=K=1024 (fp32 in the reference): here bf16
    inputs (the GPU path computes in bf16/fp16), compared with the fp32
    oracle on the same bf16-rounded values within the north-star tolerance
    (relative Frobenius error <= 1e-2), gathered layout bit-exact.
C2: GEMM+RS, world_size=8, M=2048 K=4096 N=4096 (flag/scatter correctness):
    integer data, bit-exact output rows and staging layout on every rank.
"""

import contextlib

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


def bf16_round(x):
    return torch.from_numpy(x).to(BF16).float().numpy().astype(np.float64)


def test_c1_ag_gemm_w2_1024_cube():
    W, M, N, K = 2, 1024, 1024, 1024
    g = np.random.default_rng(0)
    shards = [bf16_round(g.standard_normal((M // W, K)).astype(np.float32)) for _ in range(W)]
    b = bf16_round(g.standard_normal((K, N)).astype(np.float32))
    ref = oracle.ag_gemm_reference(shards, b)
    shape = ProblemShape(m=M, n=N, k=K, dtype="bfloat16")
    with contextlib.closing(init_world(WorldSpec(world_size=W, heap_bytes=1 << 24,
                                                 timeout_s=20.0))) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        staged = w.run(lambda pe: (torch.from_numpy(shards[pe.rank]).to(BF16).to(pe.torch_device),
                                   torch.from_numpy(b).to(BF16).to(pe.torch_device)))
        res = w.run(lambda pe: ag_gemm(pe, *staged[pe.rank], shape,
                                       ag_order_switch(pe.rank, W), bufs))
        for r in range(W):
            out = res[r].float().cpu().numpy()
            assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= TOL
            gathered = w.read_tensor(r, bufs.gathered, BF16, (M, K)).float().cpu().numpy()
            assert np.array_equal(gathered, oracle.gathered_layout(shards))


def test_c2_gemm_rs_w8_2048_4096_4096():
    W, M, N, K = 8, 2048, 4096, 4096
    g = np.random.default_rng(1)
    # integer values held in float64 (BLAS oracle); |sums| < 256: exact in bf16
    amats = [g.integers(-1, 2, (M, K)).astype(np.float64) * (g.random((M, K)) < 0.02)
             for _ in range(W)]
    bs = [g.integers(-1, 2, (K, N)).astype(np.float64) for _ in range(W)]
    ref = oracle.gemm_rs_reference(amats, bs)
    assert max(np.abs(r).max() for r in ref) < 256
    shape = ProblemShape(m=M, n=N, k=K, dtype="bfloat16")
    with contextlib.closing(init_world(WorldSpec(world_size=W, heap_bytes=1 << 25,
                                                 timeout_s=30.0))) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        staged = w.run(lambda pe: (torch.from_numpy(amats[pe.rank]).to(BF16).to(pe.torch_device),
                                   torch.from_numpy(bs[pe.rank]).to(BF16).to(pe.torch_device)))
        res = w.run(lambda pe: gemm_rs(pe, *staged[pe.rank], shape,
                                       rs_inter_order(pe.ctx, 1, W), bufs))
        rows = M // W
        for r in range(W):
            assert np.array_equal(res[r].float().cpu().numpy(), ref[r])
            staging = w.read_tensor(r, bufs.staging, BF16, (W, rows, N)).float().cpu().numpy()
            assert np.array_equal(staging, oracle.staging_layout(amats, bs, r))
