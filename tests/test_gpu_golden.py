"""The GPU path on the reference's own golden inputs (tests/golden, produced by
running minishmem): bit-exact outputs and gathered / staging layouts for the
integer cases (every value is exact in bf16), rel-Frobenius <= 1e-2 for fp32."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_19442_b200 import (ProblemShape, WorldSpec, ag_gemm, ag_order_switch,  # noqa: E402
                                   gemm_rs, init_world, make_ag_gemm_buffers,
                                   make_gemm_rs_buffers, rs_inter_order)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BF16 = torch.bfloat16


def load(name):
    return dict(np.load(os.path.join(GOLD, f"{name}.npz")))


def t(x, pe):
    return torch.from_numpy(np.ascontiguousarray(x).astype(np.float32)).to(BF16).to(pe.torch_device)


def rel_fro(x, ref):
    return np.linalg.norm(x - ref) / np.linalg.norm(ref)


@pytest.mark.parametrize("name", ["ag_w2_int", "ag_w4_int", "ag_w8_int", "ag_w2_f32"])
def test_ag_gemm_on_reference_golden(name):
    g = load(name)
    w, rows, k = g["shards"].shape
    n = g["b"].shape[2]
    shape = ProblemShape(m=w * rows, n=n, k=k, dtype="bfloat16")
    exact = g["out"].dtype.kind == "i"
    with init_world(WorldSpec(world_size=w, heap_bytes=1 << 24, timeout_s=10)) as world:
        bufs = make_ag_gemm_buffers(world, shape)

        def body(pe):
            x, b = t(g["shards"][pe.rank], pe), t(g["b"][pe.rank], pe)
            return ag_gemm(pe, x, b, shape, ag_order_switch(pe.rank, w), bufs)

        outs = [o.float().cpu().numpy() for o in world.run(body)]
        gathered = [world.read_tensor(r, bufs.gathered, BF16, (w * rows, k)).float().cpu().numpy()
                    for r in range(w)]
    for r in range(w):
        if exact:
            assert np.array_equal(outs[r], g["out"][r])
            assert np.array_equal(gathered[r], g["gathered"][r])
        else:
            assert rel_fro(outs[r], g["out"][r]) < 1e-2
            assert np.array_equal(gathered[r], torch.from_numpy(g["gathered"][r]).to(BF16)
                                  .float().numpy())


@pytest.mark.parametrize("name", ["rs_w2_int", "rs_w4_int", "rs_w8_int", "rs_w4_f32"])
def test_gemm_rs_on_reference_golden(name):
    g = load(name)
    w, m, k = g["a"].shape
    n = g["b"].shape[2]
    rows = m // w
    shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    exact = g["out"].dtype.kind == "i"
    with init_world(WorldSpec(world_size=w, heap_bytes=1 << 24, timeout_s=10)) as world:
        bufs = make_gemm_rs_buffers(world, shape)

        def body(pe):
            a, b = t(g["a"][pe.rank], pe), t(g["b"][pe.rank], pe)
            return gemm_rs(pe, a, b, shape, rs_inter_order(pe.ctx, 1, w), bufs)

        outs = [o.float().cpu().numpy() for o in world.run(body)]
        staging = [world.read_tensor(r, bufs.staging, BF16, (w, rows, n)).float().cpu().numpy()
                   for r in range(w)]
    for r in range(w):
        if exact:
            assert np.array_equal(outs[r], g["out"][r])
            assert np.array_equal(staging[r], g["staging"][r])
        else:
            assert rel_fro(outs[r], g["out"][r]) < 1e-2
            assert rel_fro(staging[r], g["staging"][r]) < 1e-2
