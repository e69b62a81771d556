"""Parity of the TP=8 per-rank kernels in the form a one-rank-per-GPU world
runs them (tp_proxy.py: rank 0 with the full persistent grid, the 7 peers'
rows and flags emulated), at the bench's C3 / C4 TP=8 shapes.

On separate GPUs the ReduceScatter defaults to the scattering GEMM followed
by the vectorised reduction kernel (ranks sharing a GPU -- the other W=8
tests -- keep the fused epilogue reduction), so this is the test of that
default at full size:

* RS output == the ascending-source fp32 sum of the 8 staging slots, bit for
  bit (reference collectives.py:163-171), preset and paced, and identical
  bits with the reduction fused into the epilogue (SHB_RS_UNFUSED=0);
* staging slot 0 (rank 0's own partial) within rel-Frobenius 1e-2 of the
  fp32 product (north-star tolerance);
* AG output within 1e-2 of the fp32 product, gathered layout bit-exact.
"""

import os
import sys

import pytest

torch = pytest.importorskip("torch")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module")
def proxy():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import tp_proxy

    px = tp_proxy.TpProxy(8, 8192, 28672 // 8, 8192, 8192, 28672 // 8, timeout_s=30.0)
    yield px
    px.close()


def _ascending_sum(px):
    stag = px.world.heap_view(0, px.rsb.staging, torch.bfloat16, (px.W, px.rows, px.rs.n))
    acc = torch.zeros(px.rows, px.rs.n, device=stag.device, dtype=torch.float32)
    for s in range(px.W):
        acc += stag[s].float()
    return stag, acc.to(torch.bfloat16)


def _rel(x, ref):
    return ((x.float() - ref).norm() / ref.norm()).item()


@pytest.mark.parametrize("mode", ["preset", "paced"])
@pytest.mark.parametrize("fused", ["default", "0"])
def test_tp8_rs_reduction_bits(proxy, monkeypatch, mode, fused):
    if fused != "default":
        monkeypatch.setenv("SHB_RS_UNFUSED", fused)
    proxy.y.fill_(float("nan"))
    proxy.time_op("rs", mode, 1, warmup=1)
    torch.cuda.synchronize()
    stag, ref = _ascending_sum(proxy)
    assert torch.equal(proxy.y.view(torch.int16), ref.view(torch.int16))
    part = proxy.a_rs[: proxy.rows].float() @ proxy.b_rs.float()
    assert _rel(stag[0], part) <= TOL
    # the peers' slots are untouched by rank 0's call
    assert torch.equal(stag[1:], proxy.peer_rows[1:])


def test_tp8_ag_product_and_layout(proxy):
    proxy.c.fill_(float("nan"))
    proxy.time_op("ag", "paced", 1, warmup=1)
    torch.cuda.synchronize()
    ref = proxy.x.reshape(-1, proxy.ag.k).float() @ proxy.b_ag.float()
    assert _rel(proxy.c, ref) <= TOL
    g = proxy.world.heap_view(0, proxy.agb.gathered, torch.bfloat16, (proxy.W * proxy.rows, proxy.ag.k))
    assert torch.equal(g, proxy.x.reshape(-1, proxy.ag.k))


@pytest.mark.parametrize("W,M", [(8, 1024), (4, 512), (2, 256)])
def test_small_chunk_pair_tiles_bits(W, M):
    # chunks of <= 128 rows: the scattering GEMM pairs two chunk positions per
    # CTA pair (SHB_RS_PAIR_CHUNKS); same bits as the ascending-source sum,
    # staging slot 0 within tolerance, for a world whose chunk count is even
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import tp_proxy

    px = tp_proxy.TpProxy(W, M, 28672 // W, 8192, 8192, 28672 // W, timeout_s=30.0)
    try:
        for mode in ("preset", "paced"):
            px.y.fill_(float("nan"))
            px.time_op("rs", mode, 1, warmup=1)
            torch.cuda.synchronize()
            stag, ref = _ascending_sum(px)
            assert torch.equal(px.y.view(torch.int16), ref.view(torch.int16))
            part = px.a_rs[: px.rows].float() @ px.b_rs.float()
            assert _rel(stag[0], part) <= TOL
            # the AG with the same pairing: product and gathered layout
            px.c.fill_(float("nan"))
            px.time_op("ag", mode, 1, warmup=1)
            torch.cuda.synchronize()
            ref_ag = px.x.reshape(-1, px.ag.k).float() @ px.b_ag.float()
            assert _rel(px.c, ref_ag) <= TOL
            g = px.world.heap_view(0, px.agb.gathered, torch.bfloat16, (px.W * px.rows, px.ag.k))
            assert torch.equal(g, px.x.reshape(-1, px.ag.k))
    finally:
        px.close()
