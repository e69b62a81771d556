"""Cross-device paths, run only where two or more GPUs are visible (the
gpurun pool grants one; a multi-GPU GPUTEST exercises these first).

* a world without ``devices`` spreads rank r over GPU r % ndev;
* the fused ops across devices (peer TMA stores of the RS epilogue into
  another GPU's staging, copy-engine pushes into another GPU's gather buffer,
  stream-memop flag writes and red.release.sys counters on peer memory, all
  over NVLink) are bit-exact against the oracle (reference pipelines.py:97-233);
* putmem + signal into a peer GPU, back to back (reference primitives.py:126-222).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2504_19442_b200 as sb  # noqa: E402
from oracle import minishmem_oracle as oracle  # noqa: E402
from paper_2504_19442_b200.primitives import SignalOp, WaitCond  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs two or more GPUs")]


def test_default_devices_spread_ranks():
    n = torch.cuda.device_count()
    W = min(8, 2 * n)
    with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 20)) as w:
        assert w.devices == [r % n for r in range(W)]


@pytest.mark.parametrize("W", [2, 4, 8])
def test_fused_ops_across_devices_exact(W):
    n = torch.cuda.device_count()
    if W > n:
        pytest.skip(f"{W} ranks need {W} GPUs")
    m, nn, k = 256 * W, 384, 256
    rows = m // W
    g = np.random.default_rng(W)
    xs = [g.integers(-2, 3, (rows, k)) for _ in range(W)]
    bs = [g.integers(-1, 2, (k, nn)) for _ in range(W)]
    amats = [g.integers(-1, 2, (m, k)) for _ in range(W)]
    shape = sb.ProblemShape(m=m, n=nn, k=k, dtype="bfloat16")
    with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 26, timeout_s=30.0,
                                    devices=tuple(range(W)))) as w:
        agb, rsb = sb.make_ag_gemm_buffers(w, shape), sb.make_gemm_rs_buffers(w, shape)
        ops = w.run(lambda pe: tuple(
            torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).to(pe.torch_device)
            for a in (xs[pe.rank], bs[pe.rank], amats[pe.rank])))
        for _ in range(3):  # back to back: epochs across devices
            res = w.run(lambda pe: (
                sb.ag_gemm(pe, ops[pe.rank][0], ops[pe.rank][1], shape,
                           sb.ag_order_switch(pe.rank, W), agb),
                sb.gemm_rs(pe, ops[pe.rank][2], ops[pe.rank][1], shape,
                           sb.rs_inter_order(pe.ctx, 1, W), rsb)))
            ys = oracle.gemm_rs_reference(amats, bs)
            for r in range(W):
                assert np.array_equal(res[r][0].float().cpu().numpy(),
                                      oracle.ag_gemm_reference(xs, bs[r])), r
                assert np.array_equal(res[r][1].float().cpu().numpy(), ys[r]), r
        for r in range(W):
            got = w.read_tensor(r, agb.gathered, torch.bfloat16, (m, k)).float().cpu().numpy()
            assert np.array_equal(got, oracle.gathered_layout(xs)), r
        assert w.sweep_signals() == {}


def test_put_signal_into_peer_gpu_back_to_back():
    N, EPOCHS = 1 << 16, 200
    with sb.init_world(sb.WorldSpec(world_size=2, heap_bytes=1 << 22, timeout_s=30.0,
                                    devices=(0, 1))) as w:
        recv = w.alloc_symmetric(N * 4)
        data_sig, ack_sig = w.alloc_signals(1).base, w.alloc_signals(1).base
        src = torch.empty(N, dtype=torch.int32, device="cuda:0")
        bad = torch.zeros((), dtype=torch.int64, device="cuda:1")

        def body(pe):
            if pe.rank == 0:
                for e in range(1, EPOCHS + 1):
                    if e > 1:
                        pe.signal_wait_until(ack_sig, WaitCond.GE, e - 1)
                    src.fill_(e)
                    pe.putmem_signal(recv, src, data_sig, e, 1)
            else:
                view = w.heap_view(1, recv, torch.int32, (N,))
                for e in range(1, EPOCHS + 1):
                    pe.signal_wait_until(data_sig, WaitCond.GE, e)
                    bad.add_((view != e).sum())
                    pe.signal_op(0, ack_sig, SignalOp.SET, e)

        w.run(body)
        assert int(bad) == 0
