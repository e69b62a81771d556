"""Data-before-signal litmus tests on the GPU (reference
pkg/tests/test_acceptance.py:277-355 stresses putmem+signal, wait/consume and
release/acquire over 10^4 iterations).

Everything is enqueued without host synchronisation and checked on the
device; a mismatch counter is read once at the end.

* primitives: rank 0 writes epoch e into a payload, puts it to rank 1 and
  signals e (copy engine + stream release); rank 1's stream waits for the
  flag, compares the payload it received against e and acknowledges; rank 0
  waits for the acknowledgement before reusing the buffers (10^4 epochs);
* fused ops: back-to-back ag_gemm + gemm_rs calls whose operands change
  every call (a per-call integer scale), so a stale chunk or a partial slot
  read before its flag shows up as a wrong product.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2504_19442_b200 as sb  # noqa: E402
from oracle import minishmem_oracle as oracle  # noqa: E402
from paper_2504_19442_b200.primitives import SignalOp, WaitCond  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_put_signal_wait_ack_10k_epochs():
    W, N, EPOCHS = 2, 4096, 10_000
    with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 20, timeout_s=60.0,
                                    devices=(0,) * W)) as w:
        recv = w.alloc_symmetric(N * 8)
        data_sig, ack_sig = w.alloc_signals(1).base, w.alloc_signals(1).base
        dev = torch.device("cuda", 0)
        src = torch.empty(N, dtype=torch.int64, device=dev)
        bad = torch.zeros((), dtype=torch.int64, device=dev)
        seen = torch.zeros((), dtype=torch.int64, device=dev)
        # load every torch kernel the bodies launch before any rank spins: a
        # lazily loaded module synchronises the context, i.e. waits for a
        # sibling's spinning wait kernel -- which waits for this very rank
        view1 = w.heap_view(1, recv, torch.int64, (N,))
        src.fill_(0)
        bad.add_((view1 != 0).sum())
        seen.add_(1)
        bad.zero_()
        seen.zero_()
        torch.cuda.synchronize(dev)

        def body(pe, lo, hi):
            if pe.rank == 0:
                for e in range(lo, hi):
                    if e > 1:  # rank 1 consumed e-1: the buffer may be reused
                        pe.signal_wait_until(ack_sig, WaitCond.GE, e - 1)
                    src.fill_(e)
                    pe.putmem_signal(recv, src, data_sig, e, 1)
            else:
                view = w.heap_view(1, recv, torch.int64, (N,))
                for e in range(lo, hi):
                    pe.signal_wait_until(data_sig, WaitCond.GE, e)
                    bad.add_((view != e).sum())
                    seen.add_(1)
                    pe.signal_op(0, ack_sig, SignalOp.SET, e)
            return None

        # rounds of 250 epochs: a rank thread must never block in a launch on a
        # full stream queue (it would hold the interpreter lock its peer needs
        # to issue the very release it waits for); flags stay monotone across
        # rounds, the joins only bound the queues
        for lo in range(1, EPOCHS + 1, 250):
            w.run(lambda pe, lo=lo: body(pe, lo, min(lo + 250, EPOCHS + 1)), timeout=120)
        assert int(seen) == EPOCHS
        assert int(bad) == 0


@pytest.mark.timeout(600)
def test_fused_ops_back_to_back_changing_operands():
    W, CALLS, ROUND = 2, 400, 50
    m, n, k = 512, 256, 256
    rows = m // W
    g = np.random.default_rng(21)
    xs = [g.integers(-1, 2, (rows, k)) for _ in range(W)]
    bs = [g.integers(-1, 2, (k, n)) for _ in range(W)]
    amats = [g.integers(-1, 2, (m, k)) for _ in range(W)]
    h_ref = [oracle.ag_gemm_reference(xs, bs[r]) for r in range(W)]
    y_ref = oracle.gemm_rs_reference(amats, bs)
    shape = sb.ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).to(dev)  # noqa: E731
    with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 24, timeout_s=60.0,
                                    devices=(0,) * W)) as w:
        agb, rsb = sb.make_ag_gemm_buffers(w, shape), sb.make_gemm_rs_buffers(w, shape)
        # per-call operand scales 1 / 2 (alternating, so a chunk left over from
        # the previous call is wrong by a factor of two); every product and
        # partial stays exact in bf16 (checked)
        S = (1, 2)
        scales = [c % 2 for c in range(CALLS)]
        xsc = {r: [t(xs[r] * s) for s in S] for r in range(W)}
        asc = {r: [t(amats[r] * s) for s in S] for r in range(W)}
        bt = {r: t(bs[r]) for r in range(W)}
        href = {r: [t(h_ref[r] * s) for s in S] for r in range(W)}
        yref = {r: [t(y_ref[r] * s) for s in S] for r in range(W)}
        assert max(np.abs(h).max() for h in h_ref) * 2 <= 256
        assert max(np.abs(y).max() for y in y_ref) * 2 <= 256
        assert max(np.abs(a @ b).max() for a, b in zip(amats, bs)) * 2 <= 256
        bad = {r: torch.zeros((), dtype=torch.int64, device=dev) for r in range(W)}
        h_out = {r: torch.empty((m, n), dtype=torch.bfloat16, device=dev) for r in range(W)}
        y_out = {r: torch.empty((rows, n), dtype=torch.bfloat16, device=dev) for r in range(W)}
        # load the comparison kernels before any rank spins (see above)
        bad[0].add_((h_out[0] != href[0][0]).sum() + (y_out[0] != yref[0][0]).sum())
        bad[0].zero_()
        torch.cuda.synchronize(dev)

        def body(pe, lo, hi):
            r = pe.rank
            for c in range(lo, hi):
                s = scales[c]
                sb.ag_gemm(pe, xsc[r][s], bt[r], shape, sb.ag_order_switch(r, W), agb,
                           reset=False, out=h_out[r])
                sb.gemm_rs(pe, asc[r][s], bt[r], shape, sb.rs_inter_order(pe.ctx, 1, W), rsb,
                           reset=False, out=y_out[r])
                bad[r].add_((h_out[r] != href[r][s]).sum() + (y_out[r] != yref[r][s]).sum())
            return None

        for lo in range(0, CALLS, ROUND):
            w.run(lambda pe, lo=lo: body(pe, lo, lo + ROUND), timeout=120)
        assert [int(bad[r]) for r in range(W)] == [0] * W
