"""Symmetric heap and one-sided primitives on the GPU world, written like the
reference's tests/test_core.py and tests/test_primitives.py (bump allocation
and alignment, exhaustion, determinism, remote views and slab isolation,
barrier visibility, put/get/signal/wait semantics, token single use)."""

import contextlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_19442_b200 import (AllocationError, ArgumentError,  # noqa: E402
                                   CollectiveFault, RangeError, SymHandle, UsageError,
                                   WorldSpec,
                                   consume_token, init_world)
from paper_2504_19442_b200.primitives import SignalOp, WaitCond  # noqa: E402

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def make_world(world_size, heap_bytes=1 << 10, timeout_s=10.0):
    w = init_world(WorldSpec(world_size=world_size, heap_bytes=heap_bytes, timeout_s=timeout_s))
    try:
        yield w
    finally:
        w.close()


def b(t):
    return t.cpu().numpy().tobytes()


def test_world_geometry_single_node():
    with make_world(4) as w:
        assert [c.node_id for c in w.ranks] == [0, 0, 0, 0]
        assert [c.local_rank for c in w.ranks] == [0, 1, 2, 3]


def test_my_pe_n_pes():
    with make_world(4) as w:
        assert w.run(lambda pe: (pe.my_pe(), pe.n_pes())) == [(r, 4) for r in range(4)]
    with make_world(1) as w:
        assert w.run(lambda pe: (pe.my_pe(), pe.n_pes())) == [(0, 1)]


def test_alloc_bump_and_alignment():
    with make_world(2) as w:
        a = w.alloc_symmetric(64, align=16)
        bb = w.alloc_symmetric(64, align=16)
        assert (a.offset, bb.offset) == (0, 64)
        w.alloc_symmetric(1)
        d = w.alloc_symmetric(8, align=8)
        assert d.offset == 136  # 128 + 1 rounded up


def test_alloc_zero_and_exhaustion():
    with make_world(2, heap_bytes=256) as w:
        z = w.alloc_symmetric(0)
        assert z.length == 0 and z.offset == 0
        w.alloc_symmetric(200)
        with pytest.raises(AllocationError):
            w.alloc_symmetric(100)


def test_alloc_determinism_across_runs():
    def offsets():
        with make_world(3, heap_bytes=1 << 12) as w:
            return [w.alloc_symmetric(n, align=a).offset
                    for n, a in ((10, 8), (100, 64), (3, 1), (40, 32))]

    assert offsets() == offsets()


def test_remote_ptr_symmetry_and_bounds():
    with make_world(4) as w:
        h = w.alloc_symmetric(64)

        def body(pe):
            view = pe.remote_ptr(h, 2)
            if pe.rank == 0:  # a device store into rank 2's replica over the peer mapping
                view[:4] = torch.tensor([1, 2, 3, 4], dtype=torch.uint8, device=view.device)
            return view.numel()

        assert w.run(body) == [64] * 4
        assert w.read_from(2, h, 0, 4) == b"\x01\x02\x03\x04"
        # the same handle resolves to the same slab offset on every rank
        for r in range(4):
            base = w.heap_ptr(r, SymHandle(0, 64))
            assert w.heap_ptr(r, h) - base == h.offset
        with pytest.raises(CollectiveFault) as info:
            w.run(lambda pe: pe.remote_ptr(h, 4))
        assert isinstance(info.value.first, ArgumentError)


def test_no_cross_slab_leakage():
    with make_world(3, heap_bytes=256) as w:
        h = w.alloc_symmetric(64)
        before = [w.read_from(r, h, 0, 64) for r in range(3)]

        def body(pe):
            if pe.rank == 0:
                pe.remote_ptr(h, 1).fill_(0xAA)

        w.run(body)
        assert w.read_from(1, h, 0, 64) == b"\xaa" * 64
        assert w.read_from(0, h, 0, 64) == before[0]
        assert w.read_from(2, h, 0, 64) == before[2]


def test_barrier_makes_puts_visible():
    with make_world(4) as w:
        h = w.alloc_symmetric(8)

        def body(pe):
            if pe.rank == 0:
                for peer in range(4):
                    pe.putmem_nbi(h, (42).to_bytes(8, "little"), peer)
            pe.barrier_all()
            return pe.local_view(h).clone()

        assert [int.from_bytes(b(t), "little") for t in w.run(body)] == [42] * 4


def test_barrier_world_of_one_returns():
    with make_world(1) as w:
        w.run(lambda pe: pe.barrier_all())


def test_quiet_and_sync_all_complete_puts():
    with make_world(2) as w:
        h = w.alloc_symmetric(16)

        def body(pe):
            pe.quiet()  # nothing pending: no-op
            if pe.rank == 0:
                pe.putmem_nbi(h, b"y" * 16, 1)
                pe.quiet()
            pe.sync_all()
            return pe.local_view(h).clone()

        assert b(w.run(body)[1]) == b"y" * 16


def test_randomized_put_barrier_read_linearization(rng):
    # any put issued before a rank's barrier entry is readable everywhere after exit
    with make_world(4, heap_bytes=1 << 12) as w:
        h = w.alloc_symmetric(4 * 8)
        for _ in range(5):
            val = int(rng.integers(1, 1 << 30))

            def body(pe):
                pe.putmem_nbi(h, (val + pe.rank).to_bytes(8, "little"), (pe.rank + 1) % 4,
                              dst_off=pe.rank * 8)
                pe.barrier_all()
                got = torch.empty(4 * 8, dtype=torch.uint8, device=pe.torch_device)
                for src in range(4):
                    pe.getmem(got, h, (src + 1) % 4, nbytes=8, dst_off=src * 8,
                              src_off=src * 8)
                pe.barrier_all()
                return got

            for t in w.run(body):
                vals = np.frombuffer(b(t), dtype=np.int64)
                assert vals.tolist() == [val + r for r in range(4)]


def test_run_reports_worker_exception():
    with make_world(2) as w:
        def body(pe):
            if pe.rank == 1:
                raise ArgumentError("boom")

        with pytest.raises(CollectiveFault) as info:
            w.run(body)
        assert isinstance(info.value.failures[1], ArgumentError)


def test_put_to_self_and_empty_put():
    with make_world(2) as w:
        h = w.alloc_symmetric(4)

        def body(pe):
            pe.putmem(h, b"self", pe.rank)
            pe.putmem(h, b"", pe.rank)  # zero bytes: no-op success
            return pe.local_view(h).clone()

        assert [b(t) for t in w.run(body)] == [b"self"] * 2


def test_put_out_of_bounds():
    with make_world(2) as w:
        h = w.alloc_symmetric(4)
        with pytest.raises(CollectiveFault) as info:
            w.run(lambda pe: pe.putmem(h, b"12345", 0))
        assert isinstance(info.value.first, RangeError)


def test_getmem_blocking_and_self():
    with make_world(2) as w:
        h = w.alloc_symmetric(8)

        def body(pe):
            pe.putmem(h, bytes([pe.rank] * 8), pe.rank)
            pe.barrier_all()
            other = torch.empty(8, dtype=torch.uint8, device=pe.torch_device)
            mine = torch.empty(8, dtype=torch.uint8, device=pe.torch_device)
            pe.getmem(other, h, 1 - pe.rank)
            pe.getmem(mine, h, pe.rank)
            return other, mine

        res = [(b(o), b(m)) for o, m in w.run(body)]
        assert res[0] == (bytes([1] * 8), bytes([0] * 8))
        assert res[1] == (bytes([0] * 8), bytes([1] * 8))


def test_putmem_signal_pure_signal_and_add_fanin():
    with make_world(5) as w:
        h = w.alloc_symmetric(16)
        s = w.alloc_signals(2)

        def body(pe):
            if pe.rank == 0:
                pe.putmem_signal(h, b"", s.at(0), 9, 1)  # zero-byte payload: pure signal
            else:
                pe.putmem_signal(h, b"", s.at(1), 1, 0, op=SignalOp.ADD)
            pe.barrier_all()
            return pe.signal_read(s.at(0)), pe.signal_read(s.at(1))

        res = w.run(body)
        assert res[1][0] == 9
        assert res[0][1] == 4  # four concurrent ADD 1 senders


def test_signal_op_and_notify_equivalence():
    with make_world(2) as w:
        s = w.alloc_signals(2)

        def body(pe):
            if pe.rank == 0:
                pe.signal_op(1, s.at(0), SignalOp.SET, 5)
                pe.notify(1, s.at(1), 5)
            pe.barrier_all()
            return pe.signal_read(s.at(0)), pe.signal_read(s.at(1))

        assert w.run(body)[1] == (5, 5)
        with pytest.raises(CollectiveFault) as info:
            w.run(lambda pe: pe.signal_op(0, 10_000, SignalOp.SET, 1))
        assert isinstance(info.value.first, ArgumentError)


def test_wait_conditions():
    with make_world(2) as w:
        s = w.alloc_signals(1)

        def body(pe):
            if pe.rank == 0:
                pe.signal_op(1, s.at(0), SignalOp.SET, 3)
            else:
                # stream-ordered waits: GE on the GPU front end, NE / LT as a
                # bounded device spin; all satisfied once rank 0's SET lands
                pe.signal_wait_until(s.at(0), WaitCond.GE, 3)
                pe.signal_wait_until(s.at(0), WaitCond.NE, 0)
                pe.signal_wait_until(s.at(0), WaitCond.LT, 10)
                return pe.signal_read(s.at(0))

        assert w.run(body)[1] == 3


def test_token_single_use():
    with make_world(2) as w:
        h = w.alloc_symmetric(8)
        s = w.alloc_signals(1)

        def body(pe):
            if pe.rank == 0:
                pe.putmem_signal(h, b"tokenpay", s.at(0), 1, 1)
                return None
            tok = pe.wait(s.at(0), 1)
            payload = consume_token(tok, pe.local_view(h).clone())
            with pytest.raises(UsageError):
                consume_token(tok, payload)
            return payload

        assert b(w.run(body)[1]) == b"tokenpay"


def test_remote_ptr_self_is_local_view():
    with make_world(2) as w:
        h = w.alloc_symmetric(16)

        def body(pe):
            pe.remote_ptr(h, pe.rank)[:4] = torch.tensor(list(b"mine"), dtype=torch.uint8,
                                                         device=pe.torch_device)
            return pe.local_view(h)[:4].clone()

        assert [b(t) for t in w.run(body)] == [b"mine", b"mine"]
