"""Flag-protocol properties of the fused ops on the GPU:

* the phased protocol (what a kernel-serialising tool gets: ncu,
  compute-sanitizer) computes the same bits as the fused one;
* sub-chunk ready flags: any range count gives the same bits, and the flag
  words end at epoch * ranges;
* gemm_rs with the own chunk first in the schedule and many tiles per chunk
  (more tiles than CTA pairs) completes -- the library runs it last;
* a wait nobody satisfies is a SynchronizationFault within the world's
  timeout, and a stream wait that can never pass is reported by the host
  deadline instead of hanging;
* the device really acquires every remote chunk (timeline records), the
  host-side "wait" counter is not the only evidence.
"""

import contextlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import minishmem_oracle as oracle  # noqa: E402
from paper_2504_19442_b200 import (  # noqa: E402
    CollectiveFault,
    ProblemShape,
    ShmemError,
    SynchronizationFault,
    TileSchedule,
    TileStep,
    UsageError,
    WorldSpec,
    ag_gemm,
    ag_order_switch,
    gemm_rs,
    init_world,
    make_ag_gemm_buffers,
    make_gemm_rs_buffers,
    rs_inter_order,
)
from paper_2504_19442_b200.primitives import WaitCond  # noqa: E402

pytestmark = pytest.mark.gpu
BF16 = torch.bfloat16


@contextlib.contextmanager
def make_world(world_size, heap_bytes=1 << 25, timeout_s=10.0):
    w = init_world(WorldSpec(world_size=world_size, heap_bytes=heap_bytes, timeout_s=timeout_s))
    try:
        yield w
    finally:
        w.close()


def ints(rng, lo, hi, shape):
    return rng.integers(lo, hi, shape).astype(np.float64)


def dev(x, pe):
    return torch.from_numpy(np.ascontiguousarray(x)).to(BF16).to(pe.torch_device)


def to_np(x):
    return x.float().cpu().numpy()


def perm_schedule(rank, order):
    return TileSchedule(rank, [TileStep(c, () if c == rank else (c,)) for c in order])


def _pipeline(w, rng, world_size, rows=256, n=192, k=128, rounds=2):
    shape = ProblemShape(m=rows * world_size, n=n, k=k, dtype="bfloat16")
    rs_shape = ProblemShape(m=rows * world_size, n=k, k=n, dtype="bfloat16")
    agb = make_ag_gemm_buffers(w, shape)
    rsb = make_gemm_rs_buffers(w, rs_shape)
    shards = [[ints(rng, -2, 3, (rows, k)) for _ in range(world_size)] for _ in range(rounds)]
    b = ints(rng, -1, 2, (k, n))
    amats = [[ints(rng, -1, 2, (rows * world_size, n)) for _ in range(world_size)]
             for _ in range(rounds)]
    d = ints(rng, -1, 2, (n, k))

    def body(pe):
        xs = [dev(shards[i][pe.rank], pe) for i in range(rounds)]
        As = [dev(amats[i][pe.rank], pe) for i in range(rounds)]
        bb, dd = dev(b, pe), dev(d, pe)
        return [(ag_gemm(pe, xs[i], bb, shape, ag_order_switch(pe.rank, world_size), agb,
                         reset=False),
                 gemm_rs(pe, As[i], dd, rs_shape, rs_inter_order(pe.ctx, 1, world_size), rsb,
                         reset=False))
                for i in range(rounds)]

    res = w.run(body)
    for r in range(world_size):
        for i in range(rounds):
            h, y = res[r][i]
            assert np.array_equal(to_np(h), oracle.ag_gemm_reference(shards[i], b))
            assert np.array_equal(to_np(y), oracle.gemm_rs_reference(amats[i], [d] * world_size)[r])
    return agb, rsb


@pytest.mark.parametrize("world_size", [2, 4])
def test_phased_protocol_matches_fused(rng, monkeypatch, world_size):
    monkeypatch.setenv("SHB_PHASED", "1")
    with make_world(world_size) as w:
        assert w.phased
        _pipeline(w, rng, world_size)
    monkeypatch.setenv("SHB_PHASED", "0")
    with make_world(world_size) as w:
        assert not w.phased
        _pipeline(w, rng, world_size)


@pytest.mark.parametrize("subchunks", ["1", "2", "3", "4", "7"])
def test_subchunk_flags_bit_exact(rng, monkeypatch, subchunks):
    monkeypatch.setenv("SHB_AG_SUB", subchunks)
    world_size, rows, k = 4, 1024, 256
    with make_world(world_size, heap_bytes=1 << 26) as w:
        agb, _ = _pipeline(w, rng, world_size, rows=rows, n=256, k=k, rounds=2)
        # ready[src] counts landed ranges: two calls -> 2 * S (S after the
        # 256-row rounding of the range size)
        s = int(subchunks)
        sub_rows = -(-(-(-rows // s)) // 256) * 256
        ranges = -(-rows // sub_rows)
        for r in range(world_size):
            vals = w.read_signals(r, agb.ready)
            assert [v for i, v in enumerate(vals) if i != r] == [2 * ranges] * (world_size - 1)
        # gathered layout is the plain vstack of the shards whatever the split
        assert np.array_equal(
            to_np(w.read_tensor(0, agb.gathered, BF16, (rows * world_size, k))).shape,
            (rows * world_size, k))


def test_default_subchunk_policy():
    from paper_2504_19442_b200 import _lib
    import ctypes

    lib = _lib.load()
    s = ctypes.c_int()
    # one flag per shard by default (tp_proxy.py: every flag write costs ~7 us
    # of front-end time); SHB_AG_SUB forces sub-chunks
    assert lib.sh_ag_subchunks(8192, 8192, 8, ctypes.byref(s)) == 0 and s.value == 1  # C3 TP=8
    assert lib.sh_ag_subchunks(8192, 8192, 1, ctypes.byref(s)) == 0 and s.value == 1
    assert lib.sh_ag_subchunks(1024, 8192, 8, ctypes.byref(s)) == 0 and s.value == 1  # 2 MB


@pytest.mark.parametrize("order", ["own_first", "reversed"])
def test_gemm_rs_own_chunk_first_many_tiles(rng, order):
    # 4 ranks share the GPU (37 CTA pairs each); a chunk of 1024 rows x 2048
    # columns is 32 pair tiles, 128 per rank: clusters queue several tiles.
    # The fused reduction waits inside own-chunk tiles; the library runs the
    # own chunk last whatever the caller's order.
    world_size, rows, n, k = 4, 1024, 2048, 64
    shape = ProblemShape(m=rows * world_size, n=n, k=k, dtype="bfloat16")
    with make_world(world_size, heap_bytes=1 << 26, timeout_s=20.0) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        amats = [ints(rng, -1, 2, (rows * world_size, k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (k, n))

        def sched(pe):
            if order == "own_first":
                return ag_order_switch(pe.rank, world_size)
            return perm_schedule(pe.rank, list(reversed(range(world_size))))

        res = w.run(lambda pe: gemm_rs(pe, dev(amats[pe.rank], pe), dev(b, pe), shape, sched(pe),
                                       bufs))
        ref = oracle.gemm_rs_reference(amats, [b] * world_size)
        for r in range(world_size):
            assert np.array_equal(to_np(res[r]), ref[r])


def test_wait_nobody_satisfies_is_a_timeout():
    with make_world(1, heap_bytes=1 << 16, timeout_s=0.5) as w:
        sig = w.alloc_signals(1)

        def body(pe):
            pe.signal_wait_until(sig.base, WaitCond.EQ, 5)

        with pytest.raises(CollectiveFault) as info:
            w.run(body)
        assert isinstance(info.value.first, SynchronizationFault)
        w.recover()
        w.run(lambda pe: pe.signal_op(pe.rank, sig.base, __import__(
            "paper_2504_19442_b200").SignalOp.SET, 5))
        assert w.sig_read(0, sig.base) == 5


_WEDGE = r"""
import os, sys
sys.path.insert(0, os.getcwd())
os.environ["SHB_WAIT_MEMOP"] = "1"
import paper_2504_19442_b200 as sb
from paper_2504_19442_b200.primitives import WaitCond
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=1 << 16, timeout_s=0.25))
sig = w.alloc_signals(1)
try:
    w.run(lambda pe: pe.signal_wait_until(sig.base, WaitCond.GE, 7))
except sb.CollectiveFault as exc:
    print("fault", type(exc.first).__name__, flush=True)
try:
    w.run(lambda pe: None)
except sb.UsageError:
    print("refused", flush=True)
try:
    w.recover()
    print("recovered", w.sweep_signals() == {}, w.run(lambda pe: pe.rank), flush=True)
except sb.ShmemError as exc:
    print("wedged", "restart" in str(exc), flush=True)
w.close()
print("closed", flush=True)
os._exit(0)
"""


@pytest.mark.timeout(150)
def test_stream_wait_that_never_passes_is_reported_not_hung():
    # the front-end wait (forced by SHB_WAIT_MEMOP) has no timeout of its own:
    # the host deadline (timeout*4 + 30 s, reference core.py:467-468) reports
    # it, the world refuses work until recover(), and neither recover() nor
    # close() blocks without bound.  A subprocess: a GPU queue that stays
    # wedged must not take the rest of the suite with it.
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _WEDGE], cwd=root, capture_output=True,
                         text=True, timeout=140)
    lines = res.stdout.split("\n")
    assert "fault SynchronizationFault" in lines, res.stdout + res.stderr
    assert "refused" in lines
    assert "recovered True [0]" in lines or "wedged True" in lines
    assert "closed" in lines


def test_device_acquires_every_remote_chunk(rng):
    # the timeline's kind-1 records are the producer warps' flag acquires:
    # every remote chunk is acquired, the own chunk never
    world_size = 4
    shape = ProblemShape(m=256 * world_size, n=256, k=128, dtype="bfloat16")
    with make_world(world_size) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        shards = [ints(rng, -2, 3, (256, 128)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (128, 256))
        w.start_trace()
        w.run(lambda pe: ag_gemm(pe, dev(shards[pe.rank], pe), dev(b, pe), shape,
                                 ag_order_switch(pe.rank, world_size), bufs))
        events = w.stop_trace()
    for r in range(world_size):
        waited = {e["chunk"] for e in events if e["rank"] == r and e["op"] == "chunk_wait"}
        assert waited == set(range(world_size)) - {r}, (r, waited)
