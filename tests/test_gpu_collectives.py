"""Standalone collectives on the GPU heap, written like the reference's
tests/test_collectives.py (push/pull AllGather layouts, RS all-ones and random
int64 bit-exact, world of one, size/dtype errors, signal hygiene)."""

import contextlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_19442_b200 import (ArgumentError, CollectiveFault, WorldSpec,  # noqa: E402
                                   init_world)
from paper_2504_19442_b200.collectives import (SYNC_TOKEN, SYNC_WAIT, ChunkLayout,  # noqa: E402
                                               allgather_pull_intra, allgather_push_intra,
                                               reducescatter_push_intra)
from paper_2504_19442_b200.primitives import SignalOp  # noqa: E402

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def make_world(world_size, heap_bytes=1 << 16):
    w = init_world(WorldSpec(world_size=world_size, heap_bytes=heap_bytes, timeout_s=10.0))
    try:
        yield w
    finally:
        w.close()


def ag_buffers(world, n):
    return world.alloc_symmetric(world.world_size * n, align=8), world.alloc_signals(world.world_size)


def view_bytes(pe, handle):
    return pe.local_view(handle).clone()  # device copy; converted after the run


def as_bytes(t):
    return t.cpu().numpy().tobytes()


def test_chunk_layout():
    lay = ChunkLayout(4, 32, 8)
    assert lay.chunk_elems == 8 and lay.chunk_bytes == 64 and lay.span(2) == (128, 64)
    with pytest.raises(ArgumentError):
        ChunkLayout(3, 32, 8)
    with pytest.raises(ArgumentError):
        lay.span(4)


def test_push_ag_concatenates_in_rank_order():
    with make_world(4) as w:
        dst, sigs = ag_buffers(w, 16)
        payloads = [np.arange(r * 10, r * 10 + 2, dtype=np.int64).tobytes() for r in range(4)]

        def body(pe):
            allgather_push_intra(pe, dst, sigs, payloads[pe.rank])
            return view_bytes(pe, dst)

        res = [as_bytes(t) for t in w.run(body)]
        want = b"".join(payloads)
        assert all(r == want for r in res)
        assert np.frombuffer(want, dtype=np.int64).tolist() == [0, 1, 10, 11, 20, 21, 30, 31]
        assert w.sweep_signals() == {}  # reset=True


def test_push_ag_world_of_one():
    with make_world(1) as w:
        dst, sigs = ag_buffers(w, 8)
        w.run(lambda pe: allgather_push_intra(pe, dst, sigs, b"lonechnk"))
        assert w.read_from(0, dst, 0, 8) == b"lonechnk"


def test_push_ag_randomized_vs_oracle(rng):
    with make_world(8) as w:
        dst, sigs = ag_buffers(w, 32)
        for _ in range(5):
            shards = [rng.integers(0, 256, 32, dtype=np.uint8).tobytes() for _ in range(8)]

            def body(pe):
                allgather_push_intra(pe, dst, sigs, shards[pe.rank])
                return view_bytes(pe, dst)

            want = b"".join(shards)
            assert all(as_bytes(r) == want for r in w.run(body))


def test_push_ag_size_mismatch():
    with make_world(2) as w:
        dst = w.alloc_symmetric(10)
        sigs = w.alloc_signals(2)
        with pytest.raises(CollectiveFault) as info:
            w.run(lambda pe: allgather_push_intra(pe, dst, sigs, b"eight..."))
        assert isinstance(info.value.first, ArgumentError)


def test_pull_ag_matches_push_and_uses_one_barrier(rng):
    with make_world(4) as w:
        dst_push, sigs_push = ag_buffers(w, 16)
        dst_pull, sigs_pull = ag_buffers(w, 16)
        shards = [rng.integers(0, 256, 16, dtype=np.uint8).tobytes() for _ in range(4)]

        def body(pe):
            allgather_push_intra(pe, dst_push, sigs_push, shards[pe.rank])
            allgather_pull_intra(pe, dst_pull, sigs_pull, shards[pe.rank], order=[3, 1, 0, 2])
            return view_bytes(pe, dst_push), view_bytes(pe, dst_pull)

        w.reset_counters()
        res = w.run(body)
        for a, b in res:
            assert as_bytes(a) == as_bytes(b) == b"".join(shards)
        for r in range(4):
            assert w.counters(r).get("barrier_all", 0) == 1


def test_push_ag_token_and_wait_styles_agree(rng):
    with make_world(4) as w:
        dst, sigs = ag_buffers(w, 16)
        shards = [rng.integers(0, 256, 16, dtype=np.uint8).tobytes() for _ in range(4)]
        outs = {}
        for style in (SYNC_WAIT, SYNC_TOKEN):
            def body(pe, style=style):
                allgather_push_intra(pe, dst, sigs, shards[pe.rank], sync_style=style)
                return view_bytes(pe, dst)

            outs[style] = [as_bytes(t) for t in w.run(body)]
        assert outs[SYNC_WAIT] == outs[SYNC_TOKEN]


def _rs_body(staging, psig, rsig, vals, chunk, dtype):
    def body(pe):
        for c in range(pe.world.world_size):
            pe.signal_op(pe.rank, psig.at(c), SignalOp.SET, 1)
        out = torch.zeros(chunk, dtype=dtype, device=pe.torch_device)
        x = torch.from_numpy(vals[pe.rank]).to(pe.torch_device)
        reducescatter_push_intra(pe, staging, psig, rsig, x, out)
        return out

    return body


def test_rs_intra_all_ones_and_world_one():
    with make_world(4) as w:
        staging, psig, rsig = w.alloc_symmetric(4 * 2 * 8), w.alloc_signals(4), w.alloc_signals(4)
        vals = [np.ones(8, dtype=np.int64)] * 4
        for out in w.run(_rs_body(staging, psig, rsig, vals, 2, torch.int64)):
            assert out.cpu().tolist() == [4, 4]
        assert w.sweep_signals() == {}
    with make_world(1) as w:
        staging, psig, rsig = w.alloc_symmetric(4 * 8), w.alloc_signals(1), w.alloc_signals(1)
        vals = [np.arange(4, dtype=np.int64)]
        assert w.run(_rs_body(staging, psig, rsig, vals, 4, torch.int64))[0].cpu().tolist() == \
            [0, 1, 2, 3]


@pytest.mark.parametrize("dtype,np_dtype", [(torch.int64, np.int64), (torch.int32, np.int32),
                                            (torch.float32, np.float32)])
def test_rs_intra_random_vs_oracle(rng, dtype, np_dtype):
    with make_world(8, heap_bytes=1 << 18) as w:
        chunk = 64
        esize = np.dtype(np_dtype).itemsize
        staging, psig, rsig = (w.alloc_symmetric(8 * chunk * esize), w.alloc_signals(8),
                               w.alloc_signals(8))
        for _ in range(3):
            if np_dtype == np.float32:
                vals = [rng.standard_normal(8 * chunk).astype(np_dtype) for _ in range(8)]
            else:
                info = np.iinfo(np_dtype)
                vals = [rng.integers(info.min // 8, info.max // 8, 8 * chunk).astype(np_dtype)
                        for _ in range(8)]
            res = w.run(_rs_body(staging, psig, rsig, vals, chunk, dtype))
            acc = np.zeros((8, chunk), dtype=np_dtype)
            for v in vals:  # ascending source order, element-type accumulation
                acc += v.reshape(8, chunk)
            for r in range(8):
                assert np.array_equal(res[r].cpu().numpy(), acc[r])


def test_rs_intra_dtype_mismatch():
    with make_world(2) as w:
        staging, psig, rsig = w.alloc_symmetric(2 * 4 * 8), w.alloc_signals(2), w.alloc_signals(2)

        def body(pe):
            out = torch.zeros(4, dtype=torch.int32, device=pe.torch_device)
            x = torch.ones(8, dtype=torch.int64, device=pe.torch_device)
            reducescatter_push_intra(pe, staging, psig, rsig, x, out)

        with pytest.raises(CollectiveFault) as info:
            w.run(body)
        assert isinstance(info.value.first, ArgumentError)


def test_primitives_put_get_signal_roundtrip():
    from paper_2504_19442_b200.primitives import WaitCond

    with make_world(2) as w:
        buf = w.alloc_symmetric(64)
        sigs = w.alloc_signals(2)

        def body(pe):
            peer = 1 - pe.rank
            pe.putmem(buf, bytes([pe.rank + 1]) * 32, peer, dst_off=32 * pe.rank)
            pe.signal_op(peer, sigs.at(pe.rank), SignalOp.ADD, 5)
            pe.signal_wait_until(sigs.at(peer), WaitCond.GE, 5)
            got = torch.empty(32, dtype=torch.uint8, device=pe.torch_device)
            pe.getmem(got, buf, pe.rank, nbytes=32, src_off=32 * peer)
            return got

        res = w.run(body)
        assert res[0].cpu().tolist() == [2] * 32 and res[1].cpu().tolist() == [1] * 32
        assert w.sig_read(0, sigs.at(1)) == 5 and w.sig_read(1, sigs.at(0)) == 5


def test_world_copy_into_and_read_from():
    with make_world(2) as w:
        h = w.alloc_symmetric(16)
        w.copy_into(1, h, 4, b"abcdefgh")
        assert w.read_from(1, h, 4, 8) == b"abcdefgh"
        assert w.read_from(0, h, 0, 16) == bytes(16)


# ---------------------------------------------------------------------------
# node-scope multimem (reference tests/test_primitives.py:211-256)

def test_multimem_st_broadcasts_within_node():
    # one NVSwitch node (multi-node worlds are out of scope): every rank's
    # replica receives rank 1's bytes, the other ranks' zeros are overwritten
    with make_world(4, heap_bytes=1 << 10) as w:
        h = w.alloc_symmetric(16)

        def body(pe):
            if pe.rank == 1:
                pe.putmem(h, b"n" * 16, pe.rank)
                pe.multimem_st(h)
            pe.barrier_all()
            return view_bytes(pe, h)

        res = [as_bytes(t) for t in w.run(body)]
        assert all(r == b"n" * 16 for r in res)
        assert w.counters(1).get("multimem_st") == 1
        assert w.counters(0).get("multimem_st", 0) == 0


def test_multimem_ld_reduce_sums_node():
    with make_world(4, heap_bytes=1 << 10) as w:
        h = w.alloc_symmetric(16)

        def body(pe):
            vals = np.full(2, pe.rank + 1, dtype=np.int64)
            pe.putmem(h, vals.tobytes(), pe.rank)
            pe.barrier_all()
            return pe.multimem_ld_reduce(h, np.int64)

        for got in w.run(body):
            assert got.cpu().tolist() == [10, 10]  # 1+2+3+4
        with pytest.raises(CollectiveFault) as info:
            w.run(lambda pe: pe.multimem_ld_reduce(h, np.int64, nbytes=12))
        assert isinstance(info.value.first, ArgumentError)


def test_multimem_single_rank_node_identity():
    # a node of one rank: multimem_st is a no-op, ld_reduce returns the replica
    with make_world(1, heap_bytes=1 << 10) as w:
        h = w.alloc_symmetric(8)

        def body(pe):
            pe.putmem(h, bytes([pe.rank + 1] * 8), pe.rank)
            pe.multimem_st(h)
            return pe.multimem_ld_reduce(h, np.uint8)

        assert [t.cpu().tolist() for t in w.run(body)] == [[1] * 8]


@pytest.mark.parametrize("dtype", ["bfloat16", "float16", "float32", "int32", "int64", "uint8",
                                   "int8"])
@pytest.mark.parametrize("nbytes_extra", [0, 8])  # 16-B vector path and the scalar tail
def test_multimem_ld_reduce_matches_numpy_accumulation(rng, dtype, nbytes_extra):
    # the per-step arithmetic of the reference's `out += replica` (floats round
    # to the element type after every add, integers wrap), ascending ranks
    import ml_dtypes  # noqa: F401  (numpy bfloat16)

    W = 4
    npdt = np.dtype("bfloat16" if dtype == "bfloat16" else dtype)
    elems = (4096 + nbytes_extra) // npdt.itemsize
    if np.issubdtype(npdt, np.integer):
        info = np.iinfo(npdt)
        reps = [rng.integers(info.min, info.max, elems, endpoint=True).astype(npdt)
                for _ in range(W)]
    else:
        reps = [(rng.standard_normal(elems) * 100).astype(np.float32).astype(npdt)
                for _ in range(W)]
    expect = np.zeros(elems, dtype=npdt)
    with np.errstate(over="ignore"):
        for r in reps:
            expect += r
    with make_world(W, heap_bytes=1 << 16) as w:
        h = w.alloc_symmetric(reps[0].nbytes, align=16)

        def body(pe):
            pe.putmem(h, reps[pe.rank].tobytes(), pe.rank)
            pe.barrier_all()
            return pe.multimem_ld_reduce(h, dtype)

        for got in w.run(body):
            g = got.cpu()
            if dtype == "bfloat16":
                g = g.view(torch.int16).numpy().view(np.uint16)
                e = expect.view(np.uint16)
            else:
                g, e = g.numpy(), expect
            assert g.tobytes() == e.tobytes()


def test_multimem_st_large_unaligned_range(rng):
    # a range that is neither 16-B aligned nor a multiple of 16 B takes the
    # byte path; a large aligned one the vector path
    W = 3
    with make_world(W, heap_bytes=1 << 21) as w:
        h = w.alloc_symmetric(1 << 20, align=256)
        data = rng.integers(0, 256, 1 << 20, dtype=np.uint8)

        def body(pe):
            if pe.rank == 2:
                pe.putmem(h, data.tobytes(), pe.rank)
                pe.multimem_st(h, off=0, nbytes=(1 << 19))        # vector path
                pe.multimem_st(h, off=(1 << 19) + 3, nbytes=1001)  # byte path
            pe.barrier_all()
            return view_bytes(pe, h)

        res = [t.cpu().numpy() for t in w.run(body)]
        for r in range(W):
            assert np.array_equal(res[r][:1 << 19], data[:1 << 19])
            lo = (1 << 19) + 3
            assert np.array_equal(res[r][lo:lo + 1001], data[lo:lo + 1001])
            if r != 2:
                assert not res[r][lo + 1001:].any() and not res[r][(1 << 19):lo].any()
