"""ag_gemm / gemm_rs on the GPU, written like the reference's own suite
(/root/reference/pkg/tests/test_pipelines.py): identity shards give back B,
random integer inputs match the dense oracle bit-exactly, schedule
invariance, shape errors -> ArgumentError inside CollectiveFault, RS all-ones
pattern, world of one.  Ranks are threads of one process (the reference's
model); on a one-GPU box all W ranks share cuda:0, each on its own stream, and
every "remote" store or flag goes through the same peer-pointer path the
multi-GPU world uses."""

import contextlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import minishmem_oracle as oracle  # noqa: E402
from paper_2504_19442_b200 import (  # noqa: E402
    ArgumentError,
    CollectiveFault,
    ProblemShape,
    TileSchedule,
    TileStep,
    WorldSpec,
    ag_gemm,
    ag_order_switch,
    gemm_rs,
    init_world,
    make_ag_gemm_buffers,
    make_gemm_rs_buffers,
    rs_inter_order,
)

pytestmark = pytest.mark.gpu
BF16 = torch.bfloat16


@contextlib.contextmanager
def make_world(world_size, heap_bytes=1 << 24, timeout_s=10.0):
    w = init_world(WorldSpec(world_size=world_size, heap_bytes=heap_bytes, timeout_s=timeout_s))
    try:
        yield w
    finally:
        w.close()


def to_np(x):
    if isinstance(x, torch.Tensor):
        return x.float().cpu().numpy()
    if isinstance(x, (list, tuple)):
        return type(x)(to_np(v) for v in x)
    return x


def run_np(world, body):
    """Run ``body`` on every rank and convert the results afterwards: a rank
    body must not block on a device->host copy while sibling ranks of the
    same process still have to launch (the driver serialises pageable
    copies, so the blocked copy would hold back a peer's launch)."""
    return [to_np(r) for r in world.run(body)]


def perm_schedule(rank, order):
    return TileSchedule(rank, [TileStep(c, () if c == rank else (c,)) for c in order])


def ints(rng, lo, hi, shape):
    # integer-valued, held in float64: the oracle's matmuls run on BLAS
    # (numpy's int64 matmul is a scalar loop) and stay exact at these sizes
    return rng.integers(lo, hi, shape).astype(np.float64)


def dev(x, rank_pe):
    return torch.from_numpy(np.ascontiguousarray(x)).to(BF16).to(rank_pe.torch_device)


def test_ag_gemm_identity_shards_give_back_b(rng):
    shape = ProblemShape(m=256, n=64, k=256, dtype="bfloat16")
    with make_world(2) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        eye = np.eye(256, dtype=np.int64)
        shards = [eye[:128], eye[128:]]
        b = ints(rng, -1, 2, (256, 64))

        def body(pe):
            out = ag_gemm(pe, dev(shards[pe.rank], pe), dev(b, pe), shape,
                          ag_order_switch(pe.rank, 2), bufs)
            return out

        for out in run_np(w, body):
            assert np.array_equal(out, b)


@pytest.mark.parametrize("world_size", [1, 2, 4, 8])
def test_ag_gemm_random_vs_dense_oracle(rng, world_size):
    shape = ProblemShape(m=256 * world_size, n=192, k=320, dtype="bfloat16")
    rows = shape.m // world_size
    with make_world(world_size) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        shards = [ints(rng, -2, 3, (rows, shape.k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (shape.k, shape.n))
        ref = oracle.ag_gemm_reference(shards, b)
        assert np.abs(ref).max() < 256  # exact in bf16

        def body(pe):
            return ag_gemm(pe, dev(shards[pe.rank], pe), dev(b, pe), shape,
                           ag_order_switch(pe.rank, world_size), bufs)

        for r, out in enumerate(run_np(w, body)):
            assert np.array_equal(out, ref)
            # bit-exact gathered layout: slot s = rank s's shard (collectives.py:95-97)
            gathered = to_np(w.read_tensor(r, bufs.gathered, BF16, (shape.m, shape.k)))
            assert np.array_equal(gathered, oracle.gathered_layout(shards))


def test_ag_gemm_schedule_invariance(rng):
    shape = ProblemShape(m=512, n=128, k=128, dtype="bfloat16")
    with make_world(4) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        shards = [ints(rng, -2, 3, (128, 128)) for _ in range(4)]
        b = ints(rng, -1, 2, (128, 128))
        ref = oracle.ag_gemm_reference(shards, b)
        orders = [
            lambda pe: ag_order_switch(pe.rank, 4),
            lambda pe: rs_inter_order(pe.ctx, 1, 4),
            lambda pe: perm_schedule(pe.rank, [3, 1, 0, 2]),
            lambda pe: perm_schedule(pe.rank, list(reversed(range(4)))),
        ]
        for make_sched in orders:
            def body(pe):
                return ag_gemm(pe, dev(shards[pe.rank], pe), dev(b, pe), shape, make_sched(pe),
                               bufs)

            for out in run_np(w, body):
                assert np.array_equal(out, ref)


def test_ag_gemm_back_to_back_without_reset(rng):
    # epochs make consecutive calls safe with no reset or join in between
    shape = ProblemShape(m=512, n=256, k=256, dtype="bfloat16")
    with make_world(4) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        rounds = 5
        shards = [[ints(rng, -1, 2, (128, 256)) for _ in range(4)] for _ in range(rounds)]
        b = ints(rng, -1, 2, (256, 256))

        def body(pe):
            bb = dev(b, pe)
            xs = [dev(shards[i][pe.rank], pe) for i in range(rounds)]  # stage first
            outs = [ag_gemm(pe, xs[i], bb, shape, ag_order_switch(pe.rank, 4), bufs, reset=False)
                    for i in range(rounds)]
            return outs

        for outs in run_np(w, body):
            for i, out in enumerate(outs):
                assert np.array_equal(out, oracle.ag_gemm_reference(shards[i], b))


def test_ag_gemm_flags_zero_after_reset(rng):
    shape = ProblemShape(m=256, n=64, k=64, dtype="bfloat16")
    with make_world(2) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        shards = [ints(rng, -2, 3, (128, 64)) for _ in range(2)]
        b = ints(rng, -1, 2, (64, 64))
        run_np(w, lambda pe: ag_gemm(pe, dev(shards[pe.rank], pe), dev(b, pe), shape,
                                 ag_order_switch(pe.rank, 2), bufs))
        assert w.sweep_signals() == {}


def test_ag_gemm_wait_counts_and_no_barriers(rng):
    shape = ProblemShape(m=512, n=64, k=64, dtype="bfloat16")
    with make_world(4) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        shards = [ints(rng, -2, 3, (128, 64)) for _ in range(4)]
        b = ints(rng, -1, 2, (64, 64))
        w.reset_counters()
        w.start_trace(records_per_cta=64, launches=2)
        run_np(w, lambda pe: ag_gemm(pe, dev(shards[pe.rank], pe), dev(b, pe), shape,
                                 ag_order_switch(pe.rank, 4), bufs))
        events = w.stop_trace()
        for r in range(4):
            c = w.counters(r)
            assert c.get("wait", 0) == 3
            assert c.get("barrier_all", 0) == 0
            # the device side of those waits (not the host wrapper's count):
            # the producers' acquire spins on ready[c] (timeline kind 1) cover
            # exactly the 3 remote chunks, never the rank's own shard
            waited = {e["chunk"] for e in events if e["rank"] == r and e["op"] == "chunk_wait"}
            assert waited == set(range(4)) - {r}


def test_ag_gemm_shape_mismatch():
    shape = ProblemShape(m=256, n=64, k=64, dtype="bfloat16")
    with make_world(2) as w:
        bufs = make_ag_gemm_buffers(w, shape)

        def body(pe):
            bad = torch.zeros((3, 64), dtype=BF16, device=pe.torch_device)
            b = torch.zeros((64, 64), dtype=BF16, device=pe.torch_device)
            return ag_gemm(pe, bad, b, shape, ag_order_switch(pe.rank, 2), bufs)

        with pytest.raises(CollectiveFault) as info:
            run_np(w, body)
        assert isinstance(info.value.first, ArgumentError)


def test_ag_gemm_non_covering_schedule_rejected():
    shape = ProblemShape(m=256, n=64, k=64, dtype="bfloat16")
    with make_world(2) as w:
        bufs = make_ag_gemm_buffers(w, shape)

        def body(pe):
            a = torch.zeros((128, 64), dtype=BF16, device=pe.torch_device)
            b = torch.zeros((64, 64), dtype=BF16, device=pe.torch_device)
            return ag_gemm(pe, a, b, shape, perm_schedule(pe.rank, [0]), bufs)

        with pytest.raises(CollectiveFault) as info:
            run_np(w, body)
        assert isinstance(info.value.first, ArgumentError)


def test_gemm_rs_world_of_one_is_plain_matmul(rng):
    shape = ProblemShape(m=256, n=128, k=192, dtype="bfloat16")
    with make_world(1) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        a = ints(rng, -2, 3, (256, 192))
        b = ints(rng, -1, 2, (192, 128))
        out = run_np(w, lambda pe: gemm_rs(pe, dev(a, pe), dev(b, pe), shape,
                                       rs_inter_order(pe.ctx, 1, 1), bufs))
        assert np.array_equal(out[0], a @ b)


def test_gemm_rs_all_ones_contribution_pattern():
    shape = ProblemShape(m=256, n=64, k=64, dtype="bfloat16")
    with make_world(2) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        a = np.ones((256, 64), dtype=np.int64)
        b = np.eye(64, dtype=np.int64)
        outs = run_np(w, lambda pe: gemm_rs(pe, dev(a, pe), dev(b, pe), shape,
                                        rs_inter_order(pe.ctx, 1, 2), bufs))
        for out in outs:
            assert (out == 2).all()


@pytest.mark.parametrize("world_size", [2, 4, 8])
def test_gemm_rs_intra_random_vs_oracle(rng, world_size):
    shape = ProblemShape(m=256 * world_size, n=192, k=128, dtype="bfloat16")
    rows = shape.m // world_size
    with make_world(world_size) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        amats = [ints(rng, -2, 3, (shape.m, shape.k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (shape.k, shape.n))
        ref = oracle.gemm_rs_reference(amats, [b] * world_size)
        assert np.abs(ref).max() < 256

        def body(pe):
            return gemm_rs(pe, dev(amats[pe.rank], pe), dev(b, pe), shape,
                           rs_inter_order(pe.ctx, 1, world_size), bufs)

        for r, out in enumerate(run_np(w, body)):
            assert np.array_equal(out, ref[r])
            staging = to_np(w.read_tensor(r, bufs.staging, BF16, (world_size, rows, shape.n)))
            # bit-exact scatter layout: slot s on rank r = rows r of A_s @ B_s
            expect = oracle.staging_layout(amats, [b] * world_size, r)
            assert np.array_equal(staging, expect)


def test_gemm_rs_schedule_invariance_intra(rng):
    shape = ProblemShape(m=1024, n=128, k=128, dtype="bfloat16")
    with make_world(4) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        amats = [ints(rng, -2, 3, (1024, 128)) for _ in range(4)]
        b = ints(rng, -1, 2, (128, 128))
        ref = oracle.gemm_rs_reference(amats, [b] * 4)
        for order in ([0, 1, 2, 3], [2, 0, 3, 1], [3, 2, 1, 0]):
            outs = run_np(w, lambda pe: gemm_rs(pe, dev(amats[pe.rank], pe), dev(b, pe), shape,
                                            perm_schedule(pe.rank, order),
                                            bufs))
            for r, out in enumerate(outs):
                assert np.array_equal(out, ref[r])


def test_gemm_rs_back_to_back_without_reset(rng):
    shape = ProblemShape(m=1024, n=256, k=128, dtype="bfloat16")
    with make_world(4) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        rounds = 4
        amats = [[ints(rng, -2, 3, (1024, 128)) for _ in range(4)] for _ in range(rounds)]
        b = ints(rng, -1, 2, (128, 256))

        def body(pe):
            bb = dev(b, pe)
            xs = [dev(amats[i][pe.rank], pe) for i in range(rounds)]  # stage first
            outs = [gemm_rs(pe, xs[i], bb, shape, rs_inter_order(pe.ctx, 1, 4), bufs, reset=False)
                    for i in range(rounds)]
            return outs

        for r, outs in enumerate(run_np(w, body)):
            for i, out in enumerate(outs):
                assert np.array_equal(out, oracle.gemm_rs_reference(amats[i], [b] * 4)[r])


def test_tp_mlp_float_tolerance():
    # the Llama-MLP pattern at reduced size: X shard -> ag_gemm -> H -> gemm_rs -> Y shard,
    # random normal bf16, rel Frobenius <= 1e-2 vs an fp32 reference (north star)
    W, M, K, N = 4, 1024, 512, 768
    g = np.random.default_rng(0)
    xs = [g.standard_normal((M // W, K)).astype(np.float32) for _ in range(W)]
    ups = [g.standard_normal((K, N // W)).astype(np.float32) * 0.05 for _ in range(W)]
    downs = [g.standard_normal((N // W, K)).astype(np.float32) * 0.05 for _ in range(W)]
    ag_shape = ProblemShape(m=M, n=N // W, k=K, dtype="bfloat16")
    rs_shape = ProblemShape(m=M, n=K, k=N // W, dtype="bfloat16")
    with make_world(W, heap_bytes=1 << 25) as w:
        agb = make_ag_gemm_buffers(w, ag_shape)
        rsb = make_gemm_rs_buffers(w, rs_shape)

        def body(pe):
            t = lambda x: torch.from_numpy(x).to(BF16).to(pe.torch_device)  # noqa: E731
            x, up, down = t(xs[pe.rank]), t(ups[pe.rank]), t(downs[pe.rank])  # stage first
            h = ag_gemm(pe, x, up, ag_shape, ag_order_switch(pe.rank, W), agb)
            y = gemm_rs(pe, h, down, rs_shape, rs_inter_order(pe.ctx, 1, W), rsb)
            return h, y

        res = run_np(w, body)
    xb = [torch.from_numpy(x).to(BF16).float().numpy() for x in xs]
    ub = [torch.from_numpy(x).to(BF16).float().numpy() for x in ups]
    db = [torch.from_numpy(x).to(BF16).float().numpy() for x in downs]
    x_full = np.vstack(xb)
    hs = [x_full @ ub[r] for r in range(W)]
    y_full = sum(torch.from_numpy(hs[r]).to(BF16).float().numpy() @ db[r] for r in range(W))
    for r, (h, y) in enumerate(res):
        assert np.linalg.norm(h - hs[r]) / np.linalg.norm(hs[r]) < 1e-2
        rows = M // W
        ref = y_full[r * rows:(r + 1) * rows]
        assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 1e-2


@pytest.mark.parametrize("dyn", ["0", "1"])
@pytest.mark.parametrize("world_size", [1, 2])
def test_ag_gemm_stream_k_tail_exact(rng, monkeypatch, world_size, dyn):
    # enough tiles for the stream-K tail (80 on 74 CTA pairs at W=1); dyn=1
    # hands the data-parallel tiles out through the atomic counter
    monkeypatch.setenv("SHB_SK", "1")
    monkeypatch.setenv("SHB_DYN", dyn)
    shape = ProblemShape(m=2560, n=2048, k=512, dtype="bfloat16")
    rows = shape.m // world_size
    with make_world(world_size, heap_bytes=1 << 26) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        shards = [ints(rng, -2, 3, (rows, shape.k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (shape.k, shape.n))
        ref = oracle.ag_gemm_reference(shards, b)
        assert np.abs(ref).max() < 256

        def body(pe):
            x, bb = dev(shards[pe.rank], pe), dev(b, pe)
            return [ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, world_size), bufs,
                            reset=False) for _ in range(2)]

        for r, outs in enumerate(run_np(w, body)):
            for out in outs:
                assert np.array_equal(out, ref)
            gathered = to_np(w.read_tensor(r, bufs.gathered, BF16, (shape.m, shape.k)))
            assert np.array_equal(gathered, oracle.gathered_layout(shards))


@pytest.mark.parametrize("dyn", ["0", "1"])
@pytest.mark.parametrize("world_size", [1, 2])
def test_gemm_rs_stream_k_tail_exact(rng, monkeypatch, world_size, dyn):
    # the fused RS epilogue behind stream-K partial tiles: finishers publish
    # the summed tile into the peers' staging slots (W=2: 160 tiles on 37
    # clusters per rank, the 49-tile stream-K range inside the own chunk)
    monkeypatch.setenv("SHB_SK", "1")
    monkeypatch.setenv("SHB_DYN", dyn)
    shape = ProblemShape(m=2560 * world_size, n=2048, k=512, dtype="bfloat16")
    with make_world(world_size, heap_bytes=1 << 26) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        amats = [ints(rng, -2, 3, (shape.m, shape.k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (shape.k, shape.n))
        ref = oracle.gemm_rs_reference(amats, [b] * world_size)
        assert max(np.abs(r).max() for r in ref) < 256

        def body(pe):
            a, bb = dev(amats[pe.rank], pe), dev(b, pe)
            return [gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, world_size), bufs,
                            reset=False) for _ in range(2)]

        for r, outs in enumerate(run_np(w, body)):
            for out in outs:
                assert np.array_equal(out, ref[r])


@pytest.mark.parametrize("world_size,rows,n,k", [(3, 200, 200, 72), (2, 130, 264, 520),
                                                 (5, 64, 136, 40), (1, 1000, 1000, 1000)])
def test_ragged_shapes_ag_and_rs_exact(rng, world_size, rows, n, k):
    # rows / n / k that are not multiples of the 256 x 256 x 64 tiles, odd worlds:
    # TMA clips the edges, chunk boundaries never mix (3D maps)
    m = rows * world_size
    ag_shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    rs_shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    with make_world(world_size, heap_bytes=1 << 26) as w:
        agb, rsb = make_ag_gemm_buffers(w, ag_shape), make_gemm_rs_buffers(w, rs_shape)
        shards = [ints(rng, -2, 3, (rows, k)) for _ in range(world_size)]
        amats = [ints(rng, -1, 2, (m, k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (k, n))
        ag_ref = oracle.ag_gemm_reference(shards, b)
        rs_ref = oracle.gemm_rs_reference(amats, [b] * world_size)
        assert np.abs(ag_ref).max() < 256 and max(np.abs(r).max() for r in rs_ref) < 256

        def body(pe):
            x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
            h = ag_gemm(pe, x, bb, ag_shape, ag_order_switch(pe.rank, world_size), agb)
            y = gemm_rs(pe, a, bb, rs_shape, rs_inter_order(pe.ctx, 1, world_size), rsb)
            return h, y

        for r, (h, y) in enumerate(run_np(w, body)):
            assert np.array_equal(h, ag_ref)
            assert np.array_equal(y, rs_ref[r])
            staging = to_np(w.read_tensor(r, rsb.staging, BF16, (world_size, rows, n)))
            assert np.array_equal(staging, oracle.staging_layout(amats, [b] * world_size, r))
            gathered = to_np(w.read_tensor(r, agb.gathered, BF16, (m, k)))
            assert np.array_equal(gathered, oracle.gathered_layout(shards))


@pytest.mark.parametrize("world_size", [1, 2])
def test_gemm_rs_fused_and_unfused_calls_interleave(rng, monkeypatch, world_size):
    # the per-source element counters advance identically with the reduction
    # fused into the epilogue or run as a separate kernel (SHB_RS_UNFUSED=1),
    # so the two can alternate on one buffer set without stalls
    shape = ProblemShape(m=512 * world_size, n=256, k=128, dtype="bfloat16")
    with make_world(world_size, heap_bytes=1 << 26, timeout_s=5.0) as w:
        bufs = make_gemm_rs_buffers(w, shape)
        amats = [ints(rng, -2, 3, (shape.m, shape.k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (shape.k, shape.n))
        ref = oracle.gemm_rs_reference(amats, [b] * world_size)
        for mode in ["0", "1", "0", "1", "1", "0"]:
            monkeypatch.setenv("SHB_RS_UNFUSED", mode)

            def body(pe):
                a, bb = dev(amats[pe.rank], pe), dev(b, pe)
                return gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, world_size), bufs,
                               reset=False)

            for r, y in enumerate(run_np(w, body)):
                assert np.array_equal(y, ref[r])
            for r in range(world_size):
                w.check_errors(r)


@pytest.mark.parametrize("cg", [0, 1, 2])  # 0: automatic (1-CTA tiles for chunks <= 128 rows)
@pytest.mark.parametrize("world_size,rows,n,k", [(8, 128, 512, 256), (4, 128, 384, 136),
                                                 (2, 384, 264, 200)])
def test_fused_ops_exact_per_tile_config(rng, world_size, rows, n, k, cg):
    # TP=8 at M=1024 gives 128-row chunks: the automatic choice switches to
    # single-CTA tiles there; both fused epilogues must stay bit-exact either way
    from paper_2504_19442_b200 import _lib

    lib = _lib.load()
    _lib.check(lib.sh_set_tile_config(0, cg))
    try:
        m = rows * world_size
        shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
        with make_world(world_size, heap_bytes=1 << 26) as w:
            agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
            shards = [ints(rng, -2, 3, (rows, k)) for _ in range(world_size)]
            amats = [ints(rng, -1, 2, (m, k)) for _ in range(world_size)]
            b = ints(rng, -1, 2, (k, n))
            ag_ref = oracle.ag_gemm_reference(shards, b)
            rs_ref = oracle.gemm_rs_reference(amats, [b] * world_size)

            def body(pe):
                x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
                hs = [ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, world_size), agb,
                              reset=False) for _ in range(2)]
                ys = [gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, world_size), rsb,
                              reset=False) for _ in range(2)]
                return hs, ys

            for r, (hs, ys) in enumerate(run_np(w, body)):
                for h in hs:
                    assert np.array_equal(h, ag_ref)
                for y in ys:
                    assert np.array_equal(y, rs_ref[r])
                staging = to_np(w.read_tensor(r, rsb.staging, BF16, (world_size, rows, n)))
                assert np.array_equal(staging, oracle.staging_layout(amats, [b] * world_size, r))
                gathered = to_np(w.read_tensor(r, agb.gathered, BF16, (m, k)))
                assert np.array_equal(gathered, oracle.gathered_layout(shards))
    finally:
        lib.sh_set_tile_config(0, 0)


def test_unaligned_row_length_padded_on_device(rng):
    # TMA rows are 16-byte multiples: a ragged n / k is zero-padded on the
    # device by the drop-in (exact -- the padding adds zeros), never routed
    # to a CPU fallback; the C ABI itself still refuses it
    shape = ProblemShape(m=256, n=12, k=60, dtype="bfloat16")
    with make_world(1) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        rs_bufs = make_gemm_rs_buffers(w, ProblemShape(m=256, n=12, k=60, dtype="bfloat16"))
        a = ints(rng, -2, 3, (256, 60))
        b = ints(rng, -1, 2, (60, 12))

        def body(pe):
            h = ag_gemm(pe, dev(a, pe), dev(b, pe), shape, ag_order_switch(0, 1), bufs)
            y = gemm_rs(pe, dev(a, pe), dev(b, pe), shape, rs_inter_order(pe.ctx, 1, 1), rs_bufs)
            return h, y

        h, y = run_np(w, body)[0]
        assert h.shape == (256, 12) and np.array_equal(h, a @ b)
        assert y.shape == (256, 12) and np.array_equal(y, a @ b)
    from paper_2504_19442_b200 import _lib

    assert _lib.load().sh_gemm(None, None, None, 256, 12, 64, 0, None, 0, None) == _lib.SH_ERR_ARG


def test_criterion_6_pipeline_correctness_on_gpu():
    # reference tests/test_acceptance.py:418-486 on the GPU path: W in {1,2,4,8},
    # ProblemShape(64, 32, 32, tile_m=4, tile_n=16), four schedules, seed 77;
    # payloads in [-1, 1] keep every product and sum exact in bf16
    from paper_2504_19442_b200 import ag_order_fullmesh

    rng = np.random.default_rng(77)
    for world_size in (1, 2, 4, 8):
        shape = ProblemShape(m=64, n=32, k=32, dtype="bfloat16", tile_m=4, tile_n=16)
        rows = shape.rows_per_rank(world_size)
        with make_world(world_size, heap_bytes=1 << 20) as w:
            ag_bufs, rs_bufs = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
            shards = [ints(rng, -1, 2, (rows, shape.k)) for _ in range(world_size)]
            amats = [ints(rng, -1, 2, (shape.m, shape.k)) for _ in range(world_size)]
            b = ints(rng, -1, 2, (shape.k, shape.n))
            ag_ref = np.vstack(shards) @ b
            rs_ref = sum(a @ b for a in amats)
            perm = list(rng.permutation(world_size))
            schedules = [
                lambda pe: ag_order_switch(pe.rank, world_size),
                lambda pe: rs_inter_order(pe.ctx, 1, world_size),
                lambda pe: perm_schedule(pe.rank, perm),
                lambda pe: ag_order_fullmesh(pe.rank, world_size, 1),
            ]
            outs = []
            for make_sched in schedules:
                def body(pe):
                    x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
                    return (ag_gemm(pe, x, bb, shape, make_sched(pe), ag_bufs),
                            gemm_rs(pe, a, bb, shape, make_sched(pe), rs_bufs))

                res = run_np(w, body)
                for r, (h, y) in enumerate(res):
                    assert np.array_equal(h, ag_ref)
                    assert np.array_equal(y, rs_ref[r * rows:(r + 1) * rows])
                outs.append(res)
            for other in outs[1:]:  # bit-identical across schedules
                for (h0, y0), (h1, y1) in zip(outs[0], other):
                    assert np.array_equal(h0, h1) and np.array_equal(y0, y1)


@pytest.mark.parametrize("world_size", [1, 2])
def test_wave_lockstep_exact(rng, monkeypatch, world_size):
    # opt-in wave lockstep (SHB_WAVE=1) of the data-parallel tiles: several
    # waves per rank, both fused ops, back-to-back calls (epoch-tagged flags)
    monkeypatch.setenv("SHB_WAVE", "1")
    shape = ProblemShape(m=4096 * world_size, n=2048, k=256, dtype="bfloat16")
    rows = shape.m // world_size
    with make_world(world_size, heap_bytes=1 << 27) as w:
        agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
        shards = [ints(rng, -2, 3, (rows, shape.k)) for _ in range(world_size)]
        amats = [ints(rng, -1, 2, (shape.m, shape.k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (shape.k, shape.n))
        ag_ref = oracle.ag_gemm_reference(shards, b)
        rs_ref = oracle.gemm_rs_reference(amats, [b] * world_size)

        def body(pe):
            x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
            hs = [ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, world_size), agb,
                          reset=False) for _ in range(3)]
            ys = [gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, world_size), rsb,
                          reset=False) for _ in range(3)]
            return hs, ys

        for r, (hs, ys) in enumerate(run_np(w, body)):
            for h in hs:
                assert np.array_equal(h, ag_ref)
            for y in ys:
                assert np.array_equal(y, rs_ref[r])


@pytest.mark.parametrize("world_size", [1, 2, 4])
def test_fp16_fused_ops_exact_and_layouts(rng, world_size):
    # the fp16 instantiation of both fused kernels: integer inputs whose sums
    # stay below 2048 are exact in fp16, layouts bit-exact
    F16 = torch.float16
    rows, n, k = 256, 320, 192
    m = rows * world_size
    shape = ProblemShape(m=m, n=n, k=k, dtype="float16")
    with make_world(world_size, heap_bytes=1 << 26) as w:
        agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
        shards = [ints(rng, -3, 4, (rows, k)) for _ in range(world_size)]
        amats = [ints(rng, -2, 3, (m, k)) for _ in range(world_size)]
        b = ints(rng, -2, 3, (k, n))
        ag_ref = oracle.ag_gemm_reference(shards, b)
        rs_ref = oracle.gemm_rs_reference(amats, [b] * world_size)
        assert np.abs(ag_ref).max() < 2048 and max(np.abs(r).max() for r in rs_ref) < 2048

        def d16(x, pe):
            return torch.from_numpy(np.ascontiguousarray(x)).to(F16).to(pe.torch_device)

        def body(pe):
            x, a, bb = d16(shards[pe.rank], pe), d16(amats[pe.rank], pe), d16(b, pe)
            h = ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, world_size), agb)
            y = gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, world_size), rsb)
            return h, y

        for r, (h, y) in enumerate(run_np(w, body)):
            assert np.array_equal(h, ag_ref)
            assert np.array_equal(y, rs_ref[r])
            gathered = to_np(w.read_tensor(r, agb.gathered, F16, (m, k)))
            assert np.array_equal(gathered, oracle.gathered_layout(shards))
            staging = to_np(w.read_tensor(r, rsb.staging, F16, (world_size, rows, n)))
            assert np.array_equal(staging, oracle.staging_layout(amats, [b] * world_size, r))


def test_fp16_tp_mlp_float_tolerance():
    # random-normal fp16 TP MLP pair against an fp32 reference (north-star
    # tolerance: relative Frobenius error <= 1e-2)
    W, M, H, F = 2, 512, 256, 384
    g = np.random.default_rng(7)
    x_full = g.standard_normal((M, H)).astype(np.float32)
    ub = [(g.standard_normal((H, F // W)) * 0.05).astype(np.float32) for _ in range(W)]
    db = [(g.standard_normal((F // W, H)) * 0.05).astype(np.float32) for _ in range(W)]
    ag_shape = ProblemShape(m=M, n=F // W, k=H, dtype="float16")
    rs_shape = ProblemShape(m=M, n=H, k=F // W, dtype="float16")
    rows = M // W
    with make_world(W, heap_bytes=1 << 24) as w:
        agb, rsb = make_ag_gemm_buffers(w, ag_shape), make_gemm_rs_buffers(w, rs_shape)

        def h16(x, pe):
            return torch.from_numpy(np.ascontiguousarray(x)).to(torch.float16).to(pe.torch_device)

        # stage every input first: a pageable host->device copy issued after a
        # rank's collective could wait behind it while a sibling rank's
        # launch waits behind the copy (World.run docstring)
        staged = w.run(lambda pe: (h16(x_full[pe.rank * rows:(pe.rank + 1) * rows], pe),
                                   h16(ub[pe.rank], pe), h16(db[pe.rank], pe)))

        def body(pe):
            x, up, dn = staged[pe.rank]
            h = ag_gemm(pe, x, up, ag_shape, ag_order_switch(pe.rank, W), agb)
            return gemm_rs(pe, h, dn, rs_shape, rs_inter_order(pe.ctx, 1, W), rsb)

        res = run_np(w, body)
    xr = torch.from_numpy(x_full).half().float().numpy()
    y_full = sum((xr @ torch.from_numpy(ub[r]).half().float().numpy()) @
                 torch.from_numpy(db[r]).half().float().numpy() for r in range(W))
    for r, y in enumerate(res):
        ref = y_full[r * rows:(r + 1) * rows]
        assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 1e-2


@pytest.mark.parametrize("world_size,rows,n,k,late", [
    (1, 2560, 2048, 4096, "18,20"),   # forced weighted partition, clipped late shares
    (1, 2560, 2048, 4096, "40,30"),
    (4, 512, 2048, 1024, None),       # automatic: own chunk has fewer tiles than clusters
    (8, 256, 1024, 2048, None),
])
def test_ag_weighted_stream_k_partition_exact(rng, monkeypatch, world_size, rows, n, k, late):
    # the stream-K share of the clusters that open on a remote chunk shrinks by
    # the expected push time; the fixup owners must follow the same partition
    if late:
        monkeypatch.setenv("SHB_SK_LATE", late)
    monkeypatch.setenv("SHB_SK", "1")
    shape = ProblemShape(m=rows * world_size, n=n, k=k, dtype="bfloat16")
    with make_world(world_size, heap_bytes=1 << 27, timeout_s=20.0) as w:
        bufs = make_ag_gemm_buffers(w, shape)
        # small integers held in float64: the oracle's matmul runs on BLAS
        # (numpy's int64 matmul is a scalar loop) and stays exact
        shards = [ints(rng, -1, 2, (rows, k)).astype(np.float64) for _ in range(world_size)]
        b = ints(rng, -1, 2, (k, n)).astype(np.float64)
        ref = oracle.ag_gemm_reference(shards, b)
        if np.abs(ref).max() >= 256:
            pytest.skip("not exact in bf16 for this draw")

        def body(pe):
            x, bb = dev(shards[pe.rank], pe), dev(b, pe)
            return [ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, world_size), bufs,
                            reset=False) for _ in range(2)]

        for outs in run_np(w, body):
            for out in outs:
                assert np.array_equal(out, ref)


def test_tensor_map_cache_same_addresses_new_shapes(rng):
    # the C ABI caches encoded tensor maps keyed on pointer + layout: calls
    # that reuse one allocation with other dims / strides must not pick up a
    # stale map (shmem_b200.cu make_map)
    shapes = [ProblemShape(m=256, n=192, k=320, dtype="bfloat16"),
              ProblemShape(m=256, n=128, k=192, dtype="bfloat16"),
              ProblemShape(m=384, n=256, k=128, dtype="bfloat16")]
    with make_world(1, heap_bytes=1 << 25) as w:
        agb = [make_ag_gemm_buffers(w, s) for s in shapes]
        rsb = [make_gemm_rs_buffers(w, s) for s in shapes]
        cases = [(i, ints(rng, -2, 3, (s.m, s.k)), ints(rng, -1, 2, (s.k, s.n)))
                 for _ in range(3) for i, s in enumerate(shapes)]

        def body(pe):
            pool_a = torch.empty(1 << 20, dtype=BF16, device=pe.torch_device)
            pool_b = torch.empty(1 << 20, dtype=BF16, device=pe.torch_device)
            outs = []
            for i, a, b in cases:
                s = shapes[i]
                av = pool_a[: s.m * s.k].view(s.m, s.k)
                bv = pool_b[: s.k * s.n].view(s.k, s.n)
                av.copy_(dev(a, pe))
                bv.copy_(dev(b, pe))
                outs.append(ag_gemm(pe, av, bv, s, ag_order_switch(0, 1), agb[i]).clone())
                outs.append(gemm_rs(pe, av, bv, s, rs_inter_order(pe.ctx, 1, 1), rsb[i]).clone())
            return outs

        outs = run_np(w, body)[0]
        for j, (i, a, b) in enumerate(cases):
            assert np.abs(a @ b).max() < 256  # exact in bf16
            assert np.array_equal(outs[2 * j], a @ b), (j, shapes[i])
            assert np.array_equal(outs[2 * j + 1], a @ b), (j, shapes[i])


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")
def test_graph_capture_refused_loudly(rng):
    # epochs are host values baked into each launch, so a CUDA graph replay
    # would race on stale flags: capture must fail, not record a wrong graph
    from paper_2504_19442_b200 import UsageError, gemm

    shape = ProblemShape(m=256, n=128, k=128, dtype="bfloat16")
    with make_world(1) as w:
        agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
        pe = w.pe(0)
        a = dev(ints(rng, -2, 3, (256, 128)), pe)
        b = dev(ints(rng, -1, 2, (128, 128)), pe)
        calls = [lambda: ag_gemm(pe, a, b, shape, ag_order_switch(0, 1), agb, reset=False),
                 lambda: gemm_rs(pe, a, b, shape, rs_inter_order(pe.ctx, 1, 1), rsb,
                                 reset=False),
                 lambda: gemm(a, b)]
        torch.cuda.synchronize()
        for call in calls:
            g = torch.cuda.CUDAGraph()
            with pytest.raises(UsageError, match="graph capture"):
                with torch.cuda.graph(g):
                    call()
        # the library still works after the refused captures
        out = ag_gemm(pe, a, b, shape, ag_order_switch(0, 1), agb)
        assert np.array_equal(to_np(out), to_np(a) @ to_np(b))


@pytest.mark.parametrize("world_size,rows,n,k", [(2, 128, 264, 200), (4, 72, 512, 136),
                                                 (4, 128, 256, 520), (8, 40, 136, 72),
                                                 # long K; a 224-wide tile (2 n-blocks)
                                                 (8, 40, 136, 8264), (4, 128, 520, 8200),
                                                 # 256-row chunks (no pairing): one tile
                                                 # per chunk, stream-K over 74 clusters with
                                                 # the late-starter weighting at its extreme
                                                 (8, 256, 136, 8264)])
@pytest.mark.parametrize("unfused", ["0", "1"])
def test_pair_chunk_tiles_exact(rng, monkeypatch, world_size, rows, n, k, unfused):
    # chunks of <= 128 rows in an even world: a CTA pair takes two chunk
    # positions (AG always; RS when the reduction is a separate pass), incl.
    # ragged rows / n / k; outputs and both layouts bit-exact
    monkeypatch.setenv("SHB_RS_UNFUSED", unfused)
    m = rows * world_size
    shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    with make_world(world_size, heap_bytes=1 << 26) as w:
        agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
        shards = [ints(rng, -2, 3, (rows, k)) for _ in range(world_size)]
        amats = [ints(rng, -1, 2, (m, k)) for _ in range(world_size)]
        b = ints(rng, -1, 2, (k, n))
        if k > 1024:
            # long K: ~64 nonzeros per column keep every sum inside bf16's
            # exact-integer range (|x| <= 256), the oracle being exact
            b *= rng.random((k, n)) < 64.0 / k
        ag_ref = oracle.ag_gemm_reference(shards, b)
        rs_ref = oracle.gemm_rs_reference(amats, [b] * world_size)

        def body(pe):
            x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
            h = ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, world_size), agb, reset=False)
            y = gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, world_size), rsb, reset=False)
            return h, y

        for _ in range(2):  # back to back: epochs advance, no reset
            for r, (h, y) in enumerate(run_np(w, body)):
                assert np.array_equal(h, ag_ref)
                assert np.array_equal(y, rs_ref[r])
        for r in range(world_size):
            staging = to_np(w.read_tensor(r, rsb.staging, BF16, (world_size, rows, n)))
            assert np.array_equal(staging, oracle.staging_layout(amats, [b] * world_size, r))
            gathered = to_np(w.read_tensor(r, agb.gathered, BF16, (m, k)))
            assert np.array_equal(gathered, oracle.gathered_layout(shards))


@pytest.mark.parametrize("exit_release", ["1", "0"])
def test_war_flags_hold_the_epoch_after_each_call(rng, monkeypatch, exit_release):
    # the write-after-read flags: done[p] (AG, "p finished reading its gather
    # buffer") and producer[d] (RS, "d reduced its staging slots") hold the
    # call's epoch on every peer after each call -- stored by the last
    # retiring CTA of the reading kernel (default) or by stream writes after
    # it (SHB_EXIT_RELEASE=0); the products stay bit-exact on every call
    monkeypatch.setenv("SHB_EXIT_RELEASE", exit_release)
    W, rows, n, k = 4, 256, 256, 512
    m = rows * W
    shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
    with make_world(W, heap_bytes=1 << 25) as w:
        agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)
        for epoch in (1, 2, 3):
            shards = [ints(rng, -2, 3, (rows, k)) for _ in range(W)]
            amats = [ints(rng, -1, 2, (m, k)) for _ in range(W)]
            b = ints(rng, -1, 2, (k, n))

            def body(pe):
                x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
                h = ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, W), agb, reset=False)
                y = gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, W), rsb, reset=False)
                return h, y

            outs = run_np(w, body)
            rs_ref = oracle.gemm_rs_reference(amats, [b] * W)
            for r, (h, y) in enumerate(outs):
                assert np.array_equal(h, oracle.ag_gemm_reference(shards, b))
                assert np.array_equal(y, rs_ref[r])
            for r in range(W):
                for p in range(W):
                    if p != r:
                        assert w.sig_read(r, agb.done.base + p) == epoch
                        assert w.sig_read(r, rsb.producer.base + p) == epoch
