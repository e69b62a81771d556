"""Seeded fuzz of both fused ops over worlds, ragged shapes and tile
configurations (pair / single-CTA tiles, stream-K on/off), bit-exact against
the oracle with integer data, layouts included."""

import contextlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import minishmem_oracle as oracle  # noqa: E402
from paper_2504_19442_b200 import (ProblemShape, WorldSpec, ag_gemm,  # noqa: E402
                                   ag_order_switch, gemm_rs, init_world,
                                   make_ag_gemm_buffers, make_gemm_rs_buffers, rs_inter_order)
from paper_2504_19442_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu
BF16 = torch.bfloat16


def cases(n_cases=None, seed=None):
    # a longer soak: SHB_FUZZ_CASES=200 SHB_FUZZ_SEED=7 pytest tests/test_gpu_fuzz.py
    import os

    n_cases = n_cases or int(os.environ.get("SHB_FUZZ_CASES", "12"))
    seed = seed if seed is not None else int(os.environ.get("SHB_FUZZ_SEED", "2024"))
    g = np.random.default_rng(seed)
    for i in range(n_cases):
        W = int(g.choice([1, 2, 3, 4, 8]))
        rows = int(g.integers(8, 90)) * 8
        n = int(g.integers(8, 100)) * 8
        k = int(g.integers(8, 100)) * 8
        cg = int(g.choice([0, 1, 2]))
        sk = int(g.choice([-1, 0, 1]))
        yield pytest.param(W, rows, n, k, cg, sk, i, id=f"W{W}-r{rows}-n{n}-k{k}-cg{cg}-sk{sk}")


@pytest.mark.parametrize("W,rows,n,k,cg,sk,seed", list(cases()))
def test_fused_ops_fuzz(W, rows, n, k, cg, sk, seed):
    lib = _lib.load()
    _lib.check(lib.sh_set_tile_config(0, cg))
    _lib.check(lib.sh_set_schedule_config(sk, 0))
    try:
        g = np.random.default_rng(seed)
        m = rows * W
        shape = ProblemShape(m=m, n=n, k=k, dtype="bfloat16")
        # integer values held in float64 (BLAS oracle, exact)
        shards = [g.integers(-2, 3, (rows, k)).astype(np.float64) for _ in range(W)]
        amats = [g.integers(-1, 2, (m, k)).astype(np.float64) for _ in range(W)]
        b = g.integers(-1, 2, (k, n)).astype(np.float64)
        ag_ref = oracle.ag_gemm_reference(shards, b)
        rs_ref = oracle.gemm_rs_reference(amats, [b] * W)
        if np.abs(ag_ref).max() >= 256 or max(np.abs(r).max() for r in rs_ref) >= 256:
            pytest.skip("products not exact in bf16 for this draw")
        with contextlib.closing(init_world(WorldSpec(world_size=W, heap_bytes=1 << 26,
                                                     timeout_s=20.0))) as w:
            agb, rsb = make_ag_gemm_buffers(w, shape), make_gemm_rs_buffers(w, shape)

            def dev(x, pe):
                return torch.from_numpy(np.ascontiguousarray(x)).to(BF16).to(pe.torch_device)

            def body(pe):
                x, a, bb = dev(shards[pe.rank], pe), dev(amats[pe.rank], pe), dev(b, pe)
                outs = []
                for _ in range(2):  # back to back, epochs
                    h = ag_gemm(pe, x, bb, shape, ag_order_switch(pe.rank, W), agb, reset=False)
                    y = gemm_rs(pe, a, bb, shape, rs_inter_order(pe.ctx, 1, W), rsb, reset=False)
                    outs.append((h, y))
                return outs

            res = w.run(body)
            for r in range(W):
                for h, y in res[r]:
                    assert np.array_equal(h.float().cpu().numpy(), ag_ref)
                    assert np.array_equal(y.float().cpu().numpy(), rs_ref[r])
                gathered = w.read_tensor(r, agb.gathered, BF16, (m, k)).float().cpu().numpy()
                assert np.array_equal(gathered, oracle.gathered_layout(shards))
                staging = w.read_tensor(r, rsb.staging, BF16, (W, rows, n)).float().cpu().numpy()
                assert np.array_equal(staging, oracle.staging_layout(amats, [b] * W, r))
    finally:
        lib.sh_set_tile_config(0, 0)
        lib.sh_set_schedule_config(-2, -1)
