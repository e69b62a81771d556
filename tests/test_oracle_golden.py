"""Pin the CPU oracle and the host-side schedules against fixtures produced by
running the reference itself (tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from oracle import minishmem_oracle as oracle
from paper_2504_19442_b200 import RankCtx, ag_order_fullmesh, ag_order_switch, rs_inter_order
from paper_2504_19442_b200.swizzle import ag_push_order

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
AG_CASES = ["ag_w2_int", "ag_w4_int", "ag_w8_int", "ag_w2_f32"]
RS_CASES = ["rs_w2_int", "rs_w4_int", "rs_w8_int", "rs_w4_f32"]


def load(name):
    return dict(np.load(os.path.join(GOLD, f"{name}.npz")))


def schedules():
    with open(os.path.join(GOLD, "schedules.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", AG_CASES)
def test_oracle_ag_gemm_matches_reference(name):
    g = load(name)
    shards = list(g["shards"])
    w = len(shards)
    for r in range(w):
        out = oracle.ag_gemm_reference(shards, g["b"][r])
        if out.dtype.kind == "i":
            assert np.array_equal(out, g["out"][r])
        else:
            np.testing.assert_allclose(out, g["out"][r], rtol=1e-5, atol=1e-4)
        assert np.array_equal(oracle.gathered_layout(shards), g["gathered"][r])


@pytest.mark.parametrize("name", AG_CASES)
def test_oracle_port_ag_gemm_matches_reference(name):
    g = load(name)
    shards = list(g["shards"])
    w = len(shards)
    orders = [oracle.ag_order_switch(r, w) for r in range(w)]
    outs, gathered = oracle.port_ag_gemm(shards, list(g["b"]), orders, tile_m=16, tile_n=32)
    for r in range(w):
        # identical tile products and order as the reference -> bit-identical
        assert np.array_equal(outs[r], g["out"][r])
        assert np.array_equal(gathered[r], g["gathered"][r])


@pytest.mark.parametrize("name", RS_CASES)
def test_oracle_gemm_rs_matches_reference(name):
    g = load(name)
    amats, bs = list(g["a"]), list(g["b"])
    w = len(amats)
    outs = oracle.gemm_rs_reference(amats, bs)
    for r in range(w):
        if g["out"].dtype.kind == "i":
            assert np.array_equal(outs[r], g["out"][r])
            assert np.array_equal(oracle.staging_layout(amats, bs, r), g["staging"][r])
        else:
            np.testing.assert_allclose(outs[r], g["out"][r], rtol=1e-5, atol=1e-4)
            np.testing.assert_allclose(oracle.staging_layout(amats, bs, r), g["staging"][r],
                                       rtol=1e-6, atol=1e-5)


@pytest.mark.parametrize("name", RS_CASES)
def test_oracle_port_gemm_rs_matches_reference(name):
    g = load(name)
    amats, bs = list(g["a"]), list(g["b"])
    w = len(amats)
    orders = [oracle.rs_inter_order(r, 0, r, 1, w) for r in range(w)]
    outs, staging = oracle.port_gemm_rs(amats, bs, orders)
    for r in range(w):
        # same per-chunk products, same ascending-source reduction -> bit-identical
        assert np.array_equal(outs[r], g["out"][r])
        assert np.array_equal(staging[r], g["staging"][r])


def test_schedules_match_reference():
    s = schedules()
    for w, per_rank in s["ag_order_switch"].items():
        w = int(w)
        for r in range(w):
            assert ag_order_switch(r, w).chunk_order() == per_rank[r]
            assert oracle.ag_order_switch(r, w) == per_rank[r]
    for w, per_rank in s["rs_inter_order_1node"].items():
        w = int(w)
        for r in range(w):
            assert rs_inter_order(RankCtx(r, 0, r), 1, w).chunk_order() == per_rank[r]
            assert oracle.rs_inter_order(r, 0, r, 1, w) == per_rank[r]
    for w, per_rank in s["rs_inter_order_2node"].items():
        w = int(w)
        lws = w // 2
        for r in range(w):
            ctx = RankCtx(r, r // lws, r % lws)
            assert rs_inter_order(ctx, 2, lws).chunk_order() == per_rank[r]
    for w, per_rank in s["ag_order_fullmesh"].items():
        w = int(w)
        for r in range(w):
            steps = [[st.chunk, st.subchunk] for st in ag_order_fullmesh(r, w, 3).steps]
            assert steps == per_rank[r]


def test_golden_anchors():
    # the reference's own known answers (tests/test_swizzle.py:11-12, :79-81)
    s = schedules()
    assert s["ag_order_switch"]["4"][1] == [1, 2, 3, 0]
    assert s["rs_inter_order_2node"]["8"][0] == [5, 6, 7, 4, 1, 2, 3, 0]
    assert s["rs_inter_order_2node"]["8"][1][0] == 6
    assert s["rs_inter_order_1node"]["4"] == [[1, 2, 3, 0], [2, 3, 0, 1], [3, 0, 1, 2],
                                              [0, 1, 2, 3]]


def test_push_order_serves_ring_consumers_first():
    # under ag_order_switch, peer p consumes chunk `rank` at step (rank - p) mod W;
    # the host pushes in increasing step order
    for w in (2, 3, 4, 8):
        for r in range(w):
            push = ag_push_order(r, w)
            steps = [ag_order_switch(p, w).chunk_order().index(r) for p in push]
            assert steps == sorted(steps) and sorted(push) == sorted(set(range(w)) - {r})
