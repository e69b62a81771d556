"""Timeline emitter (§8 f2): device stamps of the fused kernels -> events ->
Chrome trace + exposed-communication summary."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_19442_b200 import (ProblemShape, WorldSpec, ag_gemm, ag_order_switch,  # noqa: E402
                                   gemm_rs, init_world, make_ag_gemm_buffers,
                                   make_gemm_rs_buffers, rs_inter_order)
from paper_2504_19442_b200 import schemas  # noqa: E402
from paper_2504_19442_b200.timeline import exposed_comm, to_chrome_trace  # noqa: E402

pytestmark = pytest.mark.gpu


def test_trace_of_a_tp_mlp_step(tmp_path):
    W = 4
    ag_shape = ProblemShape(m=1024, n=512, k=256, dtype="bfloat16")
    rs_shape = ProblemShape(m=1024, n=256, k=512, dtype="bfloat16")
    with init_world(WorldSpec(world_size=W, heap_bytes=1 << 24, timeout_s=10)) as w:
        agb, rsb = make_ag_gemm_buffers(w, ag_shape), make_gemm_rs_buffers(w, rs_shape)
        staged = w.run(lambda pe: (torch.randn(256, 256, device=pe.torch_device).bfloat16(),
                                   torch.randn(256, 512, device=pe.torch_device).bfloat16(),
                                   torch.randn(512, 256, device=pe.torch_device).bfloat16()))
        w.start_trace(records_per_cta=64, launches=4)

        def body(pe):
            x, up, dn = staged[pe.rank]
            h = ag_gemm(pe, x, up, ag_shape, ag_order_switch(pe.rank, W), agb)
            return gemm_rs(pe, h, dn, rs_shape, rs_inter_order(pe.ctx, 1, W), rsb)

        w.run(body)
        events = w.stop_trace()
    kinds = {e["op"] for e in events}
    assert {"cta", "tile_epilogue", "chunk_wait"} <= kinds
    for r in range(W):
        mine = [e for e in events if e["rank"] == r]
        # the RS's separate reduction kernel is a launch of its own
        assert {e["kernel"] for e in mine} == {"ag_gemm", "gemm_rs", "rs_reduce"}
        assert any(e["op"] == "peer_wait" for e in mine if e["kernel"] == "rs_reduce")
        # a chunk wait is only ever recorded for a remote chunk
        assert all(e["chunk"] != r for e in mine if e["op"] == "chunk_wait")
        for e in mine:
            assert e["t1_ns"] >= e["t0_ns"] > 0
    doc = to_chrome_trace(events)
    json.dumps(doc)
    assert doc and all(ev["ph"] == "X" for ev in doc)
    schemas.validate(doc, "trace", "trace")  # the reference's trace contract
    summary = exposed_comm(events)
    assert len(summary) == 3 * W and all(s["span_us"] > 0 for s in summary)
