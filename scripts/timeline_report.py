"""Exposed-communication report from the device timeline (§8 f2).

    python scripts/timeline_report.py [W] [out.json]

Runs the TP MLP pair (ag_gemm on the C3 per-rank width, gemm_rs on the C4
per-rank depth, rows = 1024 per rank as at TP=8) with W ranks.  On a one-GPU
box all ranks share cuda:0 (each gets 1/W of the SMs and the "NVLink" pushes
are copy-engine copies inside one HBM), so the numbers describe the pipeline
(how long CTAs sat on chunk flags / peer counters), not NVLink.  Writes the
per-launch exposed_comm summary and the first launches' Chrome trace."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402
from paper_2504_19442_b200.timeline import exposed_comm, to_chrome_trace  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/timeline_w{W}.json"
    rows = 1024
    ag_shape = sb.ProblemShape(m=rows * W, n=3584, k=8192, dtype="bfloat16")
    rs_shape = sb.ProblemShape(m=rows * W, n=8192, k=3584, dtype="bfloat16")
    heap = rows * W * (8192 + 8192) * 2 + (16 << 20)
    with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=heap, timeout_s=30)) as w:
        agb, rsb = sb.make_ag_gemm_buffers(w, ag_shape), sb.make_gemm_rs_buffers(w, rs_shape)
        staged = w.run(lambda pe: (
            torch.randn(rows, 8192, device=pe.torch_device).bfloat16(),
            (torch.randn(8192, 3584, device=pe.torch_device) * .02).bfloat16(),
            (torch.randn(3584, 8192, device=pe.torch_device) * .02).bfloat16()))

        def body(pe):
            x, up, dn = staged[pe.rank]
            for _ in range(3):
                h = sb.ag_gemm(pe, x, up, ag_shape, sb.ag_order_switch(pe.rank, W), agb,
                               reset=False)
                sb.gemm_rs(pe, h, dn, rs_shape, sb.rs_inter_order(pe.ctx, 1, W), rsb,
                           reset=False)

        w.run(body)  # warm-up
        w.start_trace(records_per_cta=128, launches=6)
        w.run(body)
        events = w.stop_trace()
    summary = exposed_comm(events)
    for s in summary:
        s["exposed_frac_max"] = s["wait_max_us"] / s["span_us"] if s["span_us"] else None
        s["exposed_frac_mean"] = s["wait_mean_us"] / s["span_us"] if s["span_us"] else None
    first = [e for e in events if e["launch"] < 2]
    doc = {"what": ("TP MLP pair, rows=1024 per rank, W ranks sharing one B200 (copy-engine "
                    "pushes inside one HBM stand in for NVLink); waits = CTA time on AG chunk "
                    "flags (chunk_wait) / fused-RS peer counters (peer_wait)"),
           "world_size": W, "ag_shape": [ag_shape.m, ag_shape.n, ag_shape.k],
           "rs_shape": [rs_shape.m, rs_shape.n, rs_shape.k], "exposed_comm": summary,
           "chrome_trace_first_launches": to_chrome_trace(first)}
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump(doc, f)
    for s in summary:
        print(f"rank {s['rank']} {s['kernel']:8s} launch {s['launch']}: span {s['span_us']:8.1f} us  "
              f"wait max {s['wait_max_us']:7.1f} us ({100 * s['exposed_frac_max']:.1f} %)  "
              f"mean {s['wait_mean_us']:7.1f} us")


if __name__ == "__main__":
    main()
