"""Where the MMA warp waits: per work item, the wait for a free accumulator
and the summed operand-stage waits (trace kind 5), for the C3 ag_gemm and C4
gemm_rs calls at W=1 (diagnostic for the ~8 % tensor-idle inside active cycles)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb

AG = dict(m=8192, n=3584, k=8192); RS = dict(m=8192, n=8192, k=3584)
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags = sb.ProblemShape(dtype="bfloat16", **AG); rss = sb.ProblemShape(dtype="bfloat16", **RS)
agb = sb.make_ag_gemm_buffers(w, ags); rsb = sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
with torch.cuda.stream(pe.stream()):
    for _ in range(5):
        h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
        sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
    torch.cuda.synchronize()
    w.start_trace(records_per_cta=256, launches=4)
    for _ in range(2):
        h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
        sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
    torch.cuda.synchronize()
    ev = w.stop_trace()
for kern in ("ag_gemm", "gemm_rs"):
    items = [e for e in ev if e["kernel"] == kern and e["op"] == "mma_item"]
    launch = max(e["launch"] for e in items)
    items = [e for e in items if e["launch"] == launch]
    ctas = [e for e in ev if e["kernel"] == kern and e["op"] == "cta" and e["launch"] == launch]
    span = (max(e["t1_ns"] for e in ctas) - min(e["t0_ns"] for e in ctas)) / 1e3
    by = {}
    for e in items:
        by.setdefault(e["cta"], []).append(e)
    acc_w, stg_w, per, first = [], [], [], []
    for cta, es in by.items():
        es.sort(key=lambda e: e["t0_ns"])
        for i, e in enumerate(es):
            acc_w.append((e["t1_ns"] - e["t0_ns"]) / 1e3)
            stg_w.append(e["stage_wait_ns"] / 1e3)
            if i + 1 < len(es):
                per.append((es[i + 1]["t0_ns"] - e["t0_ns"]) / 1e3)
        first.append((es[0]["t0_ns"] - min(c["t0_ns"] for c in ctas)) / 1e3)
    cta_end = [ (max(e["t1_ns"] for e in ctas if e["cta"] == c) - min(c2["t0_ns"] for c2 in ctas)) / 1e3 for c in by]
    n = len(by)
    print(f"== {kern}: launch span {span:.1f} us, {n} MMA CTAs, {len(items)} items")
    print(f"   accumulator wait per item: mean {statistics.mean(acc_w):.2f} us  max {max(acc_w):.2f}")
    print(f"   stage waits per item     : mean {statistics.mean(stg_w):.2f} us  max {max(stg_w):.2f}  "
          f"(sum over items / CTA: {sum(stg_w)/n:.1f} us)")
    print(f"   item period              : median {statistics.median(per):.2f} us  mean {statistics.mean(per):.2f}")
    print(f"   first item start after CTA0 start: mean {statistics.mean(first):.2f} us max {max(first):.2f}")
    print(f"   CTA end times: min {min(cta_end):.1f} median {statistics.median(cta_end):.1f} max {max(cta_end):.1f} us")
for kern in ("ag_gemm", "gemm_rs"):
    ep = [e for e in ev if e["kernel"] == kern and e["op"] == "tile_epilogue"]
    launch = max(e["launch"] for e in ep)
    d = [(e["t1_ns"] - e["t0_ns"]) / 1e3 for e in ep if e["launch"] == launch]
    print(f"== {kern}: epilogue (accumulator ready -> stores issued, warp 2): "
          f"median {statistics.median(d):.2f} us  mean {statistics.mean(d):.2f}  max {max(d):.2f}")
