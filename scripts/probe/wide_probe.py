"""C3 ag_gemm / C4 gemm_rs at W=1 under a forced tile config (env WIDE_BN,
WIDE_CG; 0,0 = automatic), a few calls each (ncu target), then the MMA
warp's accumulator / operand waits from one traced call (kind 5)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb
from paper_2504_19442_b200 import _lib

bn, cg = int(os.environ.get("WIDE_BN", "0")), int(os.environ.get("WIDE_CG", "0"))
lib = _lib.load()
_lib.check(lib.sh_set_tile_config(bn, cg))
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
pe = w.pe(0)
ags = sb.ProblemShape(m=8192, n=3584, k=8192, dtype="bfloat16")
rss = sb.ProblemShape(m=8192, n=8192, k=3584, dtype="bfloat16")
agb, rsb = sb.make_ag_gemm_buffers(w, ags), sb.make_gemm_rs_buffers(w, rss)
x = torch.randn(8192, 8192, device="cuda").bfloat16()
wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
with torch.cuda.stream(pe.stream()):
    for _ in range(3):
        h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
        sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
    torch.cuda.synchronize()
    if os.environ.get("WIDE_TRACE", "1") == "1":
        w.start_trace(records_per_cta=256, launches=4)
        h = sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)
        sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)
        torch.cuda.synchronize()
        ev = w.stop_trace()
        out = {}
        for kern in ("ag_gemm", "gemm_rs"):
            items = [e for e in ev if e["kernel"] == kern and e["op"] == "mma_item"]
            ctas = [e for e in ev if e["kernel"] == kern and e["op"] == "cta"]
            span = (max(e["t1_ns"] for e in ctas) - min(e["t0_ns"] for e in ctas)) / 1e3
            by = {}
            for e in items:
                by.setdefault(e["cta"], []).append(e)
            acc = [sum(e["t1_ns"] - e["t0_ns"] for e in es) / 1e3 for es in by.values()]
            stg = [sum(e["stage_wait_ns"] for e in es) / 1e3 for es in by.values()]
            out[kern] = {"span_us": span, "items_per_cta": statistics.mean(len(es) for es in by.values()),
                         "acc_wait_us_per_cta": statistics.mean(acc),
                         "stage_wait_us_per_cta": statistics.mean(stg)}
        print(json.dumps({"bn": bn, "cg": cg, **out}))
w.close()
