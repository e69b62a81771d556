"""Back-to-back A/B of the raster group (SHB_GROUP_M) at the C5 TP=1 M=16384
points: ag_gemm (16384, 28672, 8192) and gemm_rs (16384, 8192, 28672),
configs interleaved round by round, median per config of per-round medians.
Usage: python scripts/probe/c5_group_ab.py [rounds] [calls] [groups,...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 10
groups = sys.argv[3].split(",") if len(sys.argv) > 3 else ["auto", "4", "12", "16"]
M = 16384
ag_s = sb.ProblemShape(m=M, n=28672, k=8192, dtype="bfloat16")
rs_s = sb.ProblemShape(m=M, n=8192, k=28672, dtype="bfloat16")
w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=(M * 8192 * 2 + M * 8192 * 2 + (64 << 20)),
                               timeout_s=60))
pe = w.pe(0)
agb, rsb = sb.make_ag_gemm_buffers(w, ag_s), sb.make_gemm_rs_buffers(w, rs_s)
x = torch.randn(M, 8192, device="cuda").bfloat16()
up = (torch.randn(8192, 28672, device="cuda") * .02).bfloat16()
h = torch.randn(M, 28672, device="cuda").bfloat16()
dn = (torch.randn(28672, 8192, device="cuda") * .02).bfloat16()
c = torch.empty(M, 28672, device="cuda", dtype=torch.bfloat16)
y = torch.empty(M, 8192, device="cuda", dtype=torch.bfloat16)
sched = sb.ag_order_switch(0, 1)
ops = {"ag": lambda: sb.ag_gemm(pe, x, up, ag_s, sched, agb, reset=False, out=c),
       "rs": lambda: sb.gemm_rs(pe, h, dn, rs_s, sb.rs_inter_order(pe.ctx, 1, 1), rsb,
                                reset=False, out=y)}
res = {}


def body(_pe):
    for r in range(rounds):
        for op, fn in ops.items():
            for g in groups:
                if g == "auto":
                    os.environ.pop("SHB_GROUP_M", None)
                else:
                    os.environ["SHB_GROUP_M"] = g
                fn()
                torch.cuda.synchronize()
                evs = []
                for _ in range(calls):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn()
                    b.record()
                    evs.append((a, b))
                torch.cuda.synchronize()
                # the second half only: the power controller settles in the first
                res.setdefault(f"{op}/g{g}", []).append(
                    round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in evs[calls // 2:]), 1))
    os.environ.pop("SHB_GROUP_M", None)


w.run(body)
w.close()
print(json.dumps({k: {"median_us": statistics.median(v), "rounds": v} for k, v in res.items()}))
