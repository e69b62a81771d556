"""Where a small TP=8 call's time goes (proxy, preset flags): event time of an
empty gated segment, of each op under library knobs, and the kernel span from
the device timeline.  Usage: PROXY_M=1024 python scripts/probe/call_overhead.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tp_proxy  # noqa: E402

W = int(os.environ.get("PROXY_W", "8"))
M = int(os.environ.get("PROXY_M", "1024"))
px = tp_proxy.TpProxy(W, M, 28672 // W, 8192, 8192, 28672 // W)
out = {}
knobs = {"base": {}, "sys_release": {"SHB_EXIT_SYS_RELEASE": "1"},
         "memops": {"SHB_EXIT_RELEASE": "0"},
         "flag_kernel": {"SHB_EXIT_RELEASE": "0", "SHB_FLAG_KERNEL": "1"},
         "no_flags": {"SHB_DIAG_NOFLAGS": "1"}, "all_gpu": {"SHB_DIAG_RS_GPU_SCOPE": "1"}}
try:
    evs = []
    for _ in range(30):
        a, b = px._call("preset", [], None)
        evs.append((a, b))
    px.main.synchronize()
    out["empty_us"] = statistics.median(a.elapsed_time(b) * 1e3 for a, b in evs[5:])
    for rnd in range(3):
        for name, env in knobs.items():
            for k_, v in env.items():
                os.environ[k_] = v
            for op in ("ag", "rs"):
                print(rnd, name, op, file=sys.stderr, flush=True)
                t = statistics.median(px.time_op(op, "preset", 20))
                out.setdefault(f"{op}/{name}", []).append(round(t, 1))
            for k_ in env:
                os.environ.pop(k_)
    for tname, tenv in (("base", {}), ("all_gpu", {"SHB_DIAG_RS_GPU_SCOPE": "1"})):
        os.environ.update(tenv)
        for op in ("ag", "rs"):
            px.time_op(op, "preset", 3)
            px.world.start_trace(records_per_cta=1024, launches=2)
            px.time_op(op, "preset", 1, warmup=0)
            ev = px.world.stop_trace()
            kern = "ag_gemm" if op == "ag" else "gemm_rs"
            last = max(e["launch"] for e in ev if e["kernel"] == kern)
            g = [e for e in ev if e["launch"] == last and e["op"] == "cta"]
            red = [e for e in ev if e["kernel"] == "rs_reduce" and e["launch"] > last and e["op"] == "cta"]
            span = (max(e["t1_ns"] for e in g) - min(e["t0_ns"] for e in g)) / 1e3
            out[f"{tname}/{op}/gemm_span_us"] = span
            if red:
                out[f"{tname}/{op}/reduce_span_us"] = (max(e["t1_ns"] for e in red) - min(e["t0_ns"] for e in red)) / 1e3
                out[f"{tname}/{op}/gemm_end_to_reduce_end_us"] = (max(e["t1_ns"] for e in red) - max(e["t1_ns"] for e in g)) / 1e3
                out[f"{tname}/{op}/reduce_start_after_gemm_end_us"] = (min(e["t0_ns"] for e in red) - max(e["t1_ns"] for e in g)) / 1e3
                ends = sorted(e["t1_ns"] for e in g)
                out[f"{tname}/{op}/gemm_cta_end_spread_us"] = (ends[-1] - ends[0]) / 1e3

        for k_ in tenv:
            os.environ.pop(k_)
finally:
    px.close()
print(json.dumps(out))
