"""Interleaved A/B of env-knob variants on C5 sweep points (W=1), with cuBLAS.

    python scripts/ab_sweep.py "gemm_rs:16384,gemm_rs:1024" "-" "SHB_GROUP_M=2" "SHB_SK=0"

Each round runs every variant (and torch.matmul) once per point; medians over
rounds are printed, so thermal/power drift hits all variants alike."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

FFN, HID = 28672, 8192
ROUNDS = int(os.environ.get("AB_ROUNDS", "5"))


def main():
    points = [p.split(":") for p in sys.argv[1].split(",")]
    variants = sys.argv[2:] or ["-"]
    keys = {kv.split("=")[0] for v in variants if v != "-" for kv in v.split(",")}
    heap = sum(int(pt[1]) * HID * 4 + (1 << 20) for pt in points)
    w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=heap, timeout_s=60))
    pe = w.pe(0)
    stream = pe.stream()
    sched_ag, sched_rs = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
    runs = []
    for pt in points:
        op, M = pt[0], int(pt[1])
        if len(pt) == 4:  # op:M:n:k
            s = dict(m=M, n=int(pt[2]), k=int(pt[3]))
        elif op == "ag_gemm":
            s = dict(m=M, n=FFN, k=HID)
        else:
            s = dict(m=M, n=HID, k=FFN)
        if op == "ag_gemm":
            shape = sb.ProblemShape(dtype="bfloat16", **s)
            bufs = sb.make_ag_gemm_buffers(w, shape)
            a = torch.randn(M, s["k"], device="cuda").bfloat16()
            b = (torch.randn(s["k"], s["n"], device="cuda") * .02).bfloat16()
            ours = (lambda a=a, b=b, shape=shape, bufs=bufs:
                    sb.ag_gemm(pe, a, b, shape, sched_ag, bufs, reset=False))
        else:
            shape = sb.ProblemShape(dtype="bfloat16", **s)
            bufs = sb.make_gemm_rs_buffers(w, shape)
            a = torch.randn(M, s["k"], device="cuda").bfloat16()
            b = (torch.randn(s["k"], s["n"], device="cuda") * .02).bfloat16()
            ours = (lambda a=a, b=b, shape=shape, bufs=bufs:
                    sb.gemm_rs(pe, a, b, shape, sched_rs, bufs, reset=False))
        fl = 2.0 * s["m"] * s["n"] * s["k"]
        iters = int(max(5, min(30, 0.08 / (fl / 1.2e15))))
        runs.append((":".join(pt), fl, iters, ours, lambda a=a, b=b: torch.matmul(a, b)))

    def setenv(v):
        for k in keys:
            os.environ.pop(k, None)
        if v != "-":
            for kv in v.split(","):
                k, val = kv.split("=")
                os.environ[k] = val

    def timed(fn, iters):
        with torch.cuda.stream(stream):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    res = {}
    for _ in range(ROUNDS):
        for name, fl, iters, ours, torch_fn in runs:
            for v in variants:
                setenv(v)
                res.setdefault((name, v), []).append(timed(ours, iters))
            setenv("-")
            res.setdefault((name, "cublas"), []).append(timed(torch_fn, iters))
    for name, fl, iters, _, _ in runs:
        for v in variants + ["cublas"]:
            ts = res[(name, v)]
            med = statistics.median(ts)
            print(f"{name:14s} {v:28s} median {med*1e3:8.1f} us {fl/med/1e9:7.1f} TF  "
                  f"min {min(ts)*1e3:8.1f}  max {max(ts)*1e3:8.1f}", flush=True)
    w.close()


if __name__ == "__main__":
    main()
