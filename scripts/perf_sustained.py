"""Sustained (power-capped) throughput, SM clock and board power of the fused
W=1 ops against the plain GEMM core and cuBLAS on the C3/C4 shapes.

    python scripts/perf_sustained.py [secs] [rounds]

Variants run interleaved (round-robin) so thermal drift hits all of them.
Prints one line per variant: median TFLOPS, median SM MHz under load, median
power, TFLOPS per GHz (per-clock efficiency)."""
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2504_19442_b200 as sb  # noqa: E402

SECS = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
ROUNDS = int(sys.argv[2]) if len(sys.argv) > 2 else 2


def sampler(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "50"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            try:
                out.append([float(x) for x in line.split(",")])
            except ValueError:
                pass
    p.terminate()


def run(fn, stream, secs):
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        out, stop = [], threading.Event()
        th = threading.Thread(target=sampler, args=(stop, out))
        th.start()
        time.sleep(0.15)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        t0 = time.time()
        s.record(stream)
        while time.time() - t0 < secs:
            for _ in range(10):
                fn()
            n += 10
            torch.cuda.synchronize()
        e.record(stream)
        torch.cuda.synchronize()
        stop.set()
        th.join()
    ms = s.elapsed_time(e) / n
    tail = out[len(out) // 4:] or out
    clk = statistics.median(o[0] for o in tail) if tail else float("nan")
    pw = statistics.median(o[1] for o in tail) if tail else float("nan")
    return ms, clk, pw


def main():
    AG = dict(m=8192, n=3584, k=8192)
    RS = dict(m=8192, n=8192, k=3584)
    w = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=600 << 20, timeout_s=60))
    pe = w.pe(0)
    ags = sb.ProblemShape(dtype="bfloat16", **AG)
    rss = sb.ProblemShape(dtype="bfloat16", **RS)
    agb = sb.make_ag_gemm_buffers(w, ags)
    rsb = sb.make_gemm_rs_buffers(w, rss)
    x = torch.randn(8192, 8192, device="cuda").bfloat16()
    wu = (torch.randn(8192, 3584, device="cuda") * .02).bfloat16()
    h = torch.randn(8192, 3584, device="cuda").bfloat16()
    wd = (torch.randn(3584, 8192, device="cuda") * .02).bfloat16()
    sa, sr = sb.ag_order_switch(0, 1), sb.rs_inter_order(w.ranks[0], 1, 1)
    stream = pe.stream()
    envs = ["SHB_OWN_COPY_CE", "SHB_RS_UNFUSED"]

    def with_env(fn, **kv):
        def g():
            for k in envs:
                os.environ.pop(k, None)
            os.environ.update({k: str(v) for k, v in kv.items()})
            fn()
        return g

    variants = {
        "C3 cublas": (lambda: torch.matmul(x, wu), AG),
        "C3 sh_gemm": (lambda: sb.gemm(x, wu), AG),
        "C3 ag_gemm": (with_env(lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False)), AG),
        "C3 ag_gemm own-by-CE": (with_env(lambda: sb.ag_gemm(pe, x, wu, ags, sa, agb, reset=False),
                                          SHB_OWN_COPY_CE=1), AG),
        "C4 cublas": (lambda: torch.matmul(h, wd), RS),
        "C4 sh_gemm": (lambda: sb.gemm(h, wd), RS),
        "C4 gemm_rs": (with_env(lambda: sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False)), RS),
        "C4 gemm_rs unfused-reduce": (with_env(lambda: sb.gemm_rs(pe, h, wd, rss, sr, rsb, reset=False),
                                               SHB_RS_UNFUSED=1), RS),
    }
    if len(sys.argv) > 3:
        keep = sys.argv[3].split(",")
        variants = {k: v for k, v in variants.items() if any(s in k for s in keep)}
    res = {k: [] for k in variants}
    for _ in range(ROUNDS):
        for name, (fn, shp) in variants.items():
            res[name].append(run(fn, stream, SECS))
    for name, rs in res.items():
        shp = variants[name][1]
        fl = 2.0 * shp["m"] * shp["n"] * shp["k"]
        ms = statistics.median(r[0] for r in rs)
        clk = statistics.median(r[1] for r in rs)
        pw = statistics.median(r[2] for r in rs)
        tf = fl / ms / 1e9
        print(f"{name:28s} {ms*1e3:7.1f} us {tf:7.1f} TF  sm {clk:6.0f} MHz  {pw:6.0f} W  "
              f"{tf / (clk / 1000):6.1f} TF/GHz", flush=True)


if __name__ == "__main__":
    main()
