"""Sustained throughput + clocks/power of our GEMM vs cuBLAS (2 s each)."""
import os, subprocess, sys, time, threading, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb
from paper_2504_19442_b200 import _lib
import torch

def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line: out.append([float(x) for x in line.split(",")])
    p.terminate()

def run(fn, secs=2.0):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    out, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, out)); th.start()
    time.sleep(0.2)
    n = 0; t0 = time.time()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < secs:
        for _ in range(20): fn()
        n += 20
        torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = s.elapsed_time(e) / n
    clk = statistics.median([o[0] for o in out[2:]]) if len(out) > 3 else None
    pw = statistics.median([o[1] for o in out[2:]]) if len(out) > 3 else None
    return ms, clk, pw

for (m, n, k) in [(8192, 3584, 8192), (8192, 8192, 3584), (8192, 8192, 8192)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(k, n, device="cuda").bfloat16()
    fl = 2 * m * n * k
    for name, fn in [("cublas", lambda: torch.matmul(a, b)), ("ours", lambda: sb.gemm(a, b)), ("cublas", lambda: torch.matmul(a, b)), ("ours", lambda: sb.gemm(a, b))]:
        ms, clk, pw = run(fn)
        print(f"{m}x{n}x{k} {name:7s} {fl / ms / 1e9:7.1f} TF  sm {clk} MHz  {pw} W", flush=True)
