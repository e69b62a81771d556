"""Interleaved A/B timing of environment-selected kernel variants (median of rounds).
usage: perf_ab.py M N K VAR=val[,VAR=val] VAR=val ...   ('-' = no env change)"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19442_b200 as sb
import torch

m, n, k = (int(x) for x in sys.argv[1:4])
variants = sys.argv[4:] or ["-"]
a = torch.randn(m, k, device="cuda").bfloat16()
b = torch.randn(k, n, device="cuda").bfloat16()
fl = 2 * m * n * k

def setenv(v):
    for key in [x.split("=")[0] for vv in variants if vv != "-" for x in vv.split(",")]:
        os.environ.pop(key, None)
    if v != "-":
        for kv in v.split(","):
            key, val = kv.split("=")
            os.environ[key] = val

def run(fn, iters=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

res = {v: [] for v in variants + ["cublas"]}
for rnd in range(7):
    for v in variants:
        setenv(v)
        res[v].append(run(lambda: sb.gemm(a, b)))
    res["cublas"].append(run(lambda: torch.matmul(a, b)))
for v, ts in res.items():
    med = statistics.median(ts)
    print(f"{m}x{n}x{k} {v:28s} median {med*1e3:7.1f} us  {fl / med / 1e9:7.1f} TF  (min {fl / min(ts) / 1e9:7.1f})")
