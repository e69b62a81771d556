#!/usr/bin/env python
"""Benchmark of the hot path: the tensor-parallel MLP pair

    X shard --ag_gemm--> H --gemm_rs--> Y shard

on the Llama-3-70B MLP per-rank shapes of BASELINE.json (C3: AG+GEMM
ProblemShape(m=8192, n=28672/8=3584, k=8192); C4: GEMM+RS ProblemShape(m=8192,
n=8192, k=28672/8=3584)), bf16, synthetic data.  Weak scaling: every rank
runs that per-rank pair at TP=N (N=1: no peers, the gathers/scatters are local).

    python bench.py [--gpus N --steps K --warmup W]            (torchrun for N>1)
    python bench.py --impl reference ...                       (CPU oracle arm)

Prints ONE JSON line on rank 0.  `value` = whole-job TFLOPS (all ranks'
algorithmic FLOPs / max-over-ranks device time); `e2e` = the same through the
public API with host buffers (pinned H2D of X, D2H of Y inside the timed
region); `roofline` = the dominant kernel (the fused AG+GEMM call) against the
measured dense-bf16 peak; `cpu_baseline` = the reference package itself
(baseline/_ref) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("AG+GEMM / GEMM+RS TFLOPS/GPU & % roofline at TP=1/2/4/8 vs unfused cuBLAS+NCCL")
AG = dict(m=8192, n=3584, k=8192)   # C3 per-rank ProblemShape
RS = dict(m=8192, n=8192, k=3584)   # C4 per-rank ProblemShape
FALLBACK_PEAK_TFLOPS = 1590.0       # B200_PROFILING.md fallback (burst)


def flops(shape):
    return 2.0 * shape["m"] * shape["n"] * shape["k"]


STEP_FLOPS = flops(AG) + flops(RS)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps (capped at 50)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-unfused", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip the C5 TP/M sweep")
    p.add_argument("--no-proxy", action="store_true", help="skip the single-GPU TP=8 proxy")
    return p.parse_args()


FALLBACK_SUSTAINED_TFLOPS = 1400.0  # B200_PROFILING.md: sustained near 1.4 PFLOP/s


def peaks():
    """(burst, sustained, source) dense-bf16 peaks."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return (float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "measured (MEASURED_PEAKS.json)")
    except Exception:  # noqa: BLE001
        return (FALLBACK_PEAK_TFLOPS, FALLBACK_SUSTAINED_TFLOPS,
                "fallback (B200_PROFILING.md 1.59 / 1.4 PFLOP/s)")


def ncu_traffic():
    """dram read+write bytes per launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self, t0, t1):
        win = [p for t, p in self.samples if t0 - 0.1 <= t <= t1 + 0.1]
        if not win:
            win = [p for _, p in self.samples]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(p[0]) for p in win if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for p in win if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in win for i in range(4) if p[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(win)}


# ---------------------------------------------------------------------------
# The reference's CPU path (reference arm and cpu_baseline): the unmodified
# reference package (minishmem, pure Python + numpy) installed under
# baseline/_ref, driven through its own public API -- world.run of ag_gemm
# then gemm_rs -- in fp32 on all host cores, on a row sample
# of the per-rank C3/C4 shapes.  If baseline/_ref is missing, the numpy port
# of the same algorithm (oracle/minishmem_oracle.py) stands in ("port").

def _reference_package():
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "minishmem")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import minishmem  # noqa: F401
        from minishmem import core, pipelines, swizzle
    except Exception:  # noqa: BLE001 -- e.g. a missing dependency on the box
        return None
    return core, pipelines, swizzle


def cpu_sample_step(rows_sample, rng_seed=0):
    """(step(), flops per step, kind, teardown()) for a row sample."""
    import numpy as np

    g = np.random.default_rng(rng_seed)
    x = g.standard_normal((rows_sample, AG["k"]), dtype=np.float32)
    w_up = g.standard_normal((AG["k"], AG["n"]), dtype=np.float32) * 0.02
    w_dn = g.standard_normal((RS["k"], RS["n"]), dtype=np.float32) * 0.02
    fl = 2.0 * rows_sample * (AG["n"] * AG["k"] + RS["n"] * RS["k"])
    ref = _reference_package()
    if ref is not None:
        core, pipes, swz = ref
        ags = pipes.ProblemShape(m=rows_sample, n=AG["n"], k=AG["k"], dtype="float32")
        rss = pipes.ProblemShape(m=rows_sample, n=RS["n"], k=RS["k"], dtype="float32")
        heap = rows_sample * (AG["k"] + RS["n"]) * 4 + (1 << 20)
        world = core.init_world(core.WorldSpec(world_size=1, heap_bytes=heap, timeout_s=600.0))
        agb = pipes.make_ag_gemm_buffers(world, ags)
        rsb = pipes.make_gemm_rs_buffers(world, rss)

        def body(pe):
            h = pipes.ag_gemm(pe, x, w_up, ags, swz.ag_order_switch(pe.rank, 1), agb)
            return pipes.gemm_rs(pe, h, w_dn, rss, swz.rs_inter_order(pe.ctx, 1, 1), rsb)

        return (lambda: world.run(body)), fl, "reference", world.close
    from oracle import minishmem_oracle as oracle

    def step():
        (h,), _ = oracle.port_ag_gemm([x], [w_up], [[0]])
        (y,), _ = oracle.port_gemm_rs([h], [w_dn], [[0]])
        return y

    return step, fl, "port", lambda: None


def cpu_measure(steps, warmup, budget_s=20.0):
    """Calibrate the row sample so one step takes ~budget_s/(steps+warmup)
    (0.2..4 s), then time ``warmup`` untimed and ``steps`` timed steps."""
    rows = 256
    step, fl, kind, close = cpu_sample_step(rows)
    step()
    t0 = time.perf_counter()
    step()
    dt = time.perf_counter() - t0
    close()
    per_step_target = max(0.2, min(4.0, budget_s / max(1, steps + warmup)))
    rows = int(max(128, min(AG["m"], rows * per_step_target / max(dt, 1e-3))) // 128 * 128)
    step, fl, kind, close = cpu_sample_step(rows)
    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    close()
    cores = os.cpu_count()
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
    what = ("the reference package minishmem (baseline/_ref, unmodified): world.run of "
            "ag_gemm then gemm_rs" if kind == "reference" else
            "numpy port of the reference (oracle/minishmem_oracle.py): ag_gemm + gemm_rs")
    return {
        "value": fl / dt / 1e12, "unit": "TFLOPS",
        "cores": int(threads) if threads else cores, "kind": kind,
        "sample": (f"{what}, fp32, W=1, {rows} of {AG['m']} rows of the C3/C4 per-rank shapes, "
                   f"{warmup} warm-up + {steps} timed steps, {dt * 1e3:.1f} ms/step"),
        "ms_per_step": dt * 1e3,
    }


def run_reference(args, rank, world):
    if rank != 0:
        return
    steps, warm = max(1, args.steps), max(0, args.warmup)
    cb = cpu_measure(steps, warm, budget_s=150.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "TFLOPS",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": cb["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(world),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "TFLOPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(world):
    return {
        "workload": ("Llama-3-70B MLP TP pair per rank: ag_gemm ProblemShape(m=8192,n=3584,"
                     "k=8192) -> gemm_rs ProblemShape(m=8192,n=8192,k=3584), bf16"),
        "ag_shape": AG, "rs_shape": RS, "global_batch": AG["m"], "seq_len": None,
        "parallelism": f"tp{world}",
        "l2": "no flush: per-step working set ~0.55 GB > 126 MB L2",
    }


# ---------------------------------------------------------------------------

def main():
    args = parse()
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world_env != args.gpus:
        args.gpus = world_env if world_env > 1 else args.gpus
    if args.impl == "reference":
        return run_reference(args, rank, args.gpus)

    import torch
    import torch.distributed as dist

    import paper_2504_19442_b200 as sb
    from paper_2504_19442_b200 import _lib

    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    N = world_env
    # AG gather + RS staging + the comm probe's own gather buffer (N>1) + slack
    heap = (2 * AG["m"] * AG["k"] + RS["m"] * RS["n"]) * 2 + (64 << 20)
    if not args.no_sweep:
        heap += sweep_heap_bytes(world_env)
    if N > 1:
        # BENCH_BACKEND=gloo lets several ranks share one GPU (functional check
        # of the N>1 path; NCCL refuses duplicate GPUs)
        backend = os.environ.get("BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        world = sb.init_world_dist(heap_bytes=heap, timeout_s=30.0, device=local)
    else:
        world = sb.init_world(sb.WorldSpec(world_size=1, heap_bytes=heap, timeout_s=30.0,
                                           devices=(local,)))
    pe = world.pe(rank)
    dev = pe.torch_device
    ag_shape = sb.ProblemShape(dtype="bfloat16", **AG)
    rs_shape = sb.ProblemShape(dtype="bfloat16", **RS)
    agb = sb.make_ag_gemm_buffers(world, ag_shape)
    rsb = sb.make_gemm_rs_buffers(world, rs_shape)
    ag_sched = sb.ag_order_switch(rank, N)
    rs_sched = sb.rs_inter_order(world.ranks[rank], 1, N)
    rows = AG["m"] // N
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(rows, AG["k"], device=dev, generator=g).to(torch.bfloat16)
    w_up = (torch.randn(AG["k"], AG["n"], device=dev, generator=g) * 0.02).to(torch.bfloat16)
    w_dn = (torch.randn(RS["k"], RS["n"], device=dev, generator=g) * 0.02).to(torch.bfloat16)
    stream = pe.stream()

    # outputs written into preallocated buffers (out=): a step allocates
    # nothing, so the caching allocator never grows inside a timed loop
    h_buf = torch.empty((AG["m"], AG["n"]), dtype=torch.bfloat16, device=dev)
    y_ring = [torch.empty((rows, RS["n"]), dtype=torch.bfloat16, device=dev) for _ in range(2)]

    def step(xin, y_out=None):
        h = sb.ag_gemm(pe, xin, w_up, ag_shape, ag_sched, agb, reset=False, out=h_buf)
        return sb.gemm_rs(pe, h, w_dn, rs_shape, rs_sched, rsb, reset=False,
                          out=y_ring[0] if y_out is None else y_out)

    def barrier():
        torch.cuda.synchronize(dev)
        if N > 1:
            dist.barrier()

    def max_over_ranks(v):
        if N == 1:
            return v
        from paper_2504_19442_b200.dist import max_over_ranks as mor

        return mor(v, device=dev if dist.get_backend() == "nccl" else None)

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step(x)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        t_wall0 = time.time()
        ev0.record(stream)
        for _ in range(args.steps):
            step(x)
        ev1.record(stream)
        barrier()
        t_wall1 = time.time()
        ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
        # per-call split (the fused AG+GEMM call is the dominant kernel): each
        # op timed over its own back-to-back loop on the rank's stream
        k2 = min(args.steps, 50)
        h_fixed = sb.ag_gemm(pe, x, w_up, ag_shape, ag_sched, agb, reset=False)

        def loop_ms(fn):
            fn()  # one untimed call (first use of this operand / output set)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(k2):
                fn()
            e1.record(stream)
            barrier()
            return max_over_ranks(e0.elapsed_time(e1) / k2)

        ag_ms = loop_ms(lambda: sb.ag_gemm(pe, x, w_up, ag_shape, ag_sched, agb, reset=False,
                                           out=h_buf))
        rs_ms = loop_ms(lambda: sb.gemm_rs(pe, h_fixed, w_dn, rs_shape, rs_sched, rsb,
                                           reset=False, out=y_ring[1]))
    clk = clocks.summary(t_wall0, t_wall1)

    world.check_errors(rank)
    comm = measure_comm(sb, world, pe, N, rank, x, step, stream, barrier, max_over_ranks) \
        if N > 1 else None

    # ------------------------------------------------------------- baselines
    # measured right after our K-step block, before the PCIe-bound e2e phase
    # (which idles the SMs and lets the 1 kW power budget recover), so both
    # blocks run in the same sustained power state
    unfused = None
    if not args.no_unfused:
        try:
            with torch.cuda.stream(stream):
                if N > 1:
                    xg = torch.empty((AG["m"], AG["k"]), dtype=torch.bfloat16, device=dev)
                    ys = torch.empty((rows, RS["n"]), dtype=torch.bfloat16, device=dev)

                    def ustep():
                        dist.all_gather_into_tensor(xg, x)
                        hh = torch.matmul(xg, w_up)
                        yy = torch.matmul(hh, w_dn)
                        dist.reduce_scatter_tensor(ys, yy)
                else:
                    def ustep():
                        hh = torch.matmul(x, w_up)
                        torch.matmul(hh, w_dn)
                for _ in range(3):
                    ustep()
                barrier()
                u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                u0.record(stream)
                ku = args.steps  # same block length as the fused measurement
                for _ in range(ku):
                    ustep()
                u1.record(stream)
                barrier()
                ums = max_over_ranks(u0.elapsed_time(u1) / ku)

                # Interleaved A/B in the same power state.  After a switch the
                # 1 kW power controller needs ~100 steps to settle (the variant
                # that follows the lower-power one runs fast at first, the
                # other slow), so each block discards its first 100 steps and
                # times the next 200; order flips every round.
                def block(fn, settle=100, n=200):
                    b0, b1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                    barrier()
                    for _ in range(settle):
                        fn()
                    b0.record(stream)
                    for _ in range(n):
                        fn()
                    b1.record(stream)
                    barrier()
                    return max_over_ranks(b0.elapsed_time(b1) / n)

                ab_rounds = 4
                ab = {"ours": [], "unfused": []}
                for r in range(ab_rounds):
                    order = [("ours", lambda: step(x)), ("unfused", ustep)]
                    for name, fn in (order if r % 2 == 0 else order[::-1]):
                        ab[name].append(block(fn))
                o_ms = statistics.median(ab["ours"])
                u_ms = statistics.median(ab["unfused"])
            unfused = {"impl": "torch.matmul (cuBLASLt)" + (" + NCCL all_gather/reduce_scatter"
                                                            if N > 1 else ""),
                       "value": STEP_FLOPS * N / (ums * 1e-3) / 1e12, "unit": "TFLOPS",
                       "ms_per_step": ums,
                       "interleaved": {
                           "rounds": ab_rounds, "steps_per_block": "100 settle + 200 timed",
                           "ours_ms_per_step": o_ms, "unfused_ms_per_step": u_ms,
                           "ours_tflops": STEP_FLOPS * N / (o_ms * 1e-3) / 1e12,
                           "unfused_tflops": STEP_FLOPS * N / (u_ms * 1e-3) / 1e12,
                           "speedup": u_ms / o_ms,
                           "how": "median over blocks (100 settling steps, then 200 timed "
                                  "back-to-back steps), ours and unfused alternating, order "
                                  "flipped every round"}}
        except Exception as e:  # noqa: BLE001 -- e.g. gloo has no CUDA all_gather
            unfused = {"error": f"{type(e).__name__}: {e}"[:300]}

    # ------------------------------------------------------------------ e2e
    k_e2e = args.e2e_steps or min(args.steps, 50)
    x_host = x.cpu().pin_memory()
    y_host = torch.empty((rows, RS["n"]), dtype=torch.bfloat16).pin_memory()
    x_dev = [torch.empty_like(x) for _ in range(2)]
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    def e2e_loop(k):
        """k steps of the host->device->host pipeline; returns (e0, e1)."""
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done_h2d = [torch.cuda.Event() for _ in range(2)]
        done_use = [torch.cuda.Event() for _ in range(2)]
        done_d2h = [torch.cuda.Event() for _ in range(2)]
        for i in range(k):
            slot = i % 2
            h2d.wait_event(e0)
            if i >= 2:
                h2d.wait_event(done_use[slot])
            with torch.cuda.stream(h2d):
                x_dev[slot].copy_(x_host, non_blocking=True)
            done_h2d[slot].record(h2d)
            stream.wait_event(done_h2d[slot])
            if i >= 2:
                stream.wait_event(done_d2h[slot])  # y_ring[slot] read back
            with torch.cuda.stream(stream):
                yd = step(x_dev[slot], y_ring[slot])
            done_use[slot].record(stream)
            d2h.wait_stream(stream)
            with torch.cuda.stream(d2h):
                y_host.copy_(yd, non_blocking=True)
            done_d2h[slot].record(d2h)
        stream.wait_stream(d2h)
        e1.record(stream)
        barrier()
        return e0, e1

    # untimed warm-up of the same pipeline (pinned buffers, copy engines);
    # the loop itself allocates nothing: outputs go to a two-slot ring
    # (out=), each slot reused only after its D2H finished
    e2e_loop(3)
    e0, e1 = e2e_loop(k_e2e)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / k_e2e)
    # the PCIe floor of that loop: the same H2D of X and D2H of Y, both
    # directions at once on the same pinned buffers, no compute
    y_dev = torch.empty((rows, RS["n"]), dtype=torch.bfloat16, device=dev)
    barrier()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    h2d.wait_event(p0)
    d2h.wait_event(p0)
    for _ in range(5):
        with torch.cuda.stream(h2d):
            x_dev[0].copy_(x_host, non_blocking=True)
        with torch.cuda.stream(d2h):
            y_host.copy_(y_dev, non_blocking=True)
    stream.wait_stream(h2d)
    stream.wait_stream(d2h)
    p1.record(stream)
    barrier()
    pcie_ms = max_over_ranks(p0.elapsed_time(p1) / 5)

    # ------------------------------------------------------------- roofline
    burst, sustained, peak_src = peaks()
    proxy = None
    # (before the CPU baseline -- its BLAS threads compete with the proxy's
    # host pacer -- and the C5 sweep, which heats the GPU past the state of
    # the burst peak that is the proxy's roofline denominator)
    if rank == 0 and N == 1 and not args.no_proxy:
        # rank 0 of TP=8 at the C3/C4 per-rank shapes, peers emulated on this
        # GPU (tp_proxy.py); not a scaling number -- SCALE runs measure N>1
        try:
            import tp_proxy

            proxy = tp_proxy.run(W=8, iters=20, peak_tflops=burst, ab=False)
            proxy["label"] = "tp8_proxy"
            # the same per-rank kernels at TP=2 and TP=4 (C5's TP sweep on the
            # C3/C4 shapes): preset / paced time and roofline fraction per op
            lower = {}
            for Wl in (2, 4):
                r = tp_proxy.run(W=Wl, iters=8, peak_tflops=burst, ab=False)
                lower[f"tp{Wl}"] = {
                    "parity": r["parity"],
                    **{op: {k: r[op][k] for k in ("preset_us", "paced_us", "tflops", "roofline_us",
                                                  "roofline_frac", "speedup_vs_unfused_modelled")}
                       for op in ("ag", "rs")}}
            proxy["lower_tp"] = lower
        except Exception as e:  # noqa: BLE001 -- the proxy must never cost the headline line
            proxy = {"label": "tp8_proxy", "error": f"{type(e).__name__}: {e}"[:300]}
    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        cb = cpu_measure(steps=5, warmup=1, budget_s=20.0)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    sweep = None
    if not args.no_sweep:
        # short calls (a few ms each): the burst peak is the roofline denominator
        try:
            sweep = run_sweep(sb, world, pe, N, dev, stream, barrier, max_over_ranks, burst,
                              sustained)
            world.check_errors(rank)
        except Exception as e:  # noqa: BLE001 -- the sweep must never cost the headline line
            sweep = {"error": f"{type(e).__name__}: {e}"[:300]}
    dom_ms = ag_ms
    achieved = flops(AG) / (dom_ms * 1e-3) / 1e12
    # the roofline call is timed right after K back-to-back steps: under the
    # 1 kW cap (sw_power_cap seen) that is the sustained regime
    long_step = "sw_power_cap" in (clk.get("reasons") or [])
    peak = sustained if long_step else burst
    traffic = ncu_traffic().get("ag_gemm_kernel_dram_bytes")
    bn = (ctypes_query_tile(_lib, rows, N, AG["n"]))
    line = {
        "metric": METRIC,
        "value": STEP_FLOPS * N / (ms * 1e-3) / 1e12,
        "unit": "TFLOPS",
        "n_gpus": N, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random normal, seeded)",
        "config": workload_config(N),
        "tflops_per_gpu": STEP_FLOPS / (ms * 1e-3) / 1e12,
        "breakdown": {"ag_gemm_ms": ag_ms, "gemm_rs_ms": rs_ms,
                      "ag_gemm_tflops": flops(AG) / (ag_ms * 1e-3) / 1e12,
                      "gemm_rs_tflops": flops(RS) / (rs_ms * 1e-3) / 1e12,
                      "tile": bn},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "gemm_tp_kernel<MODE_AG> (fused ag_gemm call, CUDA events)",
                     "per_launch_flops": flops(AG),
                     "peak_source": f"{peak_src}, {'sustained' if long_step else 'burst'}",
                     "frac_of_burst": achieved / burst, "frac_of_sustained": achieved / sustained,
                     "per_launch_algorithmic_bytes": (AG["m"] * AG["k"] * 2 * 2 + AG["k"] * AG["n"] * 2
                                                      + AG["m"] * AG["n"] * 2)},
        "tp_roofline": tp_roofline(N, peak, ag_ms, rs_ms, ms),
        "e2e": {"value": STEP_FLOPS * N / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
                "h2d_bytes_per_step": x.numel() * 2, "d2h_bytes_per_step": rows * RS["n"] * 2,
                "ms_per_step": e2e_ms,
                "how": ("pinned X H2D + ag_gemm + gemm_rs + Y D2H per step, double-buffered, "
                        "outputs in a preallocated ring (out=)"),
                "pcie_floor_ms": pcie_ms,
                "pcie_duplex_gbs": (x.numel() + rows * RS["n"]) * 2 / (pcie_ms * 1e-3) / 1e9,
                "frac_of_pcie_floor": pcie_ms / e2e_ms},
        "unfused_baseline": unfused,
        "sweep": sweep,
        "tp8_proxy": proxy,
        "comm": comm,
        "cpu_baseline": cpu,
        "gpu_launches": args.steps * 2,
        "gpu_launches_note": ("per step: gemm_tp_kernel<MODE_AG> + gemm_tp_kernel<MODE_RS> "
                              "(RS reduction fused into the epilogue)"),
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    clocks.stop()
    world.close()
    if N > 1:
        dist.destroy_process_group()


NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def measure_comm(sb, world, pe, N, rank, x, step, stream, barrier, max_over_ranks, reps=10):
    """N>1: achieved NVLink rate of the AG push (the comm half on its own:
    allgather_push_intra of this rank's C3 shard into every peer, copy
    engine, waits for every slot) and the exposed communication of one fused
    step from the device timeline (CTA time spent waiting on remote chunks /
    peers' rows), both max over ranks."""
    import torch

    from paper_2504_19442_b200 import collectives, timeline

    out = {}
    try:
        with torch.cuda.stream(stream):
            agb_buf = world.alloc_symmetric(N * x.numel() * 2, align=1024)
            sigs = world.alloc_signals(N)
            ts = []
            for i in range(reps + 2):
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                collectives.allgather_push_intra(pe, agb_buf, sigs, x, wait_all=True, reset=True)
                e1.record(stream)
                barrier()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            t_ms = max_over_ranks(statistics.median(ts))
            moved = (N - 1) * x.numel() * 2
            out["ag_push"] = {"bytes_per_rank_each_way": moved, "ms": t_ms,
                              "gbs_per_direction": moved / (t_ms * 1e-3) / 1e9,
                              "frac_of_900": moved / (t_ms * 1e-3) / 900e9,
                              "how": "allgather_push_intra of the C3 shard (copy engine, one flag per "
                                     "slot), all ranks at once, median of 10, max over ranks"}
    except Exception as e:  # noqa: BLE001 -- the comm probe must never cost the headline line
        out["ag_push"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    try:
        with torch.cuda.stream(stream):
            world.start_trace()
            step(x)
            barrier()
            ev = world.stop_trace()
        summ = timeline.exposed_comm(ev)
        # (rs_reduce: the separate reduction kernel of the RS on separate GPUs;
        # every rank runs the same kernels, so the collectives below match)
        for kern in ("ag_gemm", "gemm_rs", "rs_reduce"):
            rows_ = [s_ for s_ in summ if s_["kernel"] == kern]
            if rows_:
                r_ = rows_[-1]
                out[kern] = {"exposed_wait_max_us": max_over_ranks(r_["wait_max_us"]),
                             "exposed_wait_mean_us": max_over_ranks(r_["wait_mean_us"]),
                             "span_us": max_over_ranks(r_["span_us"] or 0.0)}
        out["exposed_how"] = ("device timeline of one traced step: per CTA, time spent waiting "
                              "for a remote chunk (AG) / peers' rows (fused RS epilogue, or the "
                              "separate reduction kernel rs_reduce); max over ranks")
    except Exception as e:  # noqa: BLE001
        out["exposed_error"] = f"{type(e).__name__}: {e}"[:300]
    return out

# C5 of BASELINE.json: TP sweep over M for both ops (Llama-3-70B MLP, N=28672,
# K=8192 hidden): AG ProblemShape(M, 28672/TP, 8192), RS ProblemShape(M, 8192, 28672/TP)
SWEEP_M = (1024, 4096, 16384)
FFN, HID = 28672, 8192


def sweep_shapes(tp):
    for M in SWEEP_M:
        yield "ag_gemm", M, dict(m=M, n=FFN // tp, k=HID)
        yield "gemm_rs", M, dict(m=M, n=HID, k=FFN // tp)


def sweep_heap_bytes(tp):
    return sum(s["m"] * (s["k"] if op == "ag_gemm" else s["n"]) * 2 + (1 << 20)
               for op, _, s in sweep_shapes(tp))


def run_sweep(sb, world, pe, N, dev, stream, barrier, max_over_ranks, peak, peak_sustained=None):
    """Both fused ops against the unfused cuBLAS (+ NCCL at N>1) sequence at
    TP=N for every M of C5; per point TFLOPS/GPU and the fraction of the
    BASELINE roofline max(GEMM at the tensor peak, shard bytes over NVLink)."""
    import torch
    import torch.distributed as dist

    rank = pe.rank
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    w_up = (torch.randn(HID, FFN // N, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    w_dn = (torch.randn(FFN // N, HID, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    ag_sched = sb.ag_order_switch(rank, N)
    rs_sched = sb.rs_inter_order(world.ranks[rank], 1, N)
    out = []
    for op, M, s in sweep_shapes(N):
        shape = sb.ProblemShape(dtype="bfloat16", **s)
        fl = flops(s)
        iters = int(max(5, min(30, 0.08 / (fl / 1.2e15))))
        if op == "ag_gemm":
            bufs = sb.make_ag_gemm_buffers(world, shape)
            x = torch.randn(M // N, HID, device=dev, generator=g).to(torch.bfloat16)
            ours = lambda: sb.ag_gemm(pe, x, w_up, shape, ag_sched, bufs, reset=False)  # noqa: E731
            if N > 1:
                xg = torch.empty((M, HID), dtype=torch.bfloat16, device=dev)

                def unfused():
                    dist.all_gather_into_tensor(xg, x)
                    torch.matmul(xg, w_up)
            else:
                unfused = lambda: torch.matmul(x, w_up)  # noqa: E731
            nvl_bytes = (N - 1) / N * M * HID * 2
        else:
            bufs = sb.make_gemm_rs_buffers(world, shape)
            a = torch.randn(M, FFN // N, device=dev, generator=g).to(torch.bfloat16)
            ours = lambda: sb.gemm_rs(pe, a, w_dn, shape, rs_sched, bufs, reset=False)  # noqa: E731
            if N > 1:
                ys = torch.empty((M // N, HID), dtype=torch.bfloat16, device=dev)

                def unfused():
                    dist.reduce_scatter_tensor(ys, torch.matmul(a, w_dn))
            else:
                unfused = lambda: torch.matmul(a, w_dn)  # noqa: E731
            nvl_bytes = (N - 1) / N * M * HID * 2

        def timed(fn):
            with torch.cuda.stream(stream):
                for _ in range(3):
                    fn()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(iters):
                    fn()
                e1.record(stream)
                barrier()
            return max_over_ranks(e0.elapsed_time(e1) / iters)

        # three interleaved rounds, median per implementation: the GPU's power
        # state drifts between back-to-back measurements
        t_ours, t_unf = [], []
        for _ in range(3):
            t_ours.append(timed(ours))
            t_unf.append(timed(unfused))
        ms_ours, ms_unf = statistics.median(t_ours), statistics.median(t_unf)
        t_gemm = fl / (peak * 1e12) * 1e3
        t_nvl = nvl_bytes / (NVLINK_GBS * 1e9) * 1e3
        roof = max(t_gemm, t_nvl)
        out.append({"op": op, "tp": N, "M": M, "shape": s, "iters": iters, "rounds": 3,
                    "ours_us": ms_ours * 1e3, "unfused_us": ms_unf * 1e3,
                    "ours_tflops_per_gpu": fl / (ms_ours * 1e-3) / 1e12,
                    "unfused_tflops_per_gpu": fl / (ms_unf * 1e-3) / 1e12,
                    "bound": "tensor" if t_gemm >= t_nvl else "nvlink",
                    "roofline_frac": roof / ms_ours, "unfused_roofline_frac": roof / ms_unf,
                    "roofline_frac_sustained_peak": (
                        max(fl / (peak_sustained * 1e12) * 1e3, t_nvl) / ms_ours
                        if peak_sustained else None)})
        del bufs
    return out


def tp_roofline(n_gpus, peak_tflops, ag_ms, rs_ms, step_ms):
    """BASELINE.json's roofline: per op the slower of the GEMM at the tensor
    peak and the shard bytes that must cross NVLink (AG in: (TP-1)/TP*M*K*2,
    RS out: (TP-1)/TP*M*N*2), and the measured fraction of it."""
    tp = n_gpus
    t_gemm_ag = flops(AG) / (peak_tflops * 1e12) * 1e6
    t_gemm_rs = flops(RS) / (peak_tflops * 1e12) * 1e6
    t_nvl_ag = (tp - 1) / tp * AG["m"] * AG["k"] * 2 / (NVLINK_GBS * 1e9) * 1e6
    t_nvl_rs = (tp - 1) / tp * RS["m"] * RS["n"] * 2 / (NVLINK_GBS * 1e9) * 1e6
    r_ag, r_rs = max(t_gemm_ag, t_nvl_ag), max(t_gemm_rs, t_nvl_rs)
    return {
        "ag": {"t_gemm_us": t_gemm_ag, "t_nvlink_us": t_nvl_ag,
               "bound": "tensor" if t_gemm_ag >= t_nvl_ag else "nvlink",
               "measured_us": ag_ms * 1e3, "frac": r_ag / (ag_ms * 1e3)},
        "rs": {"t_gemm_us": t_gemm_rs, "t_nvlink_us": t_nvl_rs,
               "bound": "tensor" if t_gemm_rs >= t_nvl_rs else "nvlink",
               "measured_us": rs_ms * 1e3, "frac": r_rs / (rs_ms * 1e3)},
        "step_frac": (r_ag + r_rs) / (step_ms * 1e3),
        "peak_tflops": peak_tflops, "nvlink_gbs": NVLINK_GBS,
    }


def ctypes_query_tile(_lib, rows, world, n):
    import ctypes

    bn, cg, grid = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.load().sh_query_tile_config(rows, world, n, ctypes.byref(bn), ctypes.byref(cg),
                                     ctypes.byref(grid))
    return {"bn": bn.value, "cta_group": cg.value, "grid": grid.value}


if __name__ == "__main__":
    main()
