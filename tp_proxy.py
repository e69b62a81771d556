"""Single-GPU proxy of one tensor-parallel rank (bench.py ``tp8_proxy``).

The gpurun pool grants one B200 per call, so the TP=8 per-rank
configuration of the north star (BASELINE C3 / C4: reference
pipelines.py:126-144 and :201-216 at W=8) cannot run on NVLink here.  This
proxy runs rank 0's REAL kernels at that configuration -- W=8 chunking, 7
flag-gated remote chunks, 7 peer destinations, the 8-slot fused reduction --
with the full persistent grid (``sh_set_rank_solo``), while the 7 peers are
emulated on the same GPU:

* the peers' data is placed in rank 0's symmetric buffers once, up front (AG:
  ``gathered`` slots 1..7; RS: ``staging`` slots 1..7 -- the kernel reads
  them, nobody else writes them);
* the peers' FLAGS are released during the call by stream memory operations
  (front-end writes, no SM involved) on a feeder stream, each gated on a tick
  of a host pacer (``sh_pace_host``: a host thread spinning on the clock,
  started by a word the main stream writes right before the launch), so each
  flag opens when the data would have landed:
  - AG: the owners push in ring order (``ag_push_order``), so rank 0 receives
    one shard at a time over its NVLink ingress and ``ready[src]`` of the
    chunk consumed at step i opens at ``i * chunk_bytes / bw``;
  - RS: peer s handles rank 0's chunk at position ``pos = (-s-1) mod W`` of
    its ``rs_inter_order``; with symmetric ranks it completes that chunk when
    rank 0 completes its own position-``pos`` chunk, which a traced preset
    call measures (the last tile's stores of each chunk, ``calibrate_rs``),
    so ``reduction[s]`` opens then;
* back-pressure words (``done`` / ``producer``) are saturated: no peer ever
  holds rank 0 back.

Why flags only, and why a host pacer: a same-device cudaMemcpyAsync may run
as a copy kernel on the SMs, which cannot co-reside with a persistent GEMM
using all of them (a feeder that copied data during the call stalled until the
GEMM's timeout), and pacing with host->device copies slowed the RS kernel's
epilogues by up to 30 us a tile -- the pacing has to stay off the SMs and the
copy engines.  What the proxy therefore leaves out: the HBM write traffic of
the incoming shards (7 x 16 MB per op) and NVLink contention / peer skew.
The pacer's release latency (host store -> front-end wait -> flag) is
calibrated with an idle GPU and taken off the schedule (``calibrate``), and
the release times of every paced call are recorded next to the schedule
(``arrivals``).

Modes: ``preset`` = every flag set before the launch (the kernel alone,
safe under ncu); ``paced`` = flags on the NVLink schedule (exposed
communication = paced - preset, cross-checked by the device timeline).
"""

from __future__ import annotations

import ctypes
import statistics

import torch

import paper_2504_19442_b200 as sb
from paper_2504_19442_b200 import _lib

NVLINK_BW = 770e9  # per-direction NVLink 5 rate used across DESIGN.md


def _sub_ranges(rows, S):
    """The library's sub-chunk row ranges (sh_ag_gemm_ex: multiples of 256)."""
    if S <= 1:
        return [(0, rows)]
    sub = ((rows + S - 1) // S + 255) // 256 * 256
    return [(r0, min(sub, rows - r0)) for r0 in range(0, rows, sub)]


class TpProxy:
    """Rank 0 of a W-rank world on one GPU, peers emulated by flag releases."""

    def __init__(self, W, m, n_ag, k_ag, n_rs, k_rs, *, bw=NVLINK_BW, seed=0, timeout_s=20.0):
        self.W = W
        self.bw = bw
        self.ag = sb.ProblemShape(m, n_ag, k_ag, dtype="bfloat16")
        self.rs = sb.ProblemShape(m, n_rs, k_rs, dtype="bfloat16")
        rows = m // W
        self.rows = rows
        heap = W * rows * (k_ag + n_rs) * 2 + (8 << 20)
        self.world = sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=heap, timeout_s=timeout_s,
                                                devices=(0,) * W))
        w = self.world
        self.lib = _lib.load()
        _lib.check(self.lib.sh_set_rank_solo(w.handle, 0, 1))
        self.agb = sb.make_ag_gemm_buffers(w, self.ag)
        self.rsb = sb.make_gemm_rs_buffers(w, self.rs)
        dev = torch.device("cuda", 0)
        g = torch.Generator(device=dev).manual_seed(seed)
        bf = torch.bfloat16
        self.x = torch.randn(W, rows, k_ag, device=dev, dtype=bf, generator=g)  # every rank's shard
        self.b_ag = torch.randn(k_ag, n_ag, device=dev, dtype=bf, generator=g) / k_ag ** 0.5
        self.a_rs = torch.randn(m, k_rs, device=dev, dtype=bf, generator=g)
        self.b_rs = torch.randn(k_rs, n_rs, device=dev, dtype=bf, generator=g) / k_rs ** 0.5
        self.peer_rows = torch.randn(W, rows, n_rs, device=dev, dtype=bf, generator=g)
        self.c = torch.empty(m, n_ag, device=dev, dtype=bf)
        self.y = torch.empty(rows, n_rs, device=dev, dtype=bf)
        self.main = torch.cuda.Stream(device=dev)
        # one feeder stream per peer: a stream memory op costs ~7 us of
        # front-end time, so 7 releases queued on one stream could not be
        # closer than that (small-M shards land every ~3 us)
        self.feeds = [torch.cuda.Stream(device=dev) for _ in range(W)]
        self.feed = self.feeds[0]
        # peers' data, placed once (see module doc)
        gath = w.heap_view(0, self.agb.gathered, bf, (W, rows, k_ag))
        stag = w.heap_view(0, self.rsb.staging, bf, (W, rows, n_rs))
        torch.cuda.synchronize(dev)
        gath[1:].copy_(self.x[1:])
        stag[1:].copy_(self.peer_rows[1:])
        torch.cuda.synchronize(dev)
        self.ag_order = sb.ag_order_switch(0, W).first_visit_order(W)
        self.rs_order = sb.rs_inter_order(sb.RankCtx(0, 0, 0), 1, W).first_visit_order(W)
        fs = ctypes.c_void_p(self.feed.cuda_stream)
        for base in (self.agb.done.base, self.rsb.producer.base):
            _lib.check(self.lib.sh_fill_signals(w.handle, 0, base, W, 1 << 62, fs))
        self._feeds_sync()
        # pinned words: [0] go (the host writes it once a call is fully
        # enqueued, so the timed region never holds host launch latency),
        # [1] origin (the main stream writes it right before a paced launch),
        # [2] tick (the host pacer)
        self.words = torch.zeros(3, dtype=torch.int64, pin_memory=True)
        self._go = 0
        self._origin_val = 0
        self._tick = 0
        self.release_lat_ns = 0.0
        self.ag_epoch = 0
        self.rs_epoch = 0
        self.rs_done_us = None       # per schedule position: rank 0's chunk completion
        self.diag = None            # feeder events after each release (arrival diagnostics)
        from paper_2504_19442_b200.core import serialising_tool

        self.tool = serialising_tool()

    def close(self):
        self.world.close()

    # ------------------------------------------------------------------ pacing
    def _word(self, i):
        return ctypes.c_void_p(self.words.data_ptr() + 8 * i)

    def _release(self, rank_from, sig, value, tick):
        """Feeder: (wait for the pacer's tick) then set rank 0's signal word."""
        feed = self.feeds[rank_from % len(self.feeds)]
        fs = ctypes.c_void_p(feed.cuda_stream)
        if tick is not None:
            _lib.check(self.lib.sh_stream_wait_word(self._word(2), tick, fs))
        _lib.check(self.lib.sh_signal_op(self.world.handle, rank_from, 0, sig, _lib.SH_SIG_SET, value, fs))
        if self.diag is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(feed)
            self.diag.append(ev)

    def _feeds_sync(self):
        for f in self.feeds:
            f.synchronize()

    def _call(self, mode, releases, launch):
        """One call: ``releases`` = [(rank_from, sig, value, delta_us)].
        preset: every flag before the launch.  paced: the feeder's releases
        wait on host-pacer ticks; the pacer starts on the origin word the
        main stream writes right before the launch."""
        import threading

        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        ms = ctypes.c_void_p(self.main.cuda_stream)
        self._go += 1
        pacer, rc = None, []
        for f in self.feeds:
            f.wait_stream(self.main)
        if mode == "preset":
            for r_from, sig, val, _d in releases:
                self._release(r_from, sig, val, None)
            for f in self.feeds:
                self.main.wait_stream(f)
        else:
            self._origin_val += 1
            base = self._tick
            self._tick += len(releases)
            lat = self.release_lat_ns
            arr = (ctypes.c_uint64 * max(1, len(releases)))(
                *[int(max(0.0, d * 1e3 - lat)) for *_x, d in releases])
            for i, (r_from, sig, val, _d) in enumerate(releases):
                self._release(r_from, sig, val, base + i + 1)
            origin = self._origin_val
            pacer = threading.Thread(target=lambda: rc.append(self.lib.sh_pace_host(
                self._word(1), origin, self._word(2), base, arr, len(releases), 30.0)))
            pacer.start()
        if not self.tool:
            # (a kernel-serialising tool returns from the launch only after the
            # kernel ran: a gate the host opens after the launch would hang it)
            _lib.check(self.lib.sh_stream_wait_word(self._word(0), self._go, ms))
        if mode == "paced":
            _lib.check(self.lib.sh_stream_write_word(self._word(1), self._origin_val, ms))
        start.record(self.main)
        if launch is not None:
            launch(ms)
        end.record(self.main)
        self.words[0] = self._go
        if pacer is not None:
            pacer.join()
            _lib.check(rc[0] if rc else _lib.SH_ERR_STATE)
        return start, end

    # ------------------------------------------------------------------ AG
    def _ag_call(self, mode, subchunks, kernel=True):
        W, lib, w, sh = self.W, self.lib, self.world, self.ag
        rows, k = self.rows, sh.k
        self.ag_epoch += 1
        e = self.ag_epoch
        S = subchunks if subchunks else self._auto_sub()
        ranges = _sub_ranges(rows, S)
        S_eff = len(ranges)
        # the chunk consumed at step i lands at i * chunk / bw (one ingress)
        releases, landed = [], 0
        for step in range(1, W):
            c = self.ag_order[step]
            for j, (_r0, nr) in enumerate(ranges):
                landed += nr * k * 2
                releases.append((c, self.agb.ready.base + c, (e - 1) * S_eff + j + 1,
                                 landed / self.bw * 1e6))
        order = _lib.int_array(self.ag_order)
        launch = (lambda ms: _lib.check(lib.sh_ag_gemm_ex(
            w.handle, 0, self.x[0].data_ptr(), self.b_ag.data_ptr(), self.c.data_ptr(),
            self.agb.gathered.offset, self.agb.ready.base, self.agb.done.base, sh.m, sh.n, sh.k,
            sh.dtype_code, order, e, S, _lib.SH_PHASE_COMPUTE, ms))) if kernel else None
        return self._call(mode, releases, launch)

    def _auto_sub(self):
        out = ctypes.c_int()
        _lib.check(self.lib.sh_ag_subchunks(self.ag.m, self.ag.k, self.W, ctypes.byref(out)))
        return out.value

    # ------------------------------------------------------------------ RS
    def _rs_call(self, mode, kernel=True):
        W, lib, w, sh = self.W, self.lib, self.world, self.rs
        rows, n = self.rows, sh.n
        self.rs_epoch += 1
        e = self.rs_epoch
        # peer s handles chunk 0 at position (0 - s - 1) mod W of rs_inter_order
        done = self.rs_done_us or [0.0] * W
        releases = [(s, self.rsb.reduction.base + s, e * rows * n, done[pos])
                    for pos, s in sorted(((-s - 1) % W, s) for s in range(1, W))]
        order = _lib.int_array(self.rs_order)
        launch = (lambda ms: _lib.check(lib.sh_gemm_rs_ex(
            w.handle, 0, self.a_rs.data_ptr(), self.b_rs.data_ptr(), self.y.data_ptr(),
            self.rsb.staging.offset, self.rsb.producer.base, self.rsb.reduction.base, sh.m, sh.n,
            sh.k, sh.dtype_code, order, e, _lib.SH_PHASE_ALL, ms))) if kernel else None
        return self._call(mode, releases, launch)

    # ------------------------------------------------------------------ driver
    def _ensure_rs_estimate(self):
        if self.rs_done_us is None:
            self.calibrate_rs()

    def calibrate_rs(self):
        """Completion time of each of rank 0's chunk positions in a traced
        preset call (latest tile-store issue of the chunk after the first CTA
        start): by symmetry, when a peer finishes the chunk at that position."""
        self.rs_done_us = [0.0] * self.W
        self.time_op("rs", "preset", 3)
        self.world.start_trace(records_per_cta=1024, launches=2)
        try:
            self.time_op("rs", "preset", 1, warmup=0)
        finally:
            ev = self.world.stop_trace()
        # the GEMM's launch (the separate reduction kernel is traced too)
        last = max(e["launch"] for e in ev if e["rank"] == 0 and e["kernel"] == "gemm_rs")
        ev = [e for e in ev if e["rank"] == 0 and e["launch"] == last]
        t0 = min(e["t0_ns"] for e in ev if e["op"] == "cta")
        end = {}
        for e in ev:
            if e["op"] == "tile_epilogue":
                end[e["chunk"]] = max(end.get(e["chunk"], 0), e["t1_ns"] - t0)
        self.rs_done_us = [end.get(c, 0) / 1e3 for c in self.rs_order]
        return self.rs_done_us

    def time_op(self, op, mode, iters, warmup=3, subchunks=0):
        if op == "rs" and mode == "paced":
            self._ensure_rs_estimate()
        call = (lambda: self._ag_call(mode, subchunks)) if op == "ag" else (lambda: self._rs_call(mode))
        evs = []
        for i in range(warmup + iters):
            ev = call()
            if i >= warmup:
                evs.append(ev)
        self.main.synchronize()
        self._feeds_sync()
        self.world.check_errors(0)
        return [a.elapsed_time(b) * 1e3 for a, b in evs]  # us

    def arrivals(self, op, subchunks=0, kernel=True):
        """Flag release times (us after the timed start) of one paced call."""
        if op == "rs":
            self._ensure_rs_estimate()
        self.diag = []
        try:
            start, end = (self._ag_call("paced", subchunks, kernel) if op == "ag"
                          else self._rs_call("paced", kernel))
            self.main.synchronize()
            self._feeds_sync()
            self.world.check_errors(0)
            return {"kernel_us": start.elapsed_time(end) * 1e3,
                    "released_us": [round(start.elapsed_time(ev) * 1e3, 1) for ev in self.diag]}
        finally:
            self.diag = None

    def calibrate(self, reps=5, spacing_us=30.0):
        """Release latency of the host pacer (tick due -> flag written),
        measured with no kernel running: 7 releases 30 us apart (more than
        a release's own front-end cost, ~7 us), median lateness."""
        rel = [(1, self.agb.ready.base + 1, 0, spacing_us * (i + 1)) for i in range(7)]
        self.release_lat_ns = 0.0
        late = []
        for _ in range(reps):
            self.diag = []
            try:
                start, _end = self._call("paced", rel, None)
                self._feeds_sync()
                self.main.synchronize()
                late += [start.elapsed_time(ev) * 1e3 - d for ev, (*_x, d) in zip(self.diag, rel)]
            finally:
                self.diag = None
        self.world.zero_signals(0, self.agb.ready.base, self.W)
        self.release_lat_ns = max(0.0, statistics.median(late) * 1e3)
        # the same schedule once more, latency taken off
        self.diag = []
        try:
            start, _end = self._call("paced", rel, None)
            self._feeds_sync()
            self.main.synchronize()
            err = [start.elapsed_time(ev) * 1e3 - d for ev, (*_x, d) in zip(self.diag, rel)]
        finally:
            self.diag = None
        self.world.zero_signals(0, self.agb.ready.base, self.W)
        return {"release_latency_us": self.release_lat_ns / 1e3,
                "lateness_spread_us": [round(min(late), 1), round(max(late), 1)],
                "residual_err_us": [round(x, 1) for x in err]}

    def check(self):
        """Rank 0's results against torch fp32 (rel-Frobenius, north-star 1e-2)
        after paced calls, plus the gathered layout bit for bit."""
        self._ensure_rs_estimate()
        self.time_op("ag", "paced", 1, warmup=0)
        ref = self.x.reshape(-1, self.ag.k).float() @ self.b_ag.float()
        err_ag = ((self.c.float() - ref).norm() / ref.norm()).item()
        self.time_op("rs", "paced", 1, warmup=0)
        part = self.a_rs[: self.rows].float() @ self.b_rs.float()
        ref = part.to(torch.bfloat16).float() + self.peer_rows[1:].float().sum(0)
        err_rs = ((self.y.float() - ref).norm() / ref.norm()).item()
        g = self.world.read_tensor(0, self.agb.gathered, torch.bfloat16, (self.W * self.rows, self.ag.k))
        layout_ok = bool(torch.equal(g.to(self.x.device), self.x.reshape(-1, self.ag.k)))
        return {"ag_rel_fro": err_ag, "rs_rel_fro": err_rs, "gathered_bit_exact": layout_ok}

    def trace_waits(self, op, subchunks=0, detail=False, mode="paced"):
        """One traced paced call: exposed waits per CTA from the device timeline."""
        from paper_2504_19442_b200 import timeline

        self.world.start_trace()
        try:
            self.time_op(op, mode, 1, warmup=0, subchunks=subchunks)
        finally:
            ev = self.world.stop_trace()
        summ = [s for s in timeline.exposed_comm(ev) if s["rank"] == 0]
        if not summ:
            return None
        out = dict(summ[-1])
        last = max(e["launch"] for e in ev if e["rank"] == 0)
        per = {}
        for e in ev:
            if e["rank"] == 0 and e["launch"] == last and e["op"] in ("chunk_wait", "peer_wait"):
                per[e["cta"]] = per.get(e["cta"], 0) + (e["t1_ns"] - e["t0_ns"]) / 1e3
        out["ctas_waiting"] = sum(1 for v in per.values() if v > 1.0)
        out["top_waits_us"] = sorted((round(v, 1) for v in per.values()), reverse=True)[:8]
        ctas = [e for e in ev if e["rank"] == 0 and e["launch"] == last and e["op"] == "cta"]
        if ctas:
            t0 = min(e["t0_ns"] for e in ctas)
            ends = sorted((e["t1_ns"] - t0) / 1e3 for e in ctas)
            out["cta_end_us"] = {"min": round(ends[0], 1), "median": round(ends[len(ends) // 2], 1),
                                 "max": round(ends[-1], 1)}
            if detail:
                out["per_cta"] = {e["cta"]: [round((e["t1_ns"] - t0) / 1e3, 1),
                                             round(per.get(e["cta"], 0.0), 1)] for e in ctas}
        return out


def cublas_us(m, n, k, iters=30, warmup=5):
    """torch.matmul (cuBLASLt) of one rank's GEMM, CUDA events, median."""
    dev = torch.device("cuda", 0)
    a = torch.randn(m, k, device=dev, dtype=torch.bfloat16)
    b = torch.randn(k, n, device=dev, dtype=torch.bfloat16)
    out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    ts = []
    for i in range(warmup + iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=out)
        e.record()
        if i >= warmup:
            ts.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) * 1e3 for x, y in ts)


def run(W=8, m=8192, iters=30, peak_tflops=None, ab=True):
    """The tp8_proxy block of bench.py: C3 AG and C4 RS at TP=W, rank 0."""
    import os

    k_full, n_full = 8192, 28672  # Llama-3-70B MLP (BASELINE C3/C4)
    px = TpProxy(W, m, n_full // W, k_full, k_full, n_full // W)
    try:
        out = {"what": f"single-GPU proxy of rank 0 at TP={W} (tp_proxy.py): real kernels at the "
                       f"per-rank shapes, peers' data pre-placed, their flags released on the "
                       f"NVLink schedule ({NVLINK_BW / 1e9:.0f} GB/s ingress; RS: when a symmetric "
                       f"peer finishes the chunk) by a host pacer",
               "W": W, "ag_shape": {"m": m, "n": n_full // W, "k": k_full},
               "rs_shape": {"m": m, "n": k_full, "k": n_full // W},
               "pacing": px.calibrate()}
        out["parity"] = px.check()
        flops = 2.0 * m * (n_full // W) * k_full
        nvl_bytes = (W - 1) / W * m * k_full * 2
        for op in ("ag", "rs"):
            pre = statistics.median(px.time_op(op, "preset", iters))
            paced = statistics.median(px.time_op(op, "paced", iters))
            r = {"preset_us": pre, "paced_us": paced, "exposed_us": paced - pre,
                 "tflops": flops / paced / 1e6}
            if peak_tflops:
                t_gemm = flops / (peak_tflops * 1e12) * 1e6
                t_nvl = nvl_bytes / 900e9 * 1e6
                r["roofline_us"] = max(t_gemm, t_nvl)
                r["roofline_frac"] = r["roofline_us"] / paced
            r["trace"] = px.trace_waits(op)
            r["exposed_comm_us_timeline"] = r["trace"]["wait_max_us"] if r["trace"] else None
            if op == "rs":
                r["release_schedule_us"] = [round(x, 1) for x in px.rs_done_us]
            r["arrivals"] = px.arrivals(op)
            out[op] = r
        if ab:
            out["ag"]["trace_preset"] = px.trace_waits("ag", detail=True, mode="preset")
            # sub-chunk flags and the weighted stream-K partition on the paced AG
            res = {}
            for label, env, sub in (("sub1", None, 1), ("sub4", None, 4), ("sub1_nolate", "0,0", 1)):
                if env is None:
                    os.environ.pop("SHB_SK_LATE", None)
                else:
                    os.environ["SHB_SK_LATE"] = env
                res[label] = statistics.median(px.time_op("ag", "paced", iters, subchunks=sub))
            os.environ.pop("SHB_SK_LATE", None)
            out["ag"]["ab_paced_us"] = res
        # unfused: cuBLAS of the same per-rank GEMM + the collective's bytes at
        # the same NVLink rate (modelled: no NCCL peers on a one-GPU box)
        t_comm = nvl_bytes / NVLINK_BW * 1e6
        out["ag"]["unfused_modelled_us"] = cublas_us(m, n_full // W, k_full) + t_comm
        out["rs"]["unfused_modelled_us"] = cublas_us(m, k_full, n_full // W) + t_comm
        for op in ("ag", "rs"):
            out[op]["speedup_vs_unfused_modelled"] = out[op]["unfused_modelled_us"] / out[op]["paced_us"]
        out["unfused_how"] = (f"torch.matmul of the per-rank GEMM (measured) + {nvl_bytes / 1e6:.1f} MB "
                              f"at {NVLINK_BW / 1e9:.0f} GB/s (modelled NCCL transfer, not overlapped)")
        return out
    finally:
        px.close()


if __name__ == "__main__":
    import json
    import sys

    # python tp_proxy.py [iters] [W ...]: one JSON line per TP degree (the
    # per-rank C3 / C4 shapes at TP=W: AG (8192, 28672/W, 8192), RS (8192,
    # 8192, 28672/W)), peak = MEASURED_PEAKS.json burst bf16
    import os

    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    worlds = [int(x) for x in sys.argv[2:]] or [8]
    peak = 1700.9
    mp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peak = json.load(open(mp)).get("bf16_tflops", peak)
    for W in worlds:
        sys.stdout.write(json.dumps(run(W=W, iters=iters, peak_tflops=peak, ab=False)) + "\n")
        sys.stdout.flush()
